"""Multi-GPU topology sharding (one process per GPU, torch.distributed).

Tasks are independent units solved against a replicated, immutable base
(the reference solves them in isolation too, `solver.py:977-1002`; the paper
runs independent GPUs with "no cross-device communication during the solving
process", `PAPER.md:458`).  So a batch is split into contiguous task ranges,
each rank solves its range on its own GPU with no collective on the data
path, and only the per-task results are exchanged afterwards: an all-gather
of (metric, winner, feasibility, status) and the sparse report entries
(NCCL over NVLink on GPUs, gloo on CPU for the tests).
"""

from __future__ import annotations

from typing import Callable, Optional

import numpy as np

# per-task result arrays exchanged after the solve (first axis = task)
RESULT_FIELDS = (
    "metric", "best", "feasible", "status", "status_arg", "n_islanded", "islanded_bits",
    "n0_count", "n0_pos", "n0_flow", "n0_rel", "n1_count", "n1_case", "n1_pos", "n1_flow", "n1_rel",
)


def shard_range(n_tasks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [start, stop) task range of one rank."""
    base, extra = divmod(n_tasks, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _torch_dtype(np_dtype):
    import torch

    return {
        np.dtype(np.float64): torch.float64,
        np.dtype(np.float32): torch.float32,
        np.dtype(np.int64): torch.int64,
        np.dtype(np.int32): torch.int32,
        np.dtype(np.uint32): torch.int32,
        np.dtype(np.uint8): torch.uint8,
        np.dtype(np.bool_): torch.uint8,
    }[np.dtype(np_dtype)]


def all_gather_tasks(local: dict, n_tasks: int, group=None, device=None) -> dict:
    """All-gather per-task arrays (first axis = this rank's shard) into full-batch arrays.

    Shards are padded to the largest shard so one ``all_gather_into_tensor`` per
    field suffices; the padding is dropped on unpack.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [shard_range(n_tasks, r, world) for r in range(world)]
    width = max(b - a for a, b in sizes)
    out = {}
    for name, arr in local.items():
        arr = np.ascontiguousarray(arr)
        view = arr.view(np.int32) if arr.dtype == np.uint32 else (arr.view(np.uint8) if arr.dtype == np.bool_ else arr)
        pad = np.zeros((width,) + view.shape[1:], dtype=view.dtype)
        pad[: len(view)] = view
        t = torch.from_numpy(pad)
        if device is not None:
            t = t.to(device)
        full = torch.empty((world * width,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(full, t, group=group)
        full = full.cpu().numpy()
        parts = [full[r * width : r * width + (b - a)] for r, (a, b) in enumerate(sizes)]
        res = np.concatenate(parts, axis=0)
        if arr.dtype == np.uint32:
            res = res.view(np.uint32)
        elif arr.dtype == np.bool_:
            res = res.astype(bool)
        out[name] = res
    return out


def all_gather_device(local: dict, group=None) -> dict:
    """All-gather per-task device tensors of equal shard size (first axis = task) into
    full-batch device tensors, one ``all_gather_into_tensor`` per field (NCCL over
    NVLink): the collective of the device-resident path, nothing leaves HBM."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = {}
    for name, t in local.items():
        full = torch.empty((world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(full, t.contiguous(), group=group)
        out[name] = full
    return out


def solve_shard(
    splits: np.ndarray,
    discos: np.ndarray,
    inj: np.ndarray,
    n_tasks: int,
    solver: Callable,
    group=None,
    device=None,
) -> dict:
    """Solve this rank's already-sliced shard (``shard_range(n_tasks, rank, world)``) and
    all-gather the results: the full-batch arrays on every rank plus the job-wide
    loadflow total."""
    import torch
    import torch.distributed as dist

    out = solver(splits, discos, inj)
    local = {name: getattr(out, name) for name in RESULT_FIELDS}
    full = all_gather_tasks(local, n_tasks, group=group, device=device)
    lf = torch.tensor([float(out.loadflows)], dtype=torch.float64, device=device)
    dist.all_reduce(lf, group=group)
    full["loadflows"] = int(lf.item())
    return full


def solve_sharded(
    splits: np.ndarray,
    discos: np.ndarray,
    inj: np.ndarray,
    solver: Callable,
    group=None,
    device=None,
) -> dict:
    """Solve this rank's shard of the batch with ``solver`` and all-gather the results.

    ``solver(splits, discos, inj)`` returns an object with the RESULT_FIELDS
    arrays (``engine.BatchOutput``) and a ``loadflows`` count.  Returns the
    full-batch arrays on every rank plus the job-wide loadflow total.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    B = inj.shape[0]
    a, b = shard_range(B, rank, world)
    return solve_shard(splits[a:b], discos[a:b], inj[a:b], B, solver, group=group, device=device)


def global_topk(metric, k: int, offset: int, group=None):
    """The k best topologies of the whole sharded batch (optional): each rank
    takes its shard's k smallest metrics (infeasible tasks, NaN, last), all-gathers the
    (metric, global task index) pairs and merges them -- ascending metric, lower task index
    first on ties, the reference's task order.  ``metric`` is this rank's (B,) tensor (CUDA
    with NCCL, CPU with gloo), ``offset`` the global index of its first task.  Returns the
    (k,) metrics and (k,) int64 task indices on every rank (fewer if the batch is smaller)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = metric.device
    m = torch.nan_to_num(metric.to(torch.float64), nan=float("inf"))
    idx = torch.arange(m.numel(), device=dev, dtype=torch.int64) + int(offset)
    kk = min(int(k), m.numel())
    # (metric, index) lexicographic: a stable sort by metric keeps the lower index first
    order = torch.sort(m, stable=True).indices[:kk]
    loc_m = torch.full((int(k),), float("inf"), dtype=torch.float64, device=dev)
    loc_i = torch.full((int(k),), -1, dtype=torch.int64, device=dev)
    loc_m[:kk] = m[order]
    loc_i[:kk] = idx[order]
    all_m = torch.empty((world * int(k),), dtype=torch.float64, device=dev)
    all_i = torch.empty((world * int(k),), dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(all_m, loc_m, group=group)
    dist.all_gather_into_tensor(all_i, loc_i, group=group)
    valid = all_i >= 0
    all_m, all_i = all_m[valid], all_i[valid]
    # ascending metric, then ascending global index
    o1 = torch.sort(all_i, stable=True).indices
    o2 = torch.sort(all_m[o1], stable=True).indices
    sel = o1[o2][: int(k)]
    return all_m[sel], all_i[sel]


def engine_solver(session) -> Callable:
    """Adapter: the session's GPU engine as a ``solve_sharded`` solver."""

    def run(splits, discos, inj):
        return session.engine.solve(splits, discos, inj)

    return run
