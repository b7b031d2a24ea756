"""World-size-2 gloo test of the topology-sharded path (host logic; CPU only).

Each rank solves its contiguous shard with a CPU stand-in solver built on the
oracle port (the GPU engine cannot run here), then the per-task results are
all-gathered; the gathered batch must equal a single-process solve of the
whole batch, task for task.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden_path

WORLD = 2


class _PortOut:
    """BatchOutput-shaped arrays from the oracle port (CPU stand-in)."""

    def __init__(self, grid, base, cfg, splits, discos, inj):
        from oracle import port
        from paper_2501_17529_b200.parallel import RESULT_FIELDS  # noqa: F401

        res = port.solve_arrays(grid, base, splits, discos, inj, cfg)
        B, kg = len(res), cfg.topk_global
        self.metric = np.array([r.metric if r.feasible else np.nan for r in res])
        self.best = np.array([r.best_injection if r.feasible else -1 for r in res], dtype=np.int64)
        self.feasible = np.array([r.feasible for r in res], dtype=bool)
        self.status = np.array([0 if r.feasible else 1 for r in res], dtype=np.int32)
        self.status_arg = np.zeros(B, dtype=np.int32)
        self.n_islanded = np.array([len(r.islanded_cases) for r in res], dtype=np.int32)
        self.islanded_bits = np.zeros((B, 1), dtype=np.uint32)
        self.n0_count = np.array([len(r.n0_worst or ()) for r in res], dtype=np.int32)
        self.n1_count = np.array([len(r.n1_worst or ()) for r in res], dtype=np.int32)
        self.n0_pos = np.zeros((B, kg), dtype=np.int32)
        self.n0_flow = np.zeros((B, kg))
        self.n0_rel = np.zeros((B, kg))
        self.n1_case = np.zeros((B, kg), dtype=np.int32)
        self.n1_pos = np.zeros((B, kg), dtype=np.int32)
        self.n1_flow = np.zeros((B, kg))
        self.n1_rel = np.zeros((B, kg))
        for b, r in enumerate(res):
            for i, (_bid, f, rel) in enumerate(r.n0_worst or ()):
                self.n0_flow[b, i], self.n0_rel[b, i] = f, rel
            for i, (_cid, _bid, f, rel) in enumerate(r.n1_worst or ()):
                self.n1_flow[b, i], self.n1_rel[b, i] = f, rel
        self.loadflows = sum(inj.shape[1] * (1 + r.n_feasible_cases) for r in res if r.feasible)


def _worker(rank, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(WORLD))
    import torch.distributed as dist

    from paper_2501_17529_b200.io import load_grid
    from paper_2501_17529_b200.parallel import solve_sharded
    from paper_2501_17529_b200.ptdf import prepare_base_ptdf
    from paper_2501_17529_b200.solver import SolveConfig

    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    grid = load_grid(golden_path("grids", "fixture_b.json"))
    base = prepare_base_ptdf(grid)
    cfg = SolveConfig()
    arr = np.load(golden_path("fixture_b.npz"))
    s, d, i = arr["splits"][:21], arr["disconnections"][:21], arr["injection_sets"][:21]
    full = solve_sharded(s, d, i, lambda a, b, c: _PortOut(grid, base, cfg, a, b, c))
    # the device-resident gather of the bench's timed path (gloo here, NCCL on GPUs)
    import torch

    from paper_2501_17529_b200.parallel import all_gather_device

    loc = {"metric": torch.full((3,), float(rank), dtype=torch.float64),
           "n1_case": torch.arange(6, dtype=torch.int32).reshape(3, 2) + 100 * rank}
    g = all_gather_device(loc)
    assert g["metric"].tolist() == [0.0] * 3 + [1.0] * 3
    assert g["n1_case"][3:].tolist() == (torch.arange(6, dtype=torch.int32).reshape(3, 2) + 100).tolist()
    # optional global top-k topologies: shards of a known metric vector
    from paper_2501_17529_b200.parallel import global_topk

    full_metric = torch.tensor([3.0, float("nan"), 1.0, 2.0, 1.0, 0.5, float("nan"), 2.0, 0.5, 4.0], dtype=torch.float64)
    a, b = (0, 5) if rank == 0 else (5, 10)
    tm, ti = global_topk(full_metric[a:b], 4, a)
    assert ti.tolist() == [5, 8, 2, 4], ti.tolist()
    assert tm.tolist() == [0.5, 0.5, 1.0, 1.0]
    if rank == 0:
        np.savez(out_path, **{k: v for k, v in full.items() if k != "loadflows"}, loadflows=full["loadflows"])
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def test_shard_ranges_cover_batch():
    from paper_2501_17529_b200.parallel import shard_range

    for n in (0, 1, 7, 64, 1001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1


def test_sharded_solve_equals_single_process(tmp_path):
    out = tmp_path / "full.npz"
    mp.spawn(_worker, args=(_free_port(), str(out)), nprocs=WORLD, join=True)
    got = np.load(out)
    from paper_2501_17529_b200.io import load_grid
    from paper_2501_17529_b200.ptdf import prepare_base_ptdf
    from paper_2501_17529_b200.solver import SolveConfig

    grid = load_grid(golden_path("grids", "fixture_b.json"))
    arr = np.load(golden_path("fixture_b.npz"))
    ref = _PortOut(grid, prepare_base_ptdf(grid), SolveConfig(), arr["splits"][:21], arr["disconnections"][:21], arr["injection_sets"][:21])
    np.testing.assert_array_equal(got["best"], ref.best)
    np.testing.assert_array_equal(got["feasible"], ref.feasible)
    np.testing.assert_allclose(got["metric"], ref.metric, equal_nan=True)
    np.testing.assert_allclose(got["n1_rel"], ref.n1_rel)
    assert int(got["loadflows"]) == ref.loadflows
