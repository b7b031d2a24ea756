"""Device-side random topology tasks.

The reference draws benchmark batches on the host, one task at a time, with
rejection of N-0-infeasible draws (`batchdc.bench.random_tasks`,
`src/batchdc/bench.py:33-91`; 31.8 ms/task at G1k).  For 10^5..10^6 topologies
per GPU that cannot feed the engine, so here the same distribution is drawn on
the GPU by `bdc_draw_tasks` (csrc/bdc_gen.cu) straight into the session's array
layout, and the engine itself is the acceptance test: the drawn batch is solved
with one all-home candidate, and every task the engine reports as a degenerate
or singular split or an islanding disconnection (the exceptions
`_feasible_at_n0` catches, `bench.py:96-110`) is redrawn with its next draw
number, up to `max_draws` (`_MAX_DRAWS = 500`, `bench.py:30`).

Everything stays in HBM: the returned splits / disconnections / injection rows
are CUDA tensors ready for `Engine.solve_device`.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from .engine import (
    TASK_DEGENERATE_SPLIT,
    TASK_DISCONNECT_ISLAND,
    TASK_SINGULAR_SPLIT,
    EngineUnavailable,
    _err,
)
from .errors import ValidationError

MAX_DRAWS = 500  # bench.py:30
REJECT = (TASK_DEGENERATE_SPLIT, TASK_SINGULAR_SPLIT, TASK_DISCONNECT_ISLAND)


def _vp(t) -> Optional[ctypes.c_void_p]:
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def draw_arrays(engine, seed: int, B: int, T: int, n_splits: int, n_disconnections: int,
                splits, discos, inj, attempt=None, redraw=None, stream_ptr: int = 0) -> None:
    """One `bdc_draw_tasks` call on existing CUDA tensors (no acceptance test)."""
    E = int(splits.shape[2]) if splits.dim() == 3 else 1
    D = int(discos.shape[1]) if discos is not None and discos.dim() == 2 else 0
    rc = engine.lib.bdc_draw_tasks(
        engine.handle, ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF), int(B), int(T), E, D, int(n_splits),
        int(n_disconnections), _vp(attempt), _vp(redraw), _vp(splits), _vp(discos) if D else None,
        _vp(inj), ctypes.c_void_p(stream_ptr) if stream_ptr else None,
    )
    if rc != 0:
        raise EngineUnavailable(f"bdc_draw_tasks failed ({rc}): {_err(engine.lib)}")


def random_tasks_device(session, n_tasks: int, ti_size: int, n_splits: int, seed: int,
                        n_disconnections: int = 0, max_draws: int = MAX_DRAWS, stream=None):
    """N-0-feasible random tasks drawn on the session's GPU.

    Returns ``(splits (B,S,E) u8, disconnections (B,D) i64, injection_sets (B,T,K) u8,
    draws)`` as CUDA tensors, ``draws`` the number of acceptance rounds used.
    Same distribution as `bench.random_tasks` (uniform distinct eligible substations,
    uniform non-empty assignment bits, uniform distinct disconnections, uniform
    injection bits, N-0-infeasible draws rejected)."""
    import torch

    eng = session.engine
    tb = eng.tables
    dev = torch.device("cuda", eng.device)
    S, E, K = tb.S, max(tb.E, 1), tb.K
    B, T, d = int(n_tasks), int(ti_size), int(n_disconnections)
    if d > session.config.max_simultaneous_outages:
        raise ValidationError(
            f"{d} disconnections exceed the cap of {session.config.max_simultaneous_outages}")
    splits = torch.empty((B, S, E), dtype=torch.uint8, device=dev)
    discos = torch.empty((B, d), dtype=torch.int64, device=dev)
    inj = torch.empty((B, T, K), dtype=torch.uint8, device=dev)
    attempt = torch.zeros(B, dtype=torch.int32, device=dev)
    st = stream or torch.cuda.current_stream(dev)
    sp = st.cuda_stream
    draw_arrays(eng, seed, B, T, n_splits, d, splits, discos, inj, attempt=attempt, stream_ptr=sp)
    if B == 0:
        return splits, discos, inj, 0
    # acceptance: the engine's own split chain and outage test, one all-home candidate;
    # later rounds solve only the redrawn tasks (gathered, then mapped back)
    kg = session.config.topk_global
    ncw = max(1, (len(session.grid.contingencies) + 31) // 32)
    rank = max(1, min(n_splits, sum(1 for s in session.grid.substations if len(s.branch_elements) >= 2)) + d)
    reject = torch.tensor(REJECT, dtype=torch.int32, device=dev)

    def status_of(sp_, dc_):
        n = int(sp_.shape[0])
        outs = {name: torch.empty(shape, dtype=dt, device=dev) for name, shape, dt in (
            ("metric", (n,), torch.float64), ("best", (n,), torch.int64), ("feasible", (n,), torch.uint8),
            ("status", (n,), torch.int32), ("status_arg", (n,), torch.int32), ("n_islanded", (n,), torch.int32),
            ("islanded_bits", (n, ncw), torch.int32), ("n0_count", (n,), torch.int32),
            ("n0_pos", (n, kg), torch.int32), ("n0_flow", (n, kg), torch.float64), ("n0_rel", (n, kg), torch.float64),
            ("n1_count", (n,), torch.int32), ("n1_case", (n, kg), torch.int32), ("n1_pos", (n, kg), torch.int32),
            ("n1_flow", (n, kg), torch.float64), ("n1_rel", (n, kg), torch.float64))}
        home = torch.zeros((n, 1, K), dtype=torch.uint8, device=dev)
        eng.solve_device(sp_, dc_, home, outs, sp, rank)
        return outs["status"]

    idx = None  # tasks under test (None: all)
    for draws in range(1, max_draws + 1):
        if idx is None:
            bad = torch.isin(status_of(splits, discos), reject)
        else:
            sub_bad = torch.isin(status_of(splits[idx].contiguous(), discos[idx].contiguous()), reject)
            bad = torch.zeros(B, dtype=torch.bool, device=dev)
            bad[idx[sub_bad]] = True
        nbad = int(bad.sum().item())
        if nbad == 0:
            return splits, discos, inj, draws
        attempt += bad.to(torch.int32)
        draw_arrays(eng, seed, B, T, n_splits, d, splits, discos, None, attempt=attempt,
                    redraw=bad.to(torch.uint8), stream_ptr=sp)
        idx = torch.nonzero(bad).flatten()
    raise RuntimeError("could not draw a feasible task; grid too fragile?")


def to_host(splits, discos, inj):
    """The drawn arrays as numpy (for the host API / the CPU oracle)."""
    return (splits.cpu().numpy().astype(bool), discos.cpu().numpy().astype(np.int64),
            inj.cpu().numpy().astype(bool))
