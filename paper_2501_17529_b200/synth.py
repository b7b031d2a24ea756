"""Synthetic grids and topology-task batches for tests and benchmarks.

Grids follow the recipe of the reference's fixture generator
(`pkg/tools/make_fixtures.py:73-229`), scaled to the BASELINE sizes: a ring
backbone (bridge-free) plus chords up to E = round(1.37 N); hubs with five
branch elements (two ring edges + three chords) as splittable substations;
73 % of hubs carry a reassignable load/generator slot pair; loads on 43 % of
the other nodes, generators on 15 %, rescaled to balance; x ~ U(0.05, 0.45)
with b = 1/x; ratings max(25, 1.25 |f_N0| + 15); N-1 = 90 % of branches as
single cases plus chord pairs as multi cases plus generator losses.

Task batches follow `bench.random_tasks` semantics (`pkg/src/batchdc/bench.py:33-91`):
distinct eligible substations (>= 2 elements), uniform non-all-False bits,
uniform distinct disconnections, uniform candidate bit rows, and rejection of
draws that are infeasible at N-0.  Feasibility is decided exactly as the
reference's refactorisation oracle decides it (graph connectivity of the
materialised topology, `oracle.py:102-103`) plus the degenerate-split rule
(all elements moved, `factors.py:491-495`); it is vectorised over thousands
of tasks with one sparse connected-components call so 10^5-10^6 task batches
can be drawn in seconds.  The RNG stream differs from the reference's
sequential generator; the acceptance rules are the same.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .grid import Grid, static_injection_fold
from .io import grid_from_dict


@dataclass(frozen=True)
class GridSpec:
    name: str
    n_nodes: int
    n_hubs: int
    n_branches: int
    n_multi: int
    n_injloss: int


SPECS = {
    "g14": GridSpec("g14", 14, 2, 20, 1, 1),
    "g118": GridSpec("g118", 118, 6, 162, 3, 3),
    "g300": GridSpec("g300", 300, 15, 411, 8, 5),
    "g1k": GridSpec("g1k", 1000, 50, 1370, 8, 5),
    "g3k": GridSpec("g3k", 3000, 150, 4110, 8, 5),
    "g10k": GridSpec("g10k", 10000, 500, 13700, 8, 5),
}


def _dc_flows(n, f, t, b, p, slack):
    lap = np.zeros((n, n))
    np.add.at(lap, (f, f), b)
    np.add.at(lap, (t, t), b)
    np.add.at(lap, (f, t), -b)
    np.add.at(lap, (t, f), -b)
    keep = np.array([i for i in range(n) if i != slack])
    theta = np.zeros(n)
    theta[keep] = np.linalg.solve(lap[np.ix_(keep, keep)], p[keep])
    return b * (theta[f] - theta[t])


def _connected_without(n, f, t, dead) -> bool:
    alive = np.ones(len(f), dtype=bool)
    alive[list(dead)] = False
    g = sp.coo_matrix((np.ones(alive.sum()), (f[alive], t[alive])), shape=(n, n))
    return connected_components(g, directed=False)[0] == 1


def make_grid_doc(spec: GridSpec | str, seed: int = 0) -> dict:
    """Deterministic synthetic grid document in the native JSON shape."""
    if isinstance(spec, str):
        spec = SPECS[spec]
    rng = np.random.default_rng(seed)
    N, H, E = spec.n_nodes, spec.n_hubs, spec.n_branches
    edges = [(i, (i + 1) % N) for i in range(N)]
    gap = N // H
    hubs = [gap // 2 + 1 + gap * i for i in range(H)]
    assert hubs[-1] < N and 0 not in hubs
    hubset = set(hubs)
    used = {frozenset(e) for e in edges}
    pool = np.array([i for i in range(N) if i not in hubset and i != 0])

    def chord(a):
        while True:
            b = int(pool[rng.integers(0, len(pool))])
            if b != a and frozenset((a, b)) not in used:
                used.add(frozenset((a, b)))
                edges.append((a, b))
                return

    for h in hubs:
        for _ in range(3):
            chord(h)
    while len(edges) < E:
        chord(int(pool[rng.integers(0, len(pool))]))
    f = np.array([e[0] for e in edges])
    t = np.array([e[1] for e in edges])
    x = np.round(rng.uniform(0.05, 0.45, size=E), 6)
    b = 1.0 / x

    n_inj_hubs = max(1, int(round(0.73 * H)))
    inj_hubs = hubs[:n_inj_hubs]
    load_nodes = sorted(int(i) for i in rng.choice(pool, size=max(1, int(0.43 * len(pool))), replace=False))
    rest = np.array([i for i in pool if i not in set(load_nodes)])
    gen_nodes = sorted(int(i) for i in rng.choice(rest, size=max(1, int(0.15 * len(pool))), replace=False))
    loads = {n: -float(np.round(rng.uniform(10, 110), 3)) for n in load_nodes}
    for h in inj_hubs:
        loads[h] = -float(np.round(rng.uniform(20, 80), 3))
    gens = {n: float(np.round(rng.uniform(30, 150), 3)) for n in gen_nodes}
    for h in inj_hubs:
        gens[h] = float(np.round(rng.uniform(40, 130), 3))
    scale = -sum(loads.values()) / sum(gens.values())
    gens = {n: float(np.round(p * scale, 3)) for n, p in gens.items()}
    p = np.zeros(N)
    for n_, v in loads.items():
        p[n_] += v
    for n_, v in gens.items():
        p[n_] += v
    fl = _dc_flows(N, f, t, b, p, 0)
    ratings = np.round(np.maximum(25.0, 1.25 * np.abs(fl) + 15.0), 1)

    node_ids = [f"N{i}" for i in range(N)]
    br_ids = [f"L{k}_{f[k]}_{t[k]}" for k in range(E)]
    inj_docs = []
    at = {}
    for n_ in range(N):
        if n_ in loads:
            inj_docs.append({"id": f"load{n_}", "node": node_ids[n_], "p_mw": loads[n_]})
            at.setdefault(n_, []).append(f"load{n_}")
    gen_order = sorted(gens)
    for n_ in gen_order:
        inj_docs.append({"id": f"gen{n_}", "node": node_ids[n_], "p_mw": gens[n_]})
        at.setdefault(n_, []).append(f"gen{n_}")
    subs = []
    for h in hubs:
        inc = [k for k in range(E) if f[k] == h or t[k] == h]
        assert len(inc) == 5
        subs.append(
            {
                "node": node_ids[h],
                "branch_elements": [br_ids[k] for k in inc],
                "injection_elements": at[h] if h in inj_hubs else [],
            }
        )
    cases = []
    n_single = int(round(0.9 * E))
    for k in sorted(int(k) for k in rng.permutation(E)[:n_single]):
        cases.append({"id": f"n1_{br_ids[k]}", "kind": "single_branch", "branches": [br_ids[k]]})
    chords = np.arange(N, E)
    m = 0
    tries = 0
    while m < spec.n_multi and tries < 1000:
        tries += 1
        pick = sorted(int(c) for c in rng.choice(chords, size=2, replace=False))
        if _connected_without(N, f, t, pick):
            cases.append(
                {"id": f"multi{m}", "kind": "multi_branch", "branches": [br_ids[k] for k in pick]}
            )
            m += 1
    targets = [f"gen{h}" for h in inj_hubs[:2]]
    for n_ in sorted(gens, key=lambda n_: -gens[n_]):
        if len(targets) >= spec.n_injloss:
            break
        if f"gen{n_}" not in targets:
            targets.append(f"gen{n_}")
    for tid in targets[: spec.n_injloss]:
        cases.append({"id": f"loss_{tid}", "kind": "injection", "injection": tid})
    return {
        "nodes": [{"id": i} for i in node_ids],
        "branches": [
            {
                "id": br_ids[k],
                "from": node_ids[f[k]],
                "to": node_ids[t[k]],
                "susceptance": float(b[k]),
                "rating": float(ratings[k]),
                "monitored": True,
            }
            for k in range(E)
        ],
        "injections": inj_docs,
        "slack": node_ids[0],
        "substations": subs,
        "contingencies": cases,
    }


def make_grid(spec: GridSpec | str, seed: int = 0) -> Grid:
    return grid_from_dict(make_grid_doc(spec, seed))


# ----------------------------------------------------------------------------- tasks
def folded_branches(grid: Grid) -> np.ndarray:
    """Branches with an endpoint folded into the static column of the base PTDF
    (`reduce_static`, factors.py:219-275): they cannot be disconnected."""
    static = np.array(sorted(static_injection_fold(grid).static_nodes), dtype=np.int64)
    if not len(static):
        return np.zeros(grid.n_branches, dtype=bool)
    return np.isin(grid.from_nodes, static) | np.isin(grid.to_nodes, static)


def _feasible_mask(grid: Grid, splits: np.ndarray, discos: np.ndarray) -> np.ndarray:
    """N-0 feasibility of each task: no degenerate split and a connected topology."""
    B = splits.shape[0]
    S = len(grid.substations)
    N, Eb = grid.n_nodes, grid.n_branches
    counts = np.array([len(s.branch_elements) for s in grid.substations])
    ok = np.ones(B, dtype=bool)
    if S:
        width = splits.shape[2]
        valid = np.arange(width)[None, :] < counts[:, None]  # (S, E)
        moved = splits & valid[None]
        all_moved = (moved.sum(axis=2) == counts[None, :]) & (counts[None, :] > 0)
        ok &= ~all_moved.any(axis=1)
    f = np.broadcast_to(grid.from_nodes, (B, Eb)).copy()
    t = np.broadcast_to(grid.to_nodes, (B, Eb)).copy()
    nn = N + S  # split node of substation si is N + si
    if S:
        width = splits.shape[2]
        elem = np.full((S, width), -1, dtype=np.int64)
        for si, s in enumerate(grid.substations):
            elem[si, : len(s.branch_elements)] = s.branch_elements
        bi, si_, ei = np.nonzero(splits & (elem[None] >= 0))
        k = elem[si_, ei]
        node = np.array([s.node for s in grid.substations])[si_]
        at_from = f[bi, k] == node
        f[bi[at_from], k[at_from]] = N + si_[at_from]
        t[bi[~at_from], k[~at_from]] = N + si_[~at_from]
    alive = np.ones((B, Eb), dtype=bool)
    if discos is not None and discos.size:
        bi, di = np.nonzero(discos >= 0)
        alive[bi, discos[bi, di]] = False
    off = (np.arange(B) * nn)[:, None]
    ff, tt = (f + off)[alive], (t + off)[alive]
    # unused split nodes are isolated: give each a self-edge to its substation node
    if S:
        used = splits.any(axis=2)
        bi, si_ = np.nonzero(~used)
        node = np.array([s.node for s in grid.substations])[si_]
        ff = np.concatenate([ff, bi * nn + N + si_])
        tt = np.concatenate([tt, bi * nn + node])
    g = sp.coo_matrix((np.ones(len(ff), dtype=np.int8), (ff, tt)), shape=(B * nn, B * nn))
    _n, labels = connected_components(g, directed=False)
    lab = labels.reshape(B, nn)
    comps = np.array([len(np.unique(lab[b])) for b in range(B)])
    return ok & (comps == 1)


def random_task_arrays(
    grid: Grid,
    n_tasks: int,
    ti_size: int,
    n_splits: int,
    seed: int,
    n_disconnections: int = 0,
    chunk: int = 4096,
    reject_infeasible: bool = True,
):
    """Feasible random tasks as session arrays (splits (B,S,E), discos (B,D), inj (B,T,K))."""
    rng = np.random.default_rng(seed)
    S = len(grid.substations)
    width = max((len(s.branch_elements) for s in grid.substations), default=0)
    K = len(grid.injection_slots)
    counts = np.array([len(s.branch_elements) for s in grid.substations], dtype=np.int64)
    eligible = np.flatnonzero(counts >= 2)
    k = min(n_splits, len(eligible))
    out_s, out_d, out_i = [], [], []
    have = 0
    while have < n_tasks:
        n = min(chunk, max(64, int((n_tasks - have) * 1.2)))
        splits = np.zeros((n, S, width), dtype=bool)
        if k:
            pick = np.argsort(rng.random((n, len(eligible))), axis=1)[:, :k]
            subs = eligible[pick]  # (n, k)
            bits = rng.integers(0, 2, size=(n, k, width)).astype(bool)
            cnt = counts[subs]
            valid = np.arange(width)[None, None, :] < cnt[:, :, None]
            bits &= valid
            bad = ~bits.any(axis=2)
            while bad.any():
                redraw = rng.integers(0, 2, size=(int(bad.sum()), width)).astype(bool)
                bits[bad] = redraw & valid[bad]
                bad = ~bits.any(axis=2)
            rows = np.repeat(np.arange(n), k)
            splits[rows, subs.ravel()] = bits.reshape(n * k, width)
        if n_disconnections:
            d = rng.integers(0, grid.n_branches, size=(n, n_disconnections))
            srt = np.sort(d, axis=1)
            dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
            while dup.any():
                d[dup] = rng.integers(0, grid.n_branches, size=(int(dup.sum()), n_disconnections))
                srt = np.sort(d, axis=1)
                dup = (srt[:, 1:] == srt[:, :-1]).any(axis=1)
            discos = d.astype(np.int64)
        else:
            discos = np.zeros((n, 0), dtype=np.int64)
        inj = rng.integers(0, 2, size=(n, ti_size, K)).astype(bool)
        if reject_infeasible:
            keep = _feasible_mask(grid, splits, discos)
            if n_disconnections:
                # a branch with a folded endpoint cannot be disconnected (ValidationError in
                # the reference, which random_tasks rejects, bench.py:108-109)
                keep &= ~folded_branches(grid)[discos].any(axis=1)
            splits, discos, inj = splits[keep], discos[keep], inj[keep]
        take = min(len(splits), n_tasks - have)
        out_s.append(splits[:take])
        out_d.append(discos[:take])
        out_i.append(inj[:take])
        have += take
    return np.concatenate(out_s), np.concatenate(out_d), np.concatenate(out_i)
