"""TEST INFRASTRUCTURE: numpy restatement of the reference engine's solve path.

This is the CPU oracle (and the CPU baseline timed by ``bench.py``), not the
product.  It follows the reference implementation operation for operation in
FP64 so that, on the same grid and tasks, it reproduces the reference's
results bit for bit (checked against golden vectors in
``tests/test_oracle_golden.py``).  Structure:

* ``Canon`` / ``canonical``         <- solver.py:148-197 (canonicalize_task)
* ``_State`` + ``_split``           <- factors.py:428-585 (compute_bsdf, apply_bsdf)
* ``_modf``                         <- factors.py:373-425 (compute_modf, apply_modf_to_ptdf)
* ``_lodf_outage``                  <- factors.py:333-370 (sequential outages)
* ``_branch``                       <- solver.py:381-516 (_branch_stage)
* ``_n0_block``                     <- solver.py:526-595 (static flows, slot binding, N-0)
* ``_case_flows``                   <- solver.py:598-622
* ``_inject_metric_first`` / ``_inject_symmetric``  <- solver.py:766-851
* ``_report_winner`` / ``_report_pools``            <- solver.py:652-763, 287-318
* ``solve``                         <- solver.py:887-1003 (one task / a batch)

Inputs are the product's host grid model and base PTDF
(``paper_2501_17529_b200.grid`` / ``.ptdf``), which mirror the reference's
data contract; the arithmetic below is independent of the GPU engine.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from paper_2501_17529_b200.errors import ValidationError
from paper_2501_17529_b200.grid import INJECTION, MULTI_BRANCH, SINGLE_BRANCH, Grid

TOL = 1e-8  # ISLANDING_TOL == SPLIT_TOL, factors.py:48-49


class _Island(Exception):
    pass


class _SplitFail(Exception):
    pass


# --------------------------------------------------------------------------- tasks
@dataclass(frozen=True)
class Canon:
    """A canonical task: sorted non-trivial splits, disconnections, bit rows."""

    splits: tuple  # ((substation, bits tuple), ...)
    discos: tuple
    rows: np.ndarray  # (T, K) bool


def canonical(grid: Grid, splits, discos, rows) -> Canon:
    """solver.py:148-197 -- validation messages match the reference."""
    seen = set()
    keep = []
    for si, bits in splits:
        if not 0 <= si < len(grid.substations):
            raise ValidationError(f"substation index {si} out of range")
        if si in seen:
            raise ValidationError(f"substation {si} split twice in one task")
        seen.add(si)
        n_el = len(grid.substations[si].branch_elements)
        if len(bits) != n_el:
            raise ValidationError(
                f"substation {si}: assignment has {len(bits)} bits, expected {n_el}"
            )
        if any(bits):
            keep.append((int(si), tuple(bool(b) for b in bits)))
    keep.sort()
    discos = tuple(int(k) for k in discos)
    if len(set(discos)) != len(discos):
        raise ValidationError("duplicate branch in disconnections")
    for k in discos:
        if not 0 <= k < grid.n_branches:
            raise ValidationError(f"disconnection branch {k} out of range")
    K = len(grid.injection_slots)
    if len(rows) == 0:
        raise ValidationError("task needs at least one injection set")
    out = []
    for r in rows:
        if len(r) == 0 and K > 0:
            out.append([False] * K)
            continue
        if len(r) != K:
            raise ValidationError(f"injection set has {len(r)} bits, expected {K}")
        out.append([bool(b) for b in r])
    return Canon(tuple(keep), discos, np.array(out, dtype=bool).reshape(len(out), K))


# --------------------------------------------------------------------------- state
@dataclass
class _State:
    """Materialised PTDF plus the bookkeeping of factors.py:55-109."""

    values: np.ndarray
    from_cols: np.ndarray
    to_cols: np.ndarray
    node_cols: np.ndarray
    static_col: Optional[int]
    branch_rows: np.ndarray
    split_col: dict = field(default_factory=dict)  # substation node -> column

    @classmethod
    def of(cls, base) -> "_State":
        return cls(
            base.values,
            base.from_cols.copy(),
            base.to_cols.copy(),
            base.node_cols.copy(),
            base.static_col,
            base.branch_rows,
        )


def _split(st: _State, grid: Grid, si: int, bits: tuple) -> _State:
    """One busbar split, factors.py:428-585 (coupler row, numerator, rank-one apply)."""
    sub = grid.substations[si]
    node = sub.node
    a = int(st.node_cols[node])
    C = st.values.shape[1]
    moved = [k for k, b in zip(sub.branch_elements, bits) if b]
    stay = [k for k, b in zip(sub.branch_elements, bits) if not b]

    def side(k):
        r = int(st.branch_rows[k])
        if int(st.from_cols[r]) == a:
            return r, 1.0, int(st.to_cols[r])
        if int(st.to_cols[r]) == a:
            return r, -1.0, int(st.from_cols[r])
        raise ValidationError(f"branch {k} is no longer attached to substation node {node}")

    stay_b = sum(grid.branches[k].susceptance for k in stay)
    if not stay_b > 0.0:
        raise _SplitFail(f"split of node {node} leaves busbar A without any branch")
    vals = st.values
    coupler = np.zeros(C + 1)
    for k in moved:
        r, sg, _ = side(k)
        coupler[:C] += sg * vals[r, :]
    coupler[C] = coupler[a] - 1.0
    num = np.zeros(vals.shape[0])
    den = coupler[a]
    for k in stay:
        r, sg, far = side(k)
        w = grid.branches[k].susceptance / stay_b
        num += w * (vals[:, far] - vals[:, a])
        num[r] += sg * w
        den -= w * coupler[far]
    if abs(den) < TOL:
        raise _SplitFail(
            f"split of node {node} with assignment {list(bits)} disconnects the grid"
        )
    bsdf = num / den
    new = np.hstack([vals, vals[:, a : a + 1]]) + np.outer(bsdf, coupler)
    fc, tc = st.from_cols.copy(), st.to_cols.copy()
    for k in moved:
        r = int(st.branch_rows[k])
        if int(fc[r]) == a:
            fc[r] = C
        elif int(tc[r]) == a:
            tc[r] = C
    nc = st.node_cols
    split_col = dict(st.split_col)
    split_col[node] = C
    static = st.static_col
    if static is not None:
        # static column stays last (factors.py:552-576)
        order = list(range(C + 1))
        order[static], order[-1] = order[-1], order[static]
        new = new[:, order]
        remap = np.empty(C + 1, dtype=np.int64)
        remap[order] = np.arange(C + 1)
        nc = np.where(nc >= 0, remap[np.maximum(nc, 0)], -1)
        fc = np.where(fc >= 0, remap[np.maximum(fc, 0)], -1)
        tc = np.where(tc >= 0, remap[np.maximum(tc, 0)], -1)
        split_col = {n: int(remap[c]) for n, c in split_col.items()}
        static = C
    return _State(new, fc, tc, nc, static, st.branch_rows, split_col)


def _modf(st: _State, branches: Sequence[int]):
    """compute_modf, factors.py:373-409 -> (rows, values) or raises _Island."""
    branches = tuple(int(k) for k in branches)
    rows = np.array([int(st.branch_rows[k]) for k in branches], dtype=np.int64)
    f, t = st.from_cols[rows], st.to_cols[rows]
    v = st.values
    inner = np.eye(len(rows)) - (v[np.ix_(rows, f)] - v[np.ix_(rows, t)])
    sv = np.linalg.svd(inner, compute_uv=False)
    if sv[-1] < TOL * max(1.0, float(sv[0])):
        raise _Island(f"simultaneous outage of branches {list(branches)} islands the grid")
    rhs = v[:, f] - v[:, t]
    vals = np.linalg.solve(inner.T, rhs.T).T
    for i, r in enumerate(rows):
        vals[r, :] = 0.0
        vals[r, i] = -1.0
    return rows, vals


def _lodf_outage(st: _State, k: int) -> _State:
    """lodf_column + apply_outage_to_ptdf, factors.py:333-370."""
    r = int(st.branch_rows[k])
    f, t = int(st.from_cols[r]), int(st.to_cols[r])
    v = st.values
    den = 1.0 - (v[r, f] - v[r, t])
    if abs(den) < TOL:
        raise _Island(f"outage of branch {k} islands the grid")
    col = (v[:, f] - v[:, t]) / den
    col[r] = -1.0
    nv = v + np.outer(col, v[r, :])
    nv[r, :] = 0.0
    return _State(nv, st.from_cols, st.to_cols, st.node_cols, st.static_col, st.branch_rows, st.split_col)


# --------------------------------------------------------------------------- branch stage
@dataclass
class _Case:
    order: int
    cid: str
    kind: str
    feasible: bool = True
    rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    lodf: Optional[np.ndarray] = None
    modf: Optional[np.ndarray] = None
    slot: Optional[int] = None
    col: int = -1
    sp: float = 0.0
    mask: Optional[np.ndarray] = None


@dataclass
class _Ctx:
    st: _State
    feasible: bool
    reason: Optional[str] = None
    islanded: tuple = ()
    static_flows: Optional[np.ndarray] = None
    cases: list = field(default_factory=list)
    mon_rows: Optional[np.ndarray] = None
    ratings: Optional[np.ndarray] = None
    mon_br: Optional[np.ndarray] = None
    identity: bool = False
    base_mask: Optional[np.ndarray] = None
    col_a: Optional[np.ndarray] = None
    col_b: Optional[np.ndarray] = None
    sps: Optional[np.ndarray] = None
    s_orders: Optional[np.ndarray] = None
    s_rows: Optional[np.ndarray] = None
    s_lodf: Optional[np.ndarray] = None
    s_scale: Optional[np.ndarray] = None


def _branch(grid: Grid, st: _State, discos: tuple, cfg) -> _Ctx:
    """solver.py:381-516."""
    if discos:
        if len(discos) > cfg.max_simultaneous_outages:
            raise ValidationError(
                f"{len(discos)} disconnections exceed the cap of {cfg.max_simultaneous_outages}"
            )
        try:
            if cfg.multi_outage_method == "sequential":
                for k in discos:
                    st = _lodf_outage(st, k)
            else:
                rows, vals = _modf(st, discos)
                nv = st.values + vals @ st.values[rows, :]
                nv[rows, :] = 0.0
                st = _State(nv, st.from_cols, st.to_cols, st.node_cols, st.static_col,
                            st.branch_rows, st.split_col)
        except _Island as exc:
            return _Ctx(st=st, feasible=False, reason=f"disconnections island the grid: {exc}")

    mon = np.array(grid.monitored, dtype=np.int64)
    mon_rows = st.branch_rows[mon]
    R = st.values.shape[0]
    ctx = _Ctx(
        st=st,
        feasible=True,
        mon_rows=mon_rows,
        ratings=grid.ratings[mon],
        mon_br=mon,
        identity=len(mon_rows) == R and bool(np.array_equal(mon_rows, np.arange(R))),
    )
    pos = np.full(grid.n_branches, -1, dtype=np.int64)
    pos[mon] = np.arange(len(mon))
    ctx.base_mask = np.ones(len(mon), dtype=bool)
    for k in discos:
        if pos[k] >= 0:
            ctx.base_mask[pos[k]] = False

    def mask_of(brs):
        m = ctx.base_mask.copy()
        for k in brs:
            if pos[k] >= 0:
                m[pos[k]] = False
        return m

    islanded = []
    singles = []
    slot_of = {}
    for s, (_si, j) in enumerate(grid.injection_slots):
        slot_of.setdefault(j, s)
    for order, case in enumerate(grid.contingencies):
        ce = _Case(order, case.id, case.kind)
        if case.kind == SINGLE_BRANCH:
            ce.rows = np.array([int(st.branch_rows[case.branches[0]])], dtype=np.int64)
            singles.append(ce)
            ctx.cases.append(ce)
            continue
        if case.kind == MULTI_BRANCH:
            try:
                ce.rows, ce.modf = _modf(st, case.branches)
            except _Island:
                ce.feasible = False
        else:
            j = case.injection
            ce.sp = grid.injections[j].setpoint
            s = slot_of.get(j)
            if s is not None:
                ce.slot = s
            else:
                ce.col = int(st.node_cols[grid.injections[j].node])
        if ce.feasible:
            ce.mask = mask_of(case.branches)
        else:
            islanded.append(case.id)
        ctx.cases.append(ce)

    if singles:
        rows = np.array([ce.rows[0] for ce in singles], dtype=np.int64)
        v = st.values
        diff = v[:, st.from_cols[rows]] - v[:, st.to_cols[rows]]
        den = 1.0 - diff[rows, np.arange(len(rows))]
        ok = np.abs(den) >= TOL
        lodf = diff / np.where(ok, den, 1.0)[None, :]
        lodf[rows, np.arange(len(rows))] = -1.0
        keep_o, keep_c = [], []
        for j, ce in enumerate(singles):
            if not ok[j]:
                ce.feasible = False
                islanded.append(ce.cid)
                continue
            ce.lodf = lodf[:, j]
            ce.mask = mask_of(grid.contingencies[ce.order].branches)
            keep_o.append(ce.order)
            keep_c.append(j)
        if keep_c:
            ctx.s_orders = np.array(keep_o, dtype=np.int64)
            ctx.s_rows = rows[keep_c]
            ctx.s_lodf = lodf[:, keep_c]
        order_of = {ce.cid: ce.order for ce in ctx.cases}
        islanded.sort(key=lambda cid: order_of[cid])

    if islanded and cfg.islanding_policy == "error":
        return _Ctx(
            st=st,
            feasible=False,
            reason=f"islanding under contingencies {islanded}",
            islanded=tuple(islanded),
        )
    ctx.islanded = tuple(islanded)

    # static flows (solver.py:526-552)
    v = st.values
    flows = v[:, st.static_col].copy() if st.static_col is not None else np.zeros(R)
    slotted = {j for _s, j in grid.injection_slots}
    power: dict = {}
    for j, inj in enumerate(grid.injections):
        if j not in slotted and inj.setpoint != 0.0:
            power[inj.node] = power.get(inj.node, 0.0) + inj.setpoint
    for node, mw in sorted(power.items()):
        col = int(st.node_cols[node])
        if col < 0:
            continue
        flows += v[:, col] * mw
    ctx.static_flows = flows

    # slot binding (solver.py:555-572)
    K = len(grid.injection_slots)
    ctx.col_a = np.zeros(K, dtype=np.int64)
    ctx.col_b = np.zeros(K, dtype=np.int64)
    ctx.sps = np.zeros(K)
    for s, (si, j) in enumerate(grid.injection_slots):
        a = int(st.node_cols[grid.injections[j].node])
        ctx.col_a[s] = a
        ctx.col_b[s] = st.split_col.get(grid.substations[si].node, a)
        ctx.sps[s] = grid.injections[j].setpoint
    return ctx


# --------------------------------------------------------------------------- injection stage
def _n0_block(ctx: _Ctx, bits: np.ndarray) -> np.ndarray:
    """solver.py:575-595."""
    T = bits.shape[0]
    v = ctx.st.values
    if bits.shape[1] == 0:
        return np.repeat(ctx.static_flows[:, None], T, axis=1)
    cols = np.where(bits, ctx.col_b[None, :], ctx.col_a[None, :])
    used = np.unique(cols)
    where = {int(c): i for i, c in enumerate(used)}
    w = np.zeros((len(used), T))
    for s in range(bits.shape[1]):
        mw = ctx.sps[s]
        if mw == 0.0:
            continue
        for t in range(T):
            w[where[int(cols[t, s])], t] += mw
    return ctx.static_flows[:, None] + v[:, used] @ w


def _case_flows(ctx: _Ctx, ce: _Case, n0: np.ndarray, ccols, sel) -> np.ndarray:
    """solver.py:598-622."""
    if ce.kind == SINGLE_BRANCH:
        return n0 + ce.lodf[:, None] * n0[ce.rows[0], :]
    if ce.kind == MULTI_BRANCH:
        out = n0.copy()
        for j in range(len(ce.rows)):
            out += ce.modf[:, j : j + 1] * n0[ce.rows[j], :]
        return out
    v = ctx.st.values
    if ce.slot is not None:
        return n0 - v[:, ccols[sel]] * ce.sp
    return n0 - v[:, ce.col : ce.col + 1] * ce.sp


def _rel_max(ctx: _Ctx, flows: np.ndarray) -> np.ndarray:
    if len(ctx.mon_rows) == 0:
        return np.zeros(flows.shape[1])
    sub = flows if ctx.identity else flows[ctx.mon_rows, :]
    return (np.abs(sub) / ctx.ratings[:, None]).max(axis=0)


def _scale(ctx: _Ctx) -> np.ndarray:
    if ctx.s_scale is None:
        sub = ctx.s_lodf if ctx.identity else ctx.s_lodf[ctx.mon_rows, :]
        ctx.s_scale = (np.abs(sub) / ctx.ratings[:, None]).max(axis=0)
    return ctx.s_scale


def _inj_cols(ctx: _Ctx, bits: np.ndarray) -> dict:
    return {
        ce.order: np.where(bits[:, ce.slot], ctx.col_b[ce.slot], ctx.col_a[ce.slot])
        for ce in ctx.cases
        if ce.kind == INJECTION and ce.slot is not None
    }


def _top(flows, ratings, mask, k):
    """solver.py:287-299: stable top-k by |flow|/rating -> [(pos, rel, flow)]."""
    idx = np.flatnonzero(mask) if mask is not None else np.arange(len(flows))
    if len(idx) == 0:
        return []
    rel = np.abs(flows[idx]) / ratings[idx]
    order = np.argsort(-rel, kind="stable")[:k]
    return [(int(idx[o]), float(rel[o]), float(flows[idx[o]])) for o in order]


def _merge(entries, case_ids, branch_ids, k):
    """solver.py:302-318."""
    if not entries:
        return ()
    rel = np.array([e[2] for e in entries])
    cs = np.array([e[0] for e in entries])
    ps = np.array([e[1] for e in entries])
    order = np.lexsort((ps, cs, -rel))[:k]
    return tuple(
        (case_ids[entries[o][0]], branch_ids[entries[o][1]], entries[o][3], entries[o][2])
        for o in order
    )


def _report_winner(grid, ctx, cfg, n0_block, ccols, best):
    """solver.py:652-713 (bound-stopped scan of single cases)."""
    sel = slice(best, best + 1)
    n0 = n0_block[:, sel]
    case_ids = [ce.cid for ce in ctx.cases]
    entries, pool = [], []
    for ce in ctx.cases:
        if not ce.feasible or ce.kind == SINGLE_BRANCH:
            continue
        fl = _case_flows(ctx, ce, n0, ccols.get(ce.order), sel)
        for p, r, f in _top(fl[ctx.mon_rows, 0], ctx.ratings, ce.mask, cfg.topk_per_case):
            entries.append((ce.order, p, r, f))
            pool.append(r)
    if ctx.s_lodf is not None:
        n0w = n0[:, 0]
        m0b = float(_rel_max(ctx, n0)[0])
        rv = n0_block[ctx.s_rows, best]
        bound = m0b + _scale(ctx) * np.abs(rv)
        kg = cfg.topk_global
        for c in np.argsort(-bound):
            if len(pool) >= kg:
                tk = np.partition(np.array(pool), len(pool) - kg)[len(pool) - kg]
                if bound[c] < tk:
                    break
            fl = n0w + ctx.s_lodf[:, c] * rv[c]
            vec = fl if ctx.identity else fl[ctx.mon_rows]
            ce = ctx.cases[int(ctx.s_orders[c])]
            for p, r, f in _top(vec, ctx.ratings, ce.mask, cfg.topk_per_case):
                entries.append((ce.order, p, r, f))
                pool.append(r)
    bids = [grid.branches[int(k)].id for k in ctx.mon_br]
    n1 = _merge(entries, case_ids, bids, cfg.topk_global)
    n0e = tuple(
        (bids[p], f, r)
        for p, r, f in _top(n0[ctx.mon_rows, 0], ctx.ratings, ctx.base_mask, cfg.topk_global)
    )
    return n0e, n1


def _inject_metric_first(grid, ctx, rows, cfg):
    """solver.py:798-825."""
    n0 = _n0_block(ctx, rows)
    ccols = _inj_cols(ctx, rows)
    penalty = cfg.islanding_penalty if ctx.islanded else None
    m0 = _rel_max(ctx, n0)
    metrics = m0.copy()
    if penalty is not None:
        np.maximum(metrics, penalty, out=metrics)
    for ce in ctx.cases:
        if not ce.feasible or ce.kind == SINGLE_BRANCH:
            continue
        fl = _case_flows(ctx, ce, n0, ccols.get(ce.order), slice(None))
        np.maximum(metrics, _rel_max(ctx, fl), out=metrics)
    if ctx.s_lodf is not None:
        rv = n0[ctx.s_rows, :]
        bound = m0[None, :] + _scale(ctx)[:, None] * np.abs(rv)
        for c in np.argsort(-bound.max(axis=1)):
            if np.all(bound[c] <= metrics):
                continue
            fl = n0 + ctx.s_lodf[:, c : c + 1] * rv[c : c + 1, :]
            np.maximum(metrics, _rel_max(ctx, fl), out=metrics)
    best = int(np.argmin(metrics))
    return float(metrics[best]), best, _report_winner(grid, ctx, cfg, n0, ccols, best)


def _inject_symmetric(grid, ctx, rows, cfg):
    """solver.py:826-842 with the pooled selection of :716-763 (brute force, no screen)."""
    n0 = _n0_block(ctx, rows)
    ccols = _inj_cols(ctx, rows)
    metrics = _rel_max(ctx, n0)
    pools = []
    for ce in ctx.cases:
        if not ce.feasible:
            continue
        fl = _case_flows(ctx, ce, n0, ccols.get(ce.order), slice(None))
        np.maximum(metrics, _rel_max(ctx, fl), out=metrics)
        idx = np.flatnonzero(ce.mask)
        if len(idx) == 0:
            pools.append((ce.order, None))
            continue
        sub = fl[ctx.mon_rows[idx], :]
        rel = np.abs(sub) / ctx.ratings[idx][:, None]
        order = np.argsort(-rel, axis=0, kind="stable")[: cfg.topk_per_case]
        pools.append(
            (ce.order, (idx[order], np.take_along_axis(rel, order, 0), np.take_along_axis(sub, order, 0)))
        )
    if ctx.islanded:
        np.maximum(metrics, cfg.islanding_penalty, out=metrics)
    best = int(np.argmin(metrics))
    bids = [grid.branches[int(k)].id for k in ctx.mon_br]
    case_ids = [ce.cid for ce in ctx.cases]
    entries = []
    for o, pl in pools:
        if pl is None:
            continue
        p, r, f = pl
        for i in range(p.shape[0]):
            entries.append((o, int(p[i, best]), float(r[i, best]), float(f[i, best])))
    n1 = _merge(entries, case_ids, bids, cfg.topk_global)
    n0v = n0[ctx.mon_rows, best]
    n0e = tuple(
        (bids[p], f, r) for p, r, f in _top(n0v, ctx.ratings, ctx.base_mask, cfg.topk_global)
    )
    return float(metrics[best]), best, (n0e, n1)


# --------------------------------------------------------------------------- driver
@dataclass
class PortResult:
    """Same content as the reference's SolveResult (solver.py:94-120)."""

    metric: Optional[float]
    best_injection: Optional[int]
    n0_worst: Optional[tuple]
    n1_worst: Optional[tuple]
    feasible: bool
    reason: Optional[str] = None
    islanded_cases: tuple = ()
    n_feasible_cases: int = 0

    def to_dict(self) -> dict:
        """The result document of io.py:238-259."""
        doc = {"metric": self.metric, "best_injection": self.best_injection, "feasible": self.feasible}
        if self.n0_worst is not None:
            doc["n0_worst"] = [{"branch": b, "flow_mw": f, "rel_load": r} for b, f, r in self.n0_worst]
            doc["n1_worst"] = [
                {"case": c, "branch": b, "flow_mw": f, "rel_load": r} for c, b, f, r in self.n1_worst
            ]
        diag = {}
        if self.reason:
            diag["reason"] = self.reason
        if self.islanded_cases:
            diag["islanded_cases"] = list(self.islanded_cases)
        if diag:
            doc["diagnostics"] = diag
        return doc


def solve_one(grid: Grid, base, canon: Canon, cfg) -> PortResult:
    """solver.py:863-900."""
    st = _State.of(base)
    try:
        for si, bits in canon.splits:
            st = _split(st, grid, si, bits)
    except _SplitFail as exc:
        return PortResult(None, None, None, None, False, str(exc))
    ctx = _branch(grid, st, canon.discos, cfg)
    if not ctx.feasible:
        return PortResult(None, None, None, None, False, ctx.reason, ctx.islanded)
    if cfg.mode == "symmetric":
        metric, best, (n0e, n1e) = _inject_symmetric(grid, ctx, canon.rows, cfg)
    else:
        metric, best, (n0e, n1e) = _inject_metric_first(grid, ctx, canon.rows, cfg)
    nf = sum(1 for ce in ctx.cases if ce.feasible)
    return PortResult(metric, best, n0e, n1e, True, None, tuple(sorted(ctx.islanded)), nf)


def case_flows(grid: Grid, base, canon: Canon, cfg):
    """candidate_case_flows (solver.py:919-958): n0 (R,T) and per-case (R,T) or None."""
    st = _State.of(base)
    try:
        for si, bits in canon.splits:
            st = _split(st, grid, si, bits)
    except _SplitFail as exc:
        return dict(feasible=False, reason=str(exc))
    ctx = _branch(grid, st, canon.discos, cfg)
    if not ctx.feasible:
        return dict(feasible=False, reason=ctx.reason, islanded=ctx.islanded)
    n0 = _n0_block(ctx, canon.rows)
    ccols = _inj_cols(ctx, canon.rows)
    n1 = [
        _case_flows(ctx, ce, n0, ccols.get(ce.order), slice(None)) if ce.feasible else None
        for ce in ctx.cases
    ]
    return dict(feasible=True, n0=n0, n1=n1, islanded=ctx.islanded)


def decode_arrays(grid: Grid, splits, discos, inj):
    """Session arrays -> canonical tasks (session.py:207-225 + canonicalize_task)."""
    counts = [len(s.branch_elements) for s in grid.substations]
    out = []
    for b in range(inj.shape[0]):
        sp = []
        if splits is not None:
            for si, n in enumerate(counts):
                bits = np.asarray(splits[b, si, :n], dtype=bool)
                if bits.any():
                    sp.append((si, tuple(bool(x) for x in bits)))
        d = ()
        if discos is not None and discos.shape[1]:
            row = discos[b]
            d = tuple(int(k) for k in row[row >= 0])
        out.append(canonical(grid, sp, d, inj[b]))
    return out


def solve_arrays(grid: Grid, base, splits, discos, inj, cfg) -> list[PortResult]:
    return [solve_one(grid, base, c, cfg) for c in decode_arrays(grid, splits, discos, inj)]


def evaluate(grid: Grid, base, canon: Canon, cfg, winner: Optional[int] = None):
    """Brute-force per-candidate metrics (every feasible case, like `symmetric`,
    solver.py:826-842) and the winner report of candidate ``winner`` (default:
    first argmin).  Returns None for infeasible tasks, else
    (metrics (T,), winner, n0_worst, n1_worst, islanded)."""
    st = _State.of(base)
    try:
        for si, bits in canon.splits:
            st = _split(st, grid, si, bits)
    except _SplitFail:
        return None
    ctx = _branch(grid, st, canon.discos, cfg)
    if not ctx.feasible:
        return None
    rows = canon.rows
    n0 = _n0_block(ctx, rows)
    ccols = _inj_cols(ctx, rows)
    metrics = _rel_max(ctx, n0)
    for ce in ctx.cases:
        if ce.feasible:
            fl = _case_flows(ctx, ce, n0, ccols.get(ce.order), slice(None))
            np.maximum(metrics, _rel_max(ctx, fl), out=metrics)
    if ctx.islanded:
        np.maximum(metrics, cfg.islanding_penalty, out=metrics)
    w = int(np.argmin(metrics)) if winner is None else int(winner)
    n0e, n1e = _report_winner(grid, ctx, cfg, n0, ccols, w)
    return metrics, w, n0e, n1e, tuple(sorted(ctx.islanded))
