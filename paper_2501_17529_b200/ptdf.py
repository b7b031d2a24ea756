"""Base PTDF setup (host, once per grid) and the flat tables the engine uploads.

Setup is not the hot path: the reduced susceptance matrix of the base
topology is factorised exactly once per session, the static nodes are folded
into one column, and the result is flattened into the device-resident tables
of ``BaseTables``.  Every topology after that is reached on the GPU through
low-rank updates of these tables; nothing is ever refactorised.

Follows the reference's `compute_ptdf` (`pkg/src/batchdc/factors.py:161-216`),
`reduce_static` (`:219-275`) and `prepare_base_ptdf` (`:597-612`) for the
matrix and its row/column bookkeeping, and `_static_base_flows` /
`_bind_slots` (`solver.py:526-572`) for the fixed injection pattern.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional, Sequence

import numpy as np
import scipy.linalg

from .errors import InvalidReduction, SingularSystem, ValidationError
from .grid import (
    INJECTION,
    MULTI_BRANCH,
    SINGLE_BRANCH,
    Grid,
    static_injection_fold,
    structurally_required_nodes,
)

ISLANDING_TOL = 1e-8  # reference factors.py:48
SPLIT_TOL = 1e-8      # reference factors.py:49


@dataclass(frozen=True)
class PtdfMatrix:
    """Base PTDF with the row/column bookkeeping of `factors.py:55-109`.

    ``values`` is (R, C) float64: effective node columns, then the static
    column (folded flows, always last when present).
    """

    values: np.ndarray
    row_branches: np.ndarray
    branch_rows: np.ndarray
    node_cols: np.ndarray
    from_cols: np.ndarray
    to_cols: np.ndarray
    slack_col: int
    static_col: Optional[int] = None
    col_origin: tuple = ()
    applied_updates: tuple = ()

    @property
    def n_rows(self) -> int:
        return self.values.shape[0]

    @property
    def n_cols(self) -> int:
        return self.values.shape[1]

    def row_of(self, branch: int) -> int:
        r = int(self.branch_rows[branch])
        if r < 0:
            raise ValidationError(f"branch {branch} has no retained PTDF row")
        return r


def _laplacian(grid: Grid) -> tuple[np.ndarray, np.ndarray]:
    n, e = grid.n_nodes, grid.n_branches
    f, t, b = grid.from_nodes, grid.to_nodes, grid.susceptances
    inc = np.zeros((e, n))
    inc[np.arange(e), f] = b
    inc[np.arange(e), t] -= b
    lap = np.zeros((n, n))
    np.add.at(lap, (f, f), b)
    np.add.at(lap, (t, t), b)
    np.add.at(lap, (f, t), -b)
    np.add.at(lap, (t, f), -b)
    return lap, inc


def _spd_solve_device(lap, rhs, device: int):
    """lap^-1 rhs for SPD `lap` on the GPU (`bdc_spd_solve`: blocked FP64 potrf + potrs,
    csrc/bdc_chol.cu), the device counterpart of scipy.linalg.solve(assume_a="pos").
    numpy arrays in -> numpy out; CUDA tensors in -> the solution as a CUDA tensor
    (`lap` and `rhs` are overwritten)."""
    import ctypes

    import torch

    from .engine import _err, load_library

    lib = load_library()
    on_dev = isinstance(lap, torch.Tensor)
    n, m = lap.shape[0], rhs.shape[1]
    dev = torch.device("cuda", device)
    A = lap if on_dev else torch.from_numpy(np.ascontiguousarray(lap, dtype=np.float64)).to(dev)
    B = rhs if on_dev else torch.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64)).to(dev)
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    rc = lib.bdc_spd_solve(int(device), ctypes.c_void_p(A.data_ptr()), int(n), ctypes.c_void_p(B.data_ptr()),
                           int(m), ctypes.c_void_p(info.data_ptr()), ctypes.c_void_p(st.cuda_stream))
    if rc != 0:
        raise SingularSystem(f"susceptance matrix factorization failed: {_err(lib)}")
    bad = int(info.item())
    if bad:
        raise SingularSystem(
            f"susceptance matrix factorization failed: {bad}-th leading minor not positive definite")
    return B if on_dev else B.cpu().numpy()


def _ptdf_values_device(grid: Grid, rows: np.ndarray, keep: np.ndarray, device: int) -> np.ndarray:
    """PTDF values (len(rows), n_nodes) with the susceptance matrix and the incidence
    right-hand side assembled on the device from the branch list (no dense host
    matrices), solved by `bdc_spd_solve`, the slack column left at zero."""
    import scipy.sparse as sps
    import torch

    dev = torch.device("cuda", device)
    n, nk = grid.n_nodes, len(keep)
    f, t, b = grid.from_nodes, grid.to_nodes, grid.susceptances
    # Laplacian entries (duplicates -- parallel branches -- summed), slack row/column dropped
    lap = sps.coo_matrix((np.concatenate([b, b, -b, -b]),
                          (np.concatenate([f, t, f, t]), np.concatenate([f, t, t, f]))), shape=(n, n)).tocsr()
    pos = np.full(n, -1, dtype=np.int64)
    pos[keep] = np.arange(nk)
    coo = lap[keep][:, keep].tocoo()
    L = torch.zeros((nk, nk), dtype=torch.float64, device=dev)
    L[torch.from_numpy(coo.row.astype(np.int64)).to(dev), torch.from_numpy(coo.col.astype(np.int64)).to(dev)] = \
        torch.from_numpy(coo.data).to(dev)
    # right-hand side A^T (nk x R): column r holds +b_r at its from node, -b_r at its to node
    R = len(rows)
    rhs = torch.zeros((nk, R), dtype=torch.float64, device=dev)
    for ends, sign in ((f, 1.0), (t, -1.0)):
        p = pos[ends[rows]]
        ok = p >= 0
        rhs[torch.from_numpy(p[ok]).to(dev), torch.from_numpy(np.flatnonzero(ok)).to(dev)] += \
            torch.from_numpy(sign * b[rows][ok]).to(dev)
    X = _spd_solve_device(L, rhs, device)
    vals = torch.zeros((R, n), dtype=torch.float64, device=dev)
    vals[:, torch.from_numpy(keep).to(dev)] = X.T
    return vals.cpu().numpy()


def compute_ptdf(grid: Grid, retained_rows: Optional[Sequence[int]] = None,
                 device: Optional[int] = None) -> PtdfMatrix:
    """One SPD factorisation of the slack-reduced Laplacian (`factors.py:161-216`); with
    `device` the factorisation and solve run on that GPU."""
    if retained_rows is None:
        rows = np.arange(grid.n_branches, dtype=np.int64)
    else:
        rows = np.asarray(retained_rows, dtype=np.int64)
        if len(set(rows.tolist())) != len(rows):
            raise ValidationError("duplicate retained row")
        need = {k for s in grid.substations for k in s.branch_elements}
        need.update(k for c in grid.contingencies for k in c.branches)
        missing = need - set(rows.tolist())
        if missing:
            raise ValidationError(
                "retained rows must include substation/contingency branches, "
                f"missing {sorted(missing)}"
            )
    keep = np.array([i for i in range(grid.n_nodes) if i != grid.slack], dtype=np.int64)
    if device is not None:
        values = _ptdf_values_device(grid, rows, keep, device)
    else:
        lap, inc = _laplacian(grid)
        try:
            part = scipy.linalg.solve(
                lap[np.ix_(keep, keep)], inc[rows][:, keep].T, assume_a="pos"
            ).T
        except (scipy.linalg.LinAlgError, np.linalg.LinAlgError) as exc:
            raise SingularSystem(f"susceptance matrix factorization failed: {exc}") from exc
        values = np.zeros((len(rows), grid.n_nodes))
        values[:, keep] = part
    branch_rows = np.full(grid.n_branches, -1, dtype=np.int64)
    branch_rows[rows] = np.arange(len(rows))
    return PtdfMatrix(
        values=values,
        row_branches=rows,
        branch_rows=branch_rows,
        node_cols=np.arange(grid.n_nodes, dtype=np.int64),
        from_cols=grid.from_nodes[rows].copy(),
        to_cols=grid.to_nodes[rows].copy(),
        slack_col=grid.slack,
        static_col=None,
        col_origin=tuple(("node", i) for i in range(grid.n_nodes)),
    )


def reduce_static(
    ptdf: PtdfMatrix, grid: Grid, static_nodes: Sequence[int], static_power: np.ndarray
) -> PtdfMatrix:
    """Collapse static nodes into one trailing column of fixed flows (`factors.py:219-275`)."""
    if ptdf.applied_updates:
        raise InvalidReduction("reduce_static requires an unmodified base PTDF")
    if ptdf.static_col is not None:
        raise InvalidReduction("PTDF already carries a static column")
    static = sorted({int(s) for s in static_nodes})
    required = set(structurally_required_nodes(grid))
    required.update(grid.injections[j].node for j in grid.movable_injections())
    clash = required.intersection(static)
    if clash:
        raise InvalidReduction(f"static set intersects required nodes {sorted(clash)}")
    power = np.asarray(static_power, dtype=np.float64)
    if power.shape != (grid.n_nodes,):
        raise ValidationError("static_power must have one entry per node")
    st = np.array(static, dtype=np.int64)
    folded = ptdf.values[:, st] @ power[st] if len(st) else np.zeros(ptdf.n_rows)
    static_set = set(static)
    keep = np.array([i for i in range(grid.n_nodes) if i not in static_set], dtype=np.int64)
    remap = np.full(ptdf.n_cols, -1, dtype=np.int64)
    remap[keep] = np.arange(len(keep))
    node_cols = np.full(grid.n_nodes, -1, dtype=np.int64)
    node_cols[keep] = np.arange(len(keep))

    def rm(c: np.ndarray) -> np.ndarray:
        return np.where(c >= 0, remap[np.maximum(c, 0)], -1)

    return replace(
        ptdf,
        values=np.hstack([ptdf.values[:, keep], folded[:, None]]),
        node_cols=node_cols,
        from_cols=rm(ptdf.from_cols),
        to_cols=rm(ptdf.to_cols),
        slack_col=int(remap[ptdf.slack_col]),
        static_col=len(keep),
        col_origin=tuple(("node", int(i)) for i in keep) + (("static",),),
    )


def prepare_base_ptdf(
    grid: Grid, retained_rows: Optional[Sequence[int]] = None, fold_static: bool = True,
    device: Optional[int] = None,
) -> PtdfMatrix:
    """Factorise once and fold static injections (`factors.py:597-612`); `device` runs the
    SPD solve on that GPU."""
    ptdf = compute_ptdf(grid, retained_rows, device=device)
    if not fold_static:
        return ptdf
    fold = static_injection_fold(grid)
    return reduce_static(ptdf, grid, fold.static_nodes, fold.static_power)


def check_base_ptdf(grid: Grid, base: PtdfMatrix) -> None:
    """Reject bases the engine cannot start from (`solver.py:961-967`)."""
    if base.applied_updates:
        raise ValidationError("base PTDF must be free of applied updates")
    mon = np.array(grid.monitored, dtype=np.int64)
    if len(mon) and np.any(base.branch_rows[mon] < 0):
        raise ValidationError("monitored branches must all have retained PTDF rows")


@dataclass
class BaseTables:
    """Everything the device needs about one grid, as flat numpy arrays.

    Row space: the R retained PTDF rows.  Column space: the C0 base columns
    (effective nodes + the static column).  Split columns created by a task
    live at logical ids C0 + j and are never materialised.

    Case tables are grouped by kind; ``*_order`` is each case's position in
    ``grid.contingencies`` (the reference's tie-break and report order).
    """

    R: int
    C0: int
    P0: np.ndarray              # (R, C0) f64 row-major
    P0T: np.ndarray             # (C0, R) f64: columns contiguous
    row_from: np.ndarray        # (R,) i32 base endpoint columns (-1 folded)
    row_to: np.ndarray          # (R,) i32
    f0: np.ndarray              # (R,) f64 base N-0 flows, every slot at home
    p_base: np.ndarray          # (C0,) f64 column power vector, every slot at home
    # monitored rows
    mon_row: np.ndarray         # (M,) i32
    mon_branch: np.ndarray      # (M,) i64 branch index per monitored position
    rating: np.ndarray          # (M,) f64
    row_mon_pos: np.ndarray     # (R,) i32 monitored position of a row, -1 if none
    # substations (S, E padded with -1 / 0)
    sub_col: np.ndarray         # (S,) i32 node column of the substation
    sub_count: np.ndarray       # (S,) i32 branch elements
    sub_elem_row: np.ndarray    # (S, E) i32
    sub_elem_b: np.ndarray      # (S, E) f64 susceptance
    sub_node: np.ndarray        # (S,) i64 dense node index (for reason strings)
    # injection slots
    slot_sub: np.ndarray        # (K,) i32
    slot_col: np.ndarray        # (K,) i32 home column
    slot_sp: np.ndarray         # (K,) f64 setpoint
    # single-branch cases
    sc_row: np.ndarray          # (N1,) i32
    sc_order: np.ndarray        # (N1,) i32
    sc_delta: np.ndarray        # (N1,) f64 D_base(r_c, c)
    sc_dscale: np.ndarray       # (N1,) f64 max_m |D_base(mon_row[m], c)| / rating[m]
    D64: np.ndarray             # (N1, R) f64 D_base columns, case-major
    D32: np.ndarray             # (M, N1) f32 D_base on monitored rows, row-major
    # multi-branch cases (NM cases, NMB = total member branches)
    mc_start: np.ndarray        # (NM+1,) i32 offsets into member arrays
    mc_order: np.ndarray        # (NM,) i32
    mb_row: np.ndarray          # (NMB,) i32
    Dm64: np.ndarray            # (NMB, R) f64 D_base column per member branch
    # injection cases
    ic_slot: np.ndarray         # (NI,) i32 slot index or -1
    ic_col: np.ndarray          # (NI,) i32 fixed column when not a slot
    ic_sp: np.ndarray           # (NI,) f64 setpoint
    ic_order: np.ndarray        # (NI,) i32
    # case kind per contingency order (0 single, 1 multi, 2 injection)
    case_kind: np.ndarray       # (NC,) i32
    case_local: np.ndarray      # (NC,) i32 index within its kind table
    extra: dict = field(default_factory=dict)

    @property
    def M(self) -> int:
        return len(self.mon_row)

    @property
    def S(self) -> int:
        return len(self.sub_col)

    @property
    def E(self) -> int:
        return self.sub_elem_row.shape[1] if self.sub_elem_row.ndim == 2 else 0

    @property
    def K(self) -> int:
        return len(self.slot_col)

    @property
    def N1(self) -> int:
        return len(self.sc_row)

    @property
    def NM(self) -> int:
        return len(self.mc_order)

    @property
    def NI(self) -> int:
        return len(self.ic_slot)


def _dscale(D64: np.ndarray, mon_row: np.ndarray, rating: np.ndarray) -> np.ndarray:
    """Per single case, max over monitored rows of |D_base|/rating (a session constant
    of the device dominance screen's analytic bound), in row blocks to bound memory."""
    out = np.zeros(D64.shape[0])
    if D64.size == 0 or len(mon_row) == 0:
        return out
    inv = 1.0 / rating
    for c0 in range(0, D64.shape[0], 1024):
        blk = np.abs(D64[c0 : c0 + 1024][:, mon_row]) * inv[None, :]
        out[c0 : c0 + 1024] = blk.max(axis=1)
    return out


def build_tables(grid: Grid, base: PtdfMatrix) -> BaseTables:
    """Flatten (grid, base PTDF) into the engine's device tables."""
    check_base_ptdf(grid, base)
    P0 = np.ascontiguousarray(base.values, dtype=np.float64)
    R, C0 = P0.shape
    rows = base.branch_rows

    def row(k: int) -> int:
        r = int(rows[k])
        if r < 0:
            raise ValidationError(f"branch {k} has no retained PTDF row")
        return r

    # fixed injection pattern (`_static_base_flows` + slot homes, solver.py:526-595)
    slots = grid.injection_slots
    slotted = {j for _s, j in slots}
    p_base = np.zeros(C0)
    if base.static_col is not None:
        p_base[base.static_col] = 1.0
    power: dict[int, float] = {}
    for j, inj in enumerate(grid.injections):
        if j not in slotted and inj.setpoint != 0.0:
            power[inj.node] = power.get(inj.node, 0.0) + inj.setpoint
    for node, mw in sorted(power.items()):
        col = int(base.node_cols[node])
        if col < 0:
            if base.static_col is None:
                raise ValidationError(
                    f"node {node} carries immovable power but its column is folded"
                )
            continue
        p_base[col] += mw
    slot_sub = np.zeros(len(slots), dtype=np.int32)
    slot_col = np.zeros(len(slots), dtype=np.int32)
    slot_sp = np.zeros(len(slots))
    for s, (si, j) in enumerate(slots):
        col = int(base.node_cols[grid.injections[j].node])
        if col < 0:
            raise ValidationError(f"injection slot {s}: home column folded")
        slot_sub[s], slot_col[s] = si, col
        slot_sp[s] = grid.injections[j].setpoint
        if slot_sp[s] != 0.0:
            p_base[col] += slot_sp[s]
    f0 = P0 @ p_base

    mon = np.array(grid.monitored, dtype=np.int64)
    mon_row = rows[mon].astype(np.int32) if len(mon) else np.zeros(0, np.int32)
    if np.any(mon_row < 0):
        raise ValidationError("monitored branches must all have retained PTDF rows")
    row_mon_pos = np.full(R, -1, dtype=np.int32)
    row_mon_pos[mon_row] = np.arange(len(mon_row), dtype=np.int32)

    S = len(grid.substations)
    E = max((len(s.branch_elements) for s in grid.substations), default=0)
    sub_col = np.zeros(S, np.int32)
    sub_count = np.zeros(S, np.int32)
    sub_elem_row = np.full((S, max(E, 1)), -1, np.int32)
    sub_elem_b = np.zeros((S, max(E, 1)))
    for si, sub in enumerate(grid.substations):
        a = int(base.node_cols[sub.node])
        if a < 0:
            raise ValidationError(f"substation node {sub.node} column was folded")
        sub_col[si] = a
        sub_count[si] = len(sub.branch_elements)
        for e, k in enumerate(sub.branch_elements):
            sub_elem_row[si, e] = row(k)
            sub_elem_b[si, e] = grid.branches[k].susceptance
    sub_node = np.array([s.node for s in grid.substations], dtype=np.int64)

    fc, tc = base.from_cols, base.to_cols
    sc_row, sc_order, mc_order, mc_start, mb_row = [], [], [], [0], []
    ic_slot, ic_col, ic_sp, ic_order = [], [], [], []
    case_kind = np.zeros(len(grid.contingencies), np.int32)
    case_local = np.zeros(len(grid.contingencies), np.int32)
    slot_of = {}
    for s, (_si, j) in enumerate(slots):
        slot_of.setdefault(j, s)
    for order, case in enumerate(grid.contingencies):
        if case.kind == SINGLE_BRANCH:
            r = row(case.branches[0])
            if fc[r] < 0 or tc[r] < 0:
                raise ValidationError("contingency branch endpoint column folded, cannot outage")
            case_kind[order], case_local[order] = 0, len(sc_row)
            sc_row.append(r)
            sc_order.append(order)
        elif case.kind == MULTI_BRANCH:
            case_kind[order], case_local[order] = 1, len(mc_order)
            for k in case.branches:
                r = row(k)
                if fc[r] < 0 or tc[r] < 0:
                    raise ValidationError("outage branch endpoint column folded")
                mb_row.append(r)
            mc_start.append(len(mb_row))
            mc_order.append(order)
        else:
            case_kind[order], case_local[order] = 2, len(ic_slot)
            j = case.injection
            s = slot_of.get(j)
            col = -1
            if s is None:
                col = int(base.node_cols[grid.injections[j].node])
                if col < 0:
                    raise ValidationError(f"injection contingency {case.id}: node column folded")
            ic_slot.append(-1 if s is None else s)
            ic_col.append(col)
            ic_sp.append(grid.injections[j].setpoint)
            ic_order.append(order)

    def dcols(rr: Sequence[int]) -> np.ndarray:
        rr = np.asarray(rr, dtype=np.int64)
        if len(rr) == 0:
            return np.zeros((0, R))
        return np.ascontiguousarray((P0[:, fc[rr]] - P0[:, tc[rr]]).T)

    sc_row_a = np.array(sc_row, dtype=np.int32)
    D64 = dcols(sc_row_a)
    sc_delta = D64[np.arange(len(sc_row_a)), sc_row_a] if len(sc_row_a) else np.zeros(0)
    D32 = np.ascontiguousarray(D64.T[mon_row].astype(np.float32)) if len(sc_row_a) else np.zeros(
        (len(mon_row), 0), np.float32
    )
    return BaseTables(
        R=R,
        C0=C0,
        P0=P0,
        P0T=np.ascontiguousarray(P0.T),
        row_from=fc.astype(np.int32),
        row_to=tc.astype(np.int32),
        f0=f0,
        p_base=p_base,
        mon_row=mon_row,
        mon_branch=mon,
        rating=grid.ratings[mon].astype(np.float64) if len(mon) else np.zeros(0),
        row_mon_pos=row_mon_pos,
        sub_col=sub_col,
        sub_count=sub_count,
        sub_elem_row=sub_elem_row,
        sub_elem_b=sub_elem_b,
        sub_node=sub_node,
        slot_sub=slot_sub,
        slot_col=slot_col,
        slot_sp=slot_sp,
        sc_row=sc_row_a,
        sc_order=np.array(sc_order, dtype=np.int32),
        sc_delta=np.ascontiguousarray(sc_delta),
        sc_dscale=_dscale(D64, mon_row, grid.ratings[mon] if len(mon) else np.zeros(0)),
        D64=D64,
        D32=D32,
        mc_start=np.array(mc_start, dtype=np.int32),
        mc_order=np.array(mc_order, dtype=np.int32),
        mb_row=np.array(mb_row, dtype=np.int32),
        Dm64=dcols(mb_row),
        ic_slot=np.array(ic_slot, dtype=np.int32),
        ic_col=np.array(ic_col, dtype=np.int32),
        ic_sp=np.array(ic_sp, dtype=np.float64),
        ic_order=np.array(ic_order, dtype=np.int32),
        case_kind=case_kind,
        case_local=case_local,
    )
