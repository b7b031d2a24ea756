"""ctypes binding of the C-ABI engine (include/bdc.h -> libbdc.so).

This is the only module that talks to the native library.  There is no CPU
fallback: if ``libbdc.so`` is missing, or no CUDA device is visible, every
solve raises :class:`EngineUnavailable`.

The engine returns array-first results (metrics, winners, statuses, report
entries as indices); :class:`BatchOutput` turns them into the reference's
result objects and documents lazily, so a million-task batch never pays for
a million Python dicts unless someone reads them.
"""

from __future__ import annotations

import ctypes
import os
import threading
from collections import OrderedDict
from collections.abc import Sequence
from typing import Optional

import numpy as np

from .errors import EngineUnavailable, ValidationError
from .grid import Grid
from .ptdf import BaseTables, PtdfMatrix, build_tables

LIB_NAME = "libbdc.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

MAX_RANK = 32
MAX_ELEMENTS = 32
MAX_MULTI = 8
MAX_TOPK = 32
MAX_ACTIVE_SLOTS = 64

TASK_OK = 0
TASK_DEGENERATE_SPLIT = 1
TASK_SINGULAR_SPLIT = 2
TASK_DISCONNECT_ISLAND = 3
TASK_ISLAND_ERROR = 4
TASK_TOO_MANY_OUTAGES = 5
TASK_DETACHED = 6

_P = ctypes.c_void_p

# device-time stages of bdc_solve (include/bdc.h BDC_STAGE_*)
STAGES = ("h2d", "update", "n0", "other_n1", "scale", "topk", "top", "screen", "select", "report", "d2h", "spare")
N_STAGES = len(STAGES)


class _Grid(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("R", "C0", "M", "S", "E", "K", "N1", "NM", "NMB", "NI", "NC", "NBR", "static_col")] + [
        (n, _P)
        for n in (
            "P0", "P0T", "row_from", "row_to", "branch_row", "f0", "p_base", "mon_row", "rating",
            "row_mon_pos", "sub_col", "sub_count", "sub_elem_row", "sub_elem_b", "slot_sub",
            "slot_col", "slot_sp", "sc_row", "sc_order", "sc_delta", "sc_dscale", "D64", "D32", "mc_start",
            "mc_order", "mb_row", "Dm64", "ic_slot", "ic_col", "ic_sp", "ic_order",
        )
    ]


class _Config(ctypes.Structure):
    _fields_ = [
        ("topk_per_case", ctypes.c_int32),
        ("topk_global", ctypes.c_int32),
        ("islanding_policy", ctypes.c_int32),
        ("islanding_penalty", ctypes.c_double),
        ("multi_outage_method", ctypes.c_int32),
        ("max_simultaneous_outages", ctypes.c_int32),
    ]


class _Batch(ctypes.Structure):
    _fields_ = [
        ("B", ctypes.c_int64),
        ("T", ctypes.c_int32),
        ("D", ctypes.c_int32),
        ("splits", _P),
        ("discos", _P),
        ("inj", _P),
        ("t_count", _P),
        ("max_rank", ctypes.c_int32),
        ("inputs_on_device", ctypes.c_int32),
        ("outputs_on_device", ctypes.c_int32),
        ("stream", _P),
        ("metric", _P),
        ("best", _P),
        ("feasible", _P),
        ("status", _P),
        ("status_arg", _P),
        ("n_islanded", _P),
        ("islanded_bits", _P),
        ("n0_count", _P),
        ("n0_pos", _P),
        ("n0_flow", _P),
        ("n0_rel", _P),
        ("n1_count", _P),
        ("n1_case", _P),
        ("n1_pos", _P),
        ("n1_flow", _P),
        ("n1_rel", _P),
        ("cand_metric", _P),
        ("loadflows", _P),
        ("bsdf_applications", _P),
        ("n1_pairs", _P),
        ("report_cases", _P),
        ("screen", ctypes.c_int32),
        ("stage_ms", ctypes.c_float * N_STAGES),
        ("waves", ctypes.c_int32),
        ("kernel_launches", ctypes.c_int32),
        ("rescore_stats", _P),
        ("split_shared", _P),
    ]


EXPORTS = (
    "bdc_device_count",
    "bdc_version",
    "bdc_last_error",
    "bdc_session_create",
    "bdc_session_destroy",
    "bdc_solve",
    "bdc_probe_flows",
    "bdc_session_set_wave",
    "bdc_scan_tasks",
    "bdc_draw_tasks",
    "bdc_spd_solve",
)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libbdc.so (built in-tree by ``__graft_entry__.build()``); fail loudly."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise EngineUnavailable(
                f"{path} is missing: build the CUDA engine first (python -c "
                "'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(path)
        lib.bdc_version.restype = ctypes.c_char_p
        lib.bdc_last_error.restype = ctypes.c_char_p
        lib.bdc_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        lib.bdc_session_create.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Config), ctypes.c_int, ctypes.POINTER(_P)]
        lib.bdc_session_destroy.argtypes = [_P]
        lib.bdc_solve.argtypes = [_P, ctypes.POINTER(_Batch)]
        lib.bdc_probe_flows.argtypes = [_P, _P, _P, ctypes.c_int32, _P, ctypes.c_int32, _P, _P, _P, _P, _P]
        lib.bdc_session_set_wave.argtypes = [_P, ctypes.c_int64]
        lib.bdc_scan_tasks.argtypes = [_P, _P, _P, ctypes.c_int64, ctypes.c_int32, _P, _P, _P]
        lib.bdc_spd_solve.argtypes = [ctypes.c_int, _P, ctypes.c_int32, _P, ctypes.c_int32, _P, _P]
        lib.bdc_draw_tasks.argtypes = [_P, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _P, _P, _P, _P]
        _lib = lib
        return lib


def device_count() -> int:
    lib = load_library()
    n = ctypes.c_int(0)
    lib.bdc_device_count(ctypes.byref(n))
    return int(n.value)


def _err(lib) -> str:
    msg = lib.bdc_last_error()
    return msg.decode() if msg else "unknown engine error"


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class Engine:
    """One grid + config resident on one GPU (a ``bdc_session``)."""

    _cache: "OrderedDict[tuple, Engine]" = OrderedDict()
    _cache_lock = threading.Lock()

    def __init__(self, grid: Grid, base: PtdfMatrix, config, device: int = 0):
        config.validate()
        if config.topk_per_case > MAX_TOPK or config.topk_global > MAX_TOPK:
            raise ValidationError(
                f"topk_per_case/topk_global above {MAX_TOPK} exceed the engine limit"
            )
        self.lib = load_library()
        if device_count() < 1:
            raise EngineUnavailable("no CUDA device visible; the engine has no CPU fallback")
        self.grid = grid
        self.base = base
        self.config = config
        self.device = device
        # SolveConfig.mode (solver.py:777-842): metric_first runs the exact dominance
        # screen (solver.py:798-822); symmetric and output_first evaluate every
        # (case, candidate) pair, as those modes do.  All three give bit-identical
        # results (tests/test_gpu_large.py::test_modes_are_bit_identical).
        self.screen = config.mode == "metric_first"
        self.tables = tb = build_tables(grid, base)
        if tb.E > MAX_ELEMENTS:
            raise ValidationError(f"substations with more than {MAX_ELEMENTS} branch elements")
        if tb.NM and int(np.max(np.diff(tb.mc_start))) > MAX_MULTI:
            raise ValidationError(f"multi-branch cases with more than {MAX_MULTI} branches")
        self.case_ids = [c.id for c in grid.contingencies]
        self.branch_ids = [grid.branches[int(k)].id for k in tb.mon_branch]
        self.element_counts = np.array([len(s.branch_elements) for s in grid.substations], dtype=np.int64)
        slots_per_sub = np.zeros(len(grid.substations), dtype=np.int64)
        for si, j in grid.injection_slots:
            if grid.injections[j].setpoint != 0.0:
                slots_per_sub[si] += 1
        self.slots_per_sub = slots_per_sub
        branch_row = np.ascontiguousarray(base.branch_rows.astype(np.int32))
        self.branch_row = branch_row
        self._keep = keep = {}

        def arr(name, a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            if a.size == 0:
                a = np.zeros(1, dtype=dt)
            keep[name] = a
            return ctypes.c_void_p(a.ctypes.data)

        g = _Grid()
        g.R, g.C0, g.M, g.S, g.E, g.K = tb.R, tb.C0, tb.M, tb.S, tb.E if tb.S else 1, tb.K
        g.N1, g.NM, g.NMB, g.NI, g.NC = tb.N1, tb.NM, len(tb.mb_row), tb.NI, len(grid.contingencies)
        g.NBR = grid.n_branches
        g.static_col = -1 if base.static_col is None else int(base.static_col)
        g.P0 = arr("P0", tb.P0, np.float64)
        g.P0T = arr("P0T", tb.P0T, np.float64)
        g.row_from = arr("row_from", tb.row_from, np.int32)
        g.row_to = arr("row_to", tb.row_to, np.int32)
        g.branch_row = arr("branch_row", branch_row, np.int32)
        g.f0 = arr("f0", tb.f0, np.float64)
        g.p_base = arr("p_base", tb.p_base, np.float64)
        g.mon_row = arr("mon_row", tb.mon_row, np.int32)
        g.rating = arr("rating", tb.rating, np.float64)
        g.row_mon_pos = arr("row_mon_pos", tb.row_mon_pos, np.int32)
        g.sub_col = arr("sub_col", tb.sub_col, np.int32)
        g.sub_count = arr("sub_count", tb.sub_count, np.int32)
        g.sub_elem_row = arr("sub_elem_row", tb.sub_elem_row, np.int32)
        g.sub_elem_b = arr("sub_elem_b", tb.sub_elem_b, np.float64)
        g.slot_sub = arr("slot_sub", tb.slot_sub, np.int32)
        g.slot_col = arr("slot_col", tb.slot_col, np.int32)
        g.slot_sp = arr("slot_sp", tb.slot_sp, np.float64)
        g.sc_row = arr("sc_row", tb.sc_row, np.int32)
        g.sc_order = arr("sc_order", tb.sc_order, np.int32)
        g.sc_delta = arr("sc_delta", tb.sc_delta, np.float64)
        g.sc_dscale = arr("sc_dscale", tb.sc_dscale, np.float64)
        g.D64 = arr("D64", tb.D64, np.float64)
        g.D32 = arr("D32", tb.D32, np.float32)
        g.mc_start = arr("mc_start", tb.mc_start, np.int32)
        g.mc_order = arr("mc_order", tb.mc_order, np.int32)
        g.mb_row = arr("mb_row", tb.mb_row, np.int32)
        g.Dm64 = arr("Dm64", tb.Dm64, np.float64)
        g.ic_slot = arr("ic_slot", tb.ic_slot, np.int32)
        g.ic_col = arr("ic_col", tb.ic_col, np.int32)
        g.ic_sp = arr("ic_sp", tb.ic_sp, np.float64)
        g.ic_order = arr("ic_order", tb.ic_order, np.int32)
        c = _Config()
        c.topk_per_case = config.topk_per_case
        c.topk_global = config.topk_global
        c.islanding_policy = 0 if config.islanding_policy == "penalize" else 1
        c.islanding_penalty = float(config.islanding_penalty)
        c.multi_outage_method = 0 if config.multi_outage_method == "modf" else 1
        c.max_simultaneous_outages = int(min(config.max_simultaneous_outages, 2**31 - 1))
        handle = ctypes.c_void_p()
        rc = self.lib.bdc_session_create(ctypes.byref(g), ctypes.byref(c), device, ctypes.byref(handle))
        self._keep = None  # uploaded; host copies no longer needed
        if rc != 0:
            raise EngineUnavailable(f"bdc_session_create failed ({rc}): {_err(self.lib)}")
        self.handle = handle

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.bdc_session_destroy(h)
            except Exception:
                pass
            self.handle = None

    @classmethod
    def for_grid(cls, grid: Grid, base: PtdfMatrix, config, device: int = 0) -> "Engine":
        key = (id(grid), id(base), config, device)
        with cls._cache_lock:
            eng = cls._cache.get(key)
            if eng is not None and eng.grid is grid and eng.base is base:
                cls._cache.move_to_end(key)
                return eng
        eng = cls(grid, base, config, device)
        with cls._cache_lock:
            cls._cache[key] = eng
            while len(cls._cache) > 4:
                cls._cache.popitem(last=False)
        return eng

    def set_wave(self, max_tasks: int) -> None:
        self.lib.bdc_session_set_wave(self.handle, int(max_tasks))

    # ------------------------------------------------------------------ checks
    def check_batch(self, splits: np.ndarray, discos: np.ndarray) -> int:
        """Engine limits of one batch (native scan of the task arrays, no device work);
        returns the workspace rank stride max(k + d).  ``splits`` (B,S,E) u8,
        ``discos`` (B,D) i64."""
        B = int(splits.shape[0])
        D = int(discos.shape[1]) if discos.ndim == 2 else 0
        mr, md, ma = ctypes.c_int32(0), ctypes.c_int32(0), ctypes.c_int32(0)
        sp = np.ascontiguousarray(splits, dtype=np.uint8)
        dc = np.ascontiguousarray(discos, dtype=np.int64)
        rc = self.lib.bdc_scan_tasks(
            self.handle, _ptr(sp) if sp.size else None, _ptr(dc) if dc.size else None, B, D,
            ctypes.byref(mr), ctypes.byref(md), ctypes.byref(ma),
        )
        if rc != 0:
            raise EngineUnavailable(f"bdc_scan_tasks failed ({rc}): {_err(self.lib)}")
        rmax, dmax, amax = int(mr.value), int(md.value), int(ma.value)
        if dmax > 0:
            self._check_outage_columns(dc)
        if rmax > MAX_RANK:
            raise ValidationError(
                f"a task applies {rmax} splits + disconnections; the engine supports {MAX_RANK}"
            )
        if self.config.multi_outage_method == "modf" and dmax > MAX_MULTI:
            if dmax <= self.config.max_simultaneous_outages:
                raise ValidationError(
                    f"{dmax} simultaneous disconnections exceed the engine's MODF limit of {MAX_MULTI}"
                )
        if amax > MAX_ACTIVE_SLOTS:
            raise ValidationError(
                f"a task moves {amax} injection slots; the engine supports {MAX_ACTIVE_SLOTS}"
            )
        return max(rmax, 1)

    def _check_outage_columns(self, discos: np.ndarray) -> None:
        """A disconnection needs a retained row with both endpoint columns present: the
        reference raises ValidationError for the batch otherwise (`factors.py:65-67`,
        `compute_modf` `:391-392`, `lodf_column` `:345-346`), for the first such task."""
        tb = self.tables
        d = discos[discos >= 0] if discos.size else discos
        if not d.size:
            return
        rows = self.branch_row[d]
        bad_rows = rows < 0
        safe = np.where(bad_rows, 0, rows)
        folded = (np.asarray(tb.row_from)[safe] < 0) | (np.asarray(tb.row_to)[safe] < 0)
        if not (bad_rows | folded).any():
            return
        for b in range(discos.shape[0]):
            for k in discos[b]:
                k = int(k)
                if k < 0:
                    continue
                r = int(self.branch_row[k])
                if r < 0:
                    raise ValidationError(f"branch {k} has no retained PTDF row")
                if tb.row_from[r] < 0 or tb.row_to[r] < 0:
                    if self.config.multi_outage_method == "sequential":
                        raise ValidationError(f"branch {k}: endpoint column folded, cannot outage")
                    raise ValidationError("outage branch endpoint column folded")

    # ------------------------------------------------------------------ solve
    def solve(
        self,
        splits: np.ndarray,
        discos: np.ndarray,
        inj: np.ndarray,
        t_count: Optional[np.ndarray] = None,
        want_candidates: bool = False,
        max_rank: Optional[int] = None,
    ) -> "BatchOutput":
        """Host arrays in, host arrays out (e2e path; copies inside the call)."""
        tb = self.tables
        B = int(inj.shape[0])
        T = int(inj.shape[1]) if inj.ndim == 3 else 1
        E = tb.E if tb.S else 1
        splits = np.ascontiguousarray(splits, dtype=np.uint8).reshape(B, tb.S, -1) if tb.S else np.zeros((B, 0, 1), np.uint8)
        if splits.shape[2] != E:
            pad = np.zeros((B, tb.S, E), dtype=np.uint8)
            pad[:, :, : min(E, splits.shape[2])] = splits[:, :, :E]
            splits = pad
        discos = np.ascontiguousarray(discos, dtype=np.int64).reshape(B, -1)
        inj = np.ascontiguousarray(inj, dtype=np.uint8).reshape(B, T, tb.K)
        if max_rank is None:
            max_rank = self.check_batch(splits, discos)
        kg = self.config.topk_global
        ncw = max(1, (len(self.case_ids) + 31) // 32)
        out = BatchOutput(self, B, T, kg, ncw, splits, discos, inj, want_candidates)
        bt = _Batch()
        bt.B, bt.T, bt.D = B, T, discos.shape[1]
        bt.splits, bt.discos, bt.inj = _ptr(splits), _ptr(discos) if discos.size else None, _ptr(inj)
        tc = None
        if t_count is not None:
            tc = np.ascontiguousarray(t_count, dtype=np.int32)
            bt.t_count = _ptr(tc)
        bt.max_rank = int(max_rank)
        bt.inputs_on_device = 0
        bt.outputs_on_device = 0
        out.bind(bt)
        if B:
            rc = self.lib.bdc_solve(self.handle, ctypes.byref(bt))
            if rc != 0:
                raise EngineUnavailable(f"bdc_solve failed ({rc}): {_err(self.lib)}")
        out.finish(bt)
        return out

    def solve_device(self, splits, discos, inj, outputs: dict, stream_ptr: int, max_rank: int,
                     loadflows: Optional[np.ndarray] = None):
        """Device-resident inputs and outputs (torch CUDA tensors / raw pointers).

        ``splits`` (B,S,E) u8, ``discos`` (B,D) i64, ``inj`` (B,T,K) u8 as CUDA
        tensors; ``outputs`` maps BdcBatch output names to CUDA tensors.  Runs on
        ``stream_ptr`` so callers can bracket it with their own CUDA events.
        Returns (stage_ms, waves, kernel_launches, loadflows)."""
        B, T = int(inj.shape[0]), int(inj.shape[1])
        bt = _Batch()
        bt.B, bt.T, bt.D = B, T, int(discos.shape[1])
        bt.splits = ctypes.c_void_p(splits.data_ptr())
        bt.discos = ctypes.c_void_p(discos.data_ptr()) if discos.numel() else None
        bt.inj = ctypes.c_void_p(inj.data_ptr())
        bt.t_count = None
        bt.max_rank = int(max_rank)
        bt.inputs_on_device = 1
        bt.outputs_on_device = 1
        bt.stream = ctypes.c_void_p(stream_ptr)
        for name, t in outputs.items():
            setattr(bt, name, ctypes.c_void_p(t.data_ptr()))
        lf = loadflows if loadflows is not None else np.zeros(1, dtype=np.int64)
        pairs = np.zeros(1, dtype=np.int64)
        rcases = np.zeros(1, dtype=np.int64)
        bt.loadflows = _ptr(lf)
        bt.n1_pairs = _ptr(pairs)
        bt.report_cases = _ptr(rcases)
        rstats = np.zeros(3, dtype=np.int64)
        bt.rescore_stats = _ptr(rstats)
        sshared = np.zeros(1, dtype=np.int64)
        bt.split_shared = _ptr(sshared)
        bt.screen = int(self.screen)
        rc = self.lib.bdc_solve(self.handle, ctypes.byref(bt))
        if rc != 0:
            raise EngineUnavailable(f"bdc_solve failed ({rc}): {_err(self.lib)}")
        self.last_pairs = int(pairs[0])
        self.last_report_cases = int(rcases[0])
        self.last_rescore = [int(x) for x in rstats]
        self.last_split_shared = int(sshared[0])
        return [float(x) for x in bt.stage_ms], int(bt.waves), int(bt.kernel_launches), int(lf[0])

    def probe_flows(self, splits_row: np.ndarray, discos_row: np.ndarray, inj_rows: np.ndarray):
        """Every flow of one task on the device (candidate_case_flows)."""
        tb = self.tables
        E = tb.E if tb.S else 1
        sp = np.zeros((max(tb.S, 1), E), dtype=np.uint8)
        if tb.S:
            sp[:, : splits_row.shape[1]] = splits_row
        dr = np.ascontiguousarray(discos_row, dtype=np.int64).reshape(-1)
        T = inj_rows.shape[0]
        inj = np.ascontiguousarray(inj_rows, dtype=np.uint8).reshape(T, tb.K)
        n0 = np.zeros((tb.R, T))
        nc = len(self.case_ids)
        n1 = np.zeros((max(nc, 1), tb.R, T))
        ok = np.zeros(max(nc, 1), dtype=np.uint8)
        st = ctypes.c_int32(0)
        sa = ctypes.c_int32(0)
        rc = self.lib.bdc_probe_flows(
            self.handle, _ptr(sp), _ptr(dr) if dr.size else None, int(dr.size), _ptr(inj), T,
            _ptr(n0), _ptr(n1), _ptr(ok), ctypes.byref(st), ctypes.byref(sa),
        )
        if rc != 0:
            raise EngineUnavailable(f"bdc_probe_flows failed ({rc}): {_err(self.lib)}")
        return int(st.value), int(sa.value), n0, n1[:nc], ok[:nc].astype(bool)


def task_reason(eng: Engine, st: int, arg: int, splits_row: np.ndarray, discos_row: np.ndarray,
                islanded_orders: Sequence[int]) -> Optional[str]:
    """The reference's infeasibility message for an engine status code: the str() of the
    first failing split's exception (factors.py:493-495, 516-518), the MODF / sequential
    islanding message (solver.py:401-406) or the error-policy message (solver.py:501-511)."""
    grid = eng.grid
    if st == TASK_OK:
        return None
    if st in (TASK_DEGENERATE_SPLIT, TASK_SINGULAR_SPLIT):
        si = [int(s) for s in np.flatnonzero(np.asarray(splits_row).any(axis=1))][arg]
        node = grid.substations[si].node
        if st == TASK_DEGENERATE_SPLIT:
            return f"split of node {node} leaves busbar A without any branch"
        n = len(grid.substations[si].branch_elements)
        bits = [bool(x) for x in splits_row[si, :n]]
        return f"split of node {node} with assignment {bits} disconnects the grid"
    if st == TASK_DISCONNECT_ISLAND:
        row = np.asarray(discos_row).reshape(-1)
        ks = [int(k) for k in row[row >= 0]]
        if arg >= 0:
            return f"disconnections island the grid: outage of branch {ks[arg]} islands the grid"
        return f"disconnections island the grid: simultaneous outage of branches {ks} islands the grid"
    if st == TASK_ISLAND_ERROR:
        ids = [eng.case_ids[o] for o in islanded_orders]
        return f"islanding under contingencies {ids}"
    return f"engine status {st}"


class BatchOutput:
    """Array-first results of one ``bdc_solve`` call."""

    def __init__(self, eng: Engine, B, T, kg, ncw, splits, discos, inj, want_candidates):
        self.engine = eng
        self.B, self.T, self.kg = B, T, kg
        self.splits, self.discos, self.inj = splits, discos, inj
        # every element is written by bdc_solve (report rows past their count are scratch);
        # np.empty keeps the host allocation off the e2e path
        self.metric = np.empty(B)
        self.best = np.empty(B, dtype=np.int64)
        self.feasible = np.empty(B, dtype=np.uint8)
        self.status = np.empty(B, dtype=np.int32)
        self.status_arg = np.empty(B, dtype=np.int32)
        self.n_islanded = np.empty(B, dtype=np.int32)
        self.islanded_bits = np.empty((B, ncw), dtype=np.uint32)
        self.n0_count = np.empty(B, dtype=np.int32)
        self.n0_pos = np.empty((B, kg), dtype=np.int32)
        self.n0_flow = np.empty((B, kg))
        self.n0_rel = np.empty((B, kg))
        self.n1_count = np.empty(B, dtype=np.int32)
        self.n1_case = np.empty((B, kg), dtype=np.int32)
        self.n1_pos = np.empty((B, kg), dtype=np.int32)
        self.n1_flow = np.empty((B, kg))
        self.n1_rel = np.empty((B, kg))
        self.cand_metric = np.empty((B, T), dtype=np.float32) if want_candidates else None
        self._lf = np.zeros(1, dtype=np.int64)
        self._bsdf = np.zeros(1, dtype=np.int64)
        self._pairs = np.zeros(1, dtype=np.int64)
        # [0] y-classes re-scored in FP64, [1] winners the re-score replaced,
        # [2] tasks with more than one candidate in the near-tie band
        self.rescore_stats = np.zeros(3, dtype=np.int64)
        self.split_shared = np.zeros(1, dtype=np.int64)  # split applications copied (prefix memo)
        self.stage_ms = [0.0] * N_STAGES
        self.waves = 0
        self.kernel_launches = 0

    def bind(self, bt: _Batch) -> None:
        for name in (
            "metric", "best", "feasible", "status", "status_arg", "n_islanded", "islanded_bits",
            "n0_count", "n0_pos", "n0_flow", "n0_rel", "n1_count", "n1_case", "n1_pos", "n1_flow",
            "n1_rel",
        ):
            setattr(bt, name, _ptr(getattr(self, name)))
        bt.cand_metric = _ptr(self.cand_metric)
        bt.loadflows = _ptr(self._lf)
        bt.bsdf_applications = _ptr(self._bsdf)
        bt.n1_pairs = _ptr(self._pairs)
        bt.rescore_stats = _ptr(self.rescore_stats)
        bt.split_shared = _ptr(self.split_shared)
        bt.screen = int(self.engine.screen)

    def finish(self, bt: _Batch) -> None:
        self.stage_ms = [float(x) for x in bt.stage_ms]
        self.waves = int(bt.waves)
        self.kernel_launches = int(bt.kernel_launches)
        self.feasible = self.feasible.astype(bool)
        bad = np.flatnonzero(self.status == TASK_TOO_MANY_OUTAGES)
        if len(bad):
            d = int((self.discos[bad[0]] >= 0).sum())
            raise ValidationError(
                f"{d} disconnections exceed the cap of {self.engine.config.max_simultaneous_outages}"
            )
        bad = np.flatnonzero(self.status == TASK_DETACHED)
        if len(bad):
            raise ValidationError(
                f"task {int(bad[0])}: engine consistency check failed (code {int(self.status_arg[bad[0]])})"
            )

    @property
    def loadflows(self) -> int:
        return int(self._lf[0])

    @property
    def bsdf_applications(self) -> int:
        return int(self._bsdf[0])

    @property
    def n1_pairs(self) -> int:
        """(single case, candidate) pairs the N-1 sweep evaluated (the rest were
        skipped by the exact dominance screen)."""
        return int(self._pairs[0])

    # ------------------------------------------------------------ decoding
    def islanded_orders(self, b: int) -> list[int]:
        if self.n_islanded[b] == 0:
            return []
        bits = np.unpackbits(self.islanded_bits[b].view(np.uint8), bitorder="little")
        return [int(i) for i in np.flatnonzero(bits[: len(self.engine.case_ids)])]

    def reason(self, b: int) -> Optional[str]:
        return task_reason(
            self.engine, int(self.status[b]), int(self.status_arg[b]), self.splits[b], self.discos[b],
            self.islanded_orders(b),
        )

    def result(self, b: int):
        from .solver import SolveResult, SparseReport, TaskDiagnostics

        if not self.feasible[b]:
            isl = ()
            if int(self.status[b]) == TASK_ISLAND_ERROR:
                isl = tuple(self.engine.case_ids[o] for o in self.islanded_orders(b))
            return SolveResult(None, None, None, TaskDiagnostics(False, self.reason(b), isl))
        bid, cid = self.engine.branch_ids, self.engine.case_ids
        n0 = tuple(
            (bid[int(self.n0_pos[b, i])], float(self.n0_flow[b, i]), float(self.n0_rel[b, i]))
            for i in range(int(self.n0_count[b]))
        )
        n1 = tuple(
            (cid[int(self.n1_case[b, i])], bid[int(self.n1_pos[b, i])], float(self.n1_flow[b, i]), float(self.n1_rel[b, i]))
            for i in range(int(self.n1_count[b]))
        )
        isl = tuple(sorted(cid[o] for o in self.islanded_orders(b)))
        return SolveResult(
            float(self.metric[b]), int(self.best[b]), SparseReport(n0, n1), TaskDiagnostics(True, None, isl)
        )

    def results(self) -> list:
        return [self.result(b) for b in range(self.B)]

    def report(self, b: int) -> dict:
        from .io import result_to_dict

        return result_to_dict(self.result(b))

    def reports(self) -> "LazyReports":
        return LazyReports(self)


class LazyReports(Sequence):
    """The per-task result documents, built on access (compares equal to a list)."""

    def __init__(self, out: BatchOutput):
        self._out = out
        self._cache: dict[int, dict] = {}

    def __len__(self) -> int:
        return self._out.B

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        doc = self._cache.get(i)
        if doc is None:
            doc = self._cache[i] = self._out.report(i)
        return doc

    def __eq__(self, other):
        if isinstance(other, (list, tuple, LazyReports)):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __repr__(self) -> str:
        return f"LazyReports({len(self)} tasks)"
