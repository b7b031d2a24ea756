"""Library-level solver API, mirroring the reference's `batchdc.solver` entry points.

Types (`SplitAction`, `TopologyTask`, `SolveConfig`, `SparseReport`,
`TaskDiagnostics`, `SolveResult`, `Instrumentation`) and functions
(`canonicalize_task`, `solve_batch`, `solve_prepared`-free flat route) keep the
reference's names, fields, defaults and error messages
(`pkg/src/batchdc/solver.py:44-197, 970-1003`).  The numerical work of
``solve_batch`` runs entirely on the GPU through the C-ABI engine
(``engine.py`` -> ``libbdc.so``); there is no CPU fallback.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .errors import ValidationError
from .grid import Grid

MODES = ("output_first", "metric_first", "symmetric")
ISLANDING_POLICIES = ("penalize", "error")
MULTI_OUTAGE_METHODS = ("modf", "sequential")


@dataclass(frozen=True)
class SplitAction:
    """Split one substation with the given branch-element assignment bits."""

    substation: int
    assignment: tuple[bool, ...]


@dataclass(frozen=True)
class TopologyTask:
    """One branch topology plus the injection candidates to brute-force over it."""

    splits: tuple[SplitAction, ...] = ()
    disconnections: tuple[int, ...] = ()
    injection_sets: tuple[tuple[bool, ...], ...] = ((),)


@dataclass(frozen=True)
class SolveConfig:
    """Solver knobs with the reference's defaults (`solver.py:61-91`).

    ``mode`` selects the reference's evaluation order; all three modes are
    bit-identical there and produce identical results here: ``metric_first`` runs
    the engine's exact dominance screen (pairs that provably cannot move a metric
    are skipped), ``symmetric`` and ``output_first`` evaluate every (case,
    candidate) pair; the winner's report is built once, in FP64, either way.
    ``workers`` / ``max_batch`` are accepted for drop-in compatibility: the
    device engine processes tasks in waves sized by device memory.
    """

    mode: str = "metric_first"
    topk_per_case: int = 5
    topk_global: int = 10
    workers: int = 1
    islanding_policy: str = "penalize"
    islanding_penalty: float = 10.0
    multi_outage_method: str = "modf"
    max_simultaneous_outages: int = 8
    max_batch: int = 0

    def validate(self) -> None:
        if self.mode not in MODES:
            raise ValidationError(f"unknown mode {self.mode!r}")
        if self.islanding_policy not in ISLANDING_POLICIES:
            raise ValidationError(f"unknown islanding policy {self.islanding_policy!r}")
        if self.multi_outage_method not in MULTI_OUTAGE_METHODS:
            raise ValidationError(f"unknown multi-outage method {self.multi_outage_method!r}")
        if self.topk_per_case < 1 or self.topk_global < 1:
            raise ValidationError("top-k limits must be >= 1")
        if self.workers < 1:
            raise ValidationError("workers must be >= 1")
        if self.max_simultaneous_outages < 1:
            raise ValidationError("max_simultaneous_outages must be >= 1")
        if not self.islanding_penalty > 0.0:
            raise ValidationError("islanding penalty must be > 0")


@dataclass(frozen=True)
class SparseReport:
    """Worst loadings of the winning candidate (`solver.py:94-105`)."""

    n0_worst: tuple[tuple[str, float, float], ...]
    n1_worst: tuple[tuple[str, str, float, float], ...]


@dataclass(frozen=True)
class TaskDiagnostics:
    feasible: bool
    reason: Optional[str] = None
    islanded_cases: tuple[str, ...] = ()


@dataclass(frozen=True)
class SolveResult:
    metric: Optional[float]
    best_injection: Optional[int]
    report: Optional[SparseReport]
    diagnostics: TaskDiagnostics


class Instrumentation:
    """Thread-safe counters (`solver.py:123-145`)."""

    def __init__(self) -> None:
        self._lock = threading.Lock()
        self.bsdf_applications = 0
        self.tasks_solved = 0
        self.loadflows = 0
        self.peak_live_ptdfs = 0

    def count_bsdf(self, n: int = 1) -> None:
        with self._lock:
            self.bsdf_applications += n

    def count_task(self, loadflows: int) -> None:
        with self._lock:
            self.tasks_solved += 1
            self.loadflows += loadflows

    def count_tasks(self, n: int, loadflows: int) -> None:
        with self._lock:
            self.tasks_solved += n
            self.loadflows += loadflows

    def note_live_ptdfs(self, n: int) -> None:
        with self._lock:
            self.peak_live_ptdfs = max(self.peak_live_ptdfs, n)


def canonicalize_task(grid: Grid, task: TopologyTask) -> TopologyTask:
    """Validate and canonicalise one task (`solver.py:148-197`)."""
    seen: set[int] = set()
    splits = []
    for sp in task.splits:
        if not 0 <= sp.substation < len(grid.substations):
            raise ValidationError(f"substation index {sp.substation} out of range")
        if sp.substation in seen:
            raise ValidationError(f"substation {sp.substation} split twice in one task")
        seen.add(sp.substation)
        n_el = len(grid.substations[sp.substation].branch_elements)
        if len(sp.assignment) != n_el:
            raise ValidationError(
                f"substation {sp.substation}: assignment has {len(sp.assignment)} bits, "
                f"expected {n_el}"
            )
        if any(sp.assignment):
            splits.append(SplitAction(sp.substation, tuple(bool(b) for b in sp.assignment)))
    splits.sort(key=lambda s: (s.substation, s.assignment))
    if len(set(task.disconnections)) != len(task.disconnections):
        raise ValidationError("duplicate branch in disconnections")
    for k in task.disconnections:
        if not 0 <= k < grid.n_branches:
            raise ValidationError(f"disconnection branch {k} out of range")
    K = len(grid.injection_slots)
    if not task.injection_sets:
        raise ValidationError("task needs at least one injection set")
    rows = []
    for row in task.injection_sets:
        if len(row) == 0 and K > 0:
            rows.append((False,) * K)
            continue
        if len(row) != K:
            raise ValidationError(f"injection set has {len(row)} bits, expected {K}")
        rows.append(tuple(bool(b) for b in row))
    return TopologyTask(tuple(splits), tuple(task.disconnections), tuple(rows))


def tasks_to_arrays(grid: Grid, tasks: Sequence[TopologyTask]):
    """Canonical tasks -> engine arrays (splits (B,S,E) u8, discos (B,D) i64,
    inj (B,Tmax,K) u8, t_count (B,) i32).  Tasks with fewer candidates are padded
    by repeating candidate 0; the engine ignores rows >= t_count."""
    B = len(tasks)
    S = len(grid.substations)
    E = max((len(s.branch_elements) for s in grid.substations), default=0)
    K = len(grid.injection_slots)
    D = max((len(t.disconnections) for t in tasks), default=0)
    Tm = max((len(t.injection_sets) for t in tasks), default=1)
    splits = np.zeros((B, S, max(E, 1)), dtype=np.uint8)
    discos = np.full((B, D), -1, dtype=np.int64)
    inj = np.zeros((B, Tm, K), dtype=np.uint8)
    tcount = np.zeros(B, dtype=np.int32)
    for b, t in enumerate(tasks):
        for sp in t.splits:
            splits[b, sp.substation, : len(sp.assignment)] = sp.assignment
        discos[b, : len(t.disconnections)] = t.disconnections
        rows = np.array(t.injection_sets, dtype=np.uint8).reshape(len(t.injection_sets), K)
        inj[b, : len(rows)] = rows
        inj[b, len(rows):] = rows[0]
        tcount[b] = len(rows)
    return splits, discos, inj, tcount


@dataclass
class CaseFlows:
    """Raw engine flows of one task (`solver.py:903-916`): ``n0`` is (R, T); ``n1`` has
    one (R, T) array per contingency case in contingency order, None where the case
    islands the topology.  Rows follow ``row_branches``."""

    feasible: bool
    reason: Optional[str] = None
    row_branches: Optional[np.ndarray] = None
    n0: Optional[np.ndarray] = None
    n1: Optional[list] = None
    islanded_cases: tuple[str, ...] = ()


def candidate_case_flows(grid: Grid, base, task: TopologyTask, config: Optional[SolveConfig] = None) -> CaseFlows:
    """Every flow vector the solver scores for one task (`solver.py:919-958`), computed on
    the GPU by the production kernels' factors (``bdc_probe_flows`` -> ``k_probe``, FP64):
    splits, disconnections, case factors and candidate columns exactly as ``solve_batch``
    forms them, returned instead of aggregated."""
    from .engine import TASK_ISLAND_ERROR, TASK_OK, Engine, task_reason
    from .ptdf import check_base_ptdf

    config = config or SolveConfig()
    config.validate()
    check_base_ptdf(grid, base)
    canon = canonicalize_task(grid, task)
    engine = Engine.for_grid(grid, base, config)
    splits, discos, inj, _ = tasks_to_arrays(grid, [canon])
    st, sa, n0, n1, ok = engine.probe_flows(splits[0], discos[0], inj[0])
    islanded = [i for i in range(len(ok)) if not ok[i]]
    if st not in (TASK_OK, TASK_ISLAND_ERROR):
        return CaseFlows(feasible=False, reason=task_reason(engine, st, sa, splits[0], discos[0], []))
    ids = tuple(grid.contingencies[i].id for i in islanded)
    if st == TASK_ISLAND_ERROR:
        # the error policy reports the islanded cases in case order (solver.py:501-511)
        return CaseFlows(feasible=False, reason=task_reason(engine, st, sa, splits[0], discos[0], islanded),
                         islanded_cases=ids)
    return CaseFlows(
        feasible=True,
        row_branches=np.array(base.row_branches, copy=True),
        n0=n0,
        n1=[None if not ok[i] else n1[i] for i in range(len(ok))],
        islanded_cases=ids,
    )


def solve_batch(
    grid: Grid,
    base,
    tasks: Sequence[TopologyTask],
    config: Optional[SolveConfig] = None,
    instrumentation: Optional[Instrumentation] = None,
) -> list[SolveResult]:
    """Evaluate tasks independently against one shared base PTDF (`solver.py:970-1003`).

    Results come back in task order.  All tasks are canonicalised (and
    validated) before any device work starts.
    """
    from .engine import Engine

    config = config or SolveConfig()
    config.validate()
    canon = [canonicalize_task(grid, t) for t in tasks]
    if instrumentation is not None:
        instrumentation.note_live_ptdfs(1)
    if not canon:
        return []
    engine = Engine.for_grid(grid, base, config)
    splits, discos, inj, tcount = tasks_to_arrays(grid, canon)
    out = engine.solve(splits, discos, inj, t_count=tcount)
    if instrumentation is not None:
        instrumentation.count_tasks(len(canon), int(out.loadflows))
        instrumentation.count_bsdf(int(out.bsdf_applications))
    return out.results()
