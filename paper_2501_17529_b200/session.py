"""Session-based array API -- the drop-in for `batchdc_session`.

Same entry points, argument meaning, validation messages and result shape
as the reference binding (`pkg/bindings/src/batchdc_session/session.py:53-225`):

    session = session_open(grid_or_path_or_doc, config=None)
    out = solve_batch(session, splits (B,S,E), disconnections (B,D), injection_sets (B,T,K))
    out["metrics"], out["best_injection"], out["feasible"], out["reports"]

Differences that are deliberate: opening a session also uploads the grid's
base tables to the GPU, and ``solve_batch`` runs the whole batch there; the
``out["reports"]`` is the reference's list of dicts; ``solve_batch_output`` returns the
array-first results with the documents built lazily on access instead.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Optional, Union

import numpy as np

from .engine import Engine
from .errors import ValidationError
from .grid import Grid
from .io import grid_from_dict, load_grid
from .ptdf import PtdfMatrix, prepare_base_ptdf
from .solver import SolveConfig

__all__ = ["SolverSession", "session_open", "solve_batch", "solve_batch_output"]

GridSource = Union[str, Path, dict, Grid]


@dataclass(frozen=True)
class SolverSession:
    """A grid pinned with its base PTDF, config and device-resident engine."""

    grid: Grid
    base: PtdfMatrix
    config: SolveConfig
    element_counts: tuple[int, ...]
    engine: Engine = field(repr=False, compare=False, default=None)

    @property
    def n_nodes(self) -> int:
        return len(self.grid.node_ids)

    @property
    def n_branches(self) -> int:
        return len(self.grid.branches)

    @property
    def n_cases(self) -> int:
        return len(self.grid.contingencies)

    @property
    def n_substations(self) -> int:
        return len(self.grid.substations)

    @property
    def n_slots(self) -> int:
        return len(self.grid.injection_slots)

    @property
    def split_shape(self) -> tuple[int, int]:
        return (len(self.element_counts), max(self.element_counts, default=0))


def session_open(
    grid: GridSource, config: Optional[SolveConfig] = None, device: int = 0, base_setup: str = "host"
) -> SolverSession:
    """Load a grid, prepare its base PTDF once and upload it (`session.py:92-113`).

    ``base_setup="gpu"`` factorises the susceptance matrix on the session's GPU
    (`bdc_spd_solve`) instead of the host's scipy SPD solve; the base agrees to rounding
    (the reference's own bits come from the host path, the default)."""
    if isinstance(grid, (str, Path)):
        loaded = load_grid(str(grid))
    elif isinstance(grid, dict):
        loaded = grid_from_dict(grid)
    elif isinstance(grid, Grid):
        loaded = grid
    else:
        raise ValidationError(f"unsupported grid source: {type(grid).__name__}")
    cfg = config if config is not None else SolveConfig()
    cfg.validate()
    if base_setup not in ("host", "gpu"):
        raise ValidationError(f"unknown base_setup {base_setup!r}")
    base = prepare_base_ptdf(loaded, device=device if base_setup == "gpu" else None)
    return SolverSession(
        grid=loaded,
        base=base,
        config=cfg,
        element_counts=tuple(len(s.branch_elements) for s in loaded.substations),
        engine=Engine(loaded, base, cfg, device),
    )


def _checked_bits(arr: Any, name: str, ndim: int) -> np.ndarray:
    a = np.ascontiguousarray(arr)
    if a.dtype.kind not in "bui":
        raise ValidationError(f"{name} must be boolean (or 0/1 integer), got {a.dtype}")
    if a.ndim != ndim:
        raise ValidationError(f"{name} must be {ndim}-dimensional, got shape {a.shape}")
    return a.astype(bool, copy=False)


def validate_arrays(session: SolverSession, splits, disconnections, injection_sets):
    """All of `session.py:135-176` plus the canonicalisation checks (`solver.py:174-178`),
    vectorised; raises before any device work."""
    inj = _checked_bits(injection_sets, "injection_sets", 3)
    n_tasks, n_cand, n_bits = inj.shape
    if n_bits != session.n_slots:
        raise ValidationError(
            f"injection_sets has {n_bits} slot bits per row, grid has {session.n_slots}"
        )
    if n_cand == 0:
        raise ValidationError("injection_sets needs at least one candidate row per task")
    sub_count, width = session.split_shape
    if splits is None:
        move = np.zeros((n_tasks, sub_count, width), dtype=bool)
    else:
        move = _checked_bits(splits, "splits", 3)
        if move.shape != (n_tasks, sub_count, width):
            raise ValidationError(
                f"splits shape {move.shape} does not match ({n_tasks}, {sub_count}, {width})"
            )
    for si, count in enumerate(session.element_counts):
        if count < width and move[:, si, count:].any():
            raise ValidationError(f"splits sets bits past the {count} elements of substation {si}")
    if disconnections is None:
        outages = np.empty((n_tasks, 0), dtype=np.int64)
    else:
        outages = np.ascontiguousarray(disconnections)
        if outages.dtype.kind not in "iu":
            raise ValidationError(
                f"disconnections must be integer branch indices, got {outages.dtype}"
            )
        if outages.ndim != 2 or outages.shape[0] != n_tasks:
            raise ValidationError(
                f"disconnections shape {outages.shape} does not match ({n_tasks}, D)"
            )
        outages = outages.astype(np.int64, copy=False)
        if outages.size and (outages.min() < -1 or outages.max() >= session.n_branches):
            raise ValidationError(
                f"disconnection indices must be -1 or in [0, {session.n_branches})"
            )
    if outages.shape[1] > 1:
        srt = np.sort(outages, axis=1)
        if ((srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)).any():
            raise ValidationError("duplicate branch in disconnections")
    return move, outages, inj


def solve_batch(
    session: SolverSession,
    splits: Optional[Any],
    disconnections: Optional[Any],
    injection_sets: Any,
) -> dict[str, Any]:
    """Solve one batch against an open session (`session.py:116-195`)."""
    move, outages, inj = validate_arrays(session, splits, disconnections, injection_sets)
    n_tasks = inj.shape[0]
    if n_tasks == 0:
        return {
            "metrics": np.zeros(0),
            "best_injection": np.zeros(0, dtype=np.int64),
            "feasible": np.zeros(0, dtype=bool),
            "reports": [],
        }
    out = session.engine.solve(move.view(np.uint8), outages, inj.view(np.uint8))
    return {
        "metrics": out.metric,
        "best_injection": out.best,
        "feasible": out.feasible,
        # a real list of dicts, as the reference returns (session.py:182-195); the lazy
        # per-task view is BatchOutput.reports() through solve_batch_output
        "reports": list(out.reports()),
    }


def solve_batch_output(session: SolverSession, splits, disconnections, injection_sets):
    """Same as :func:`solve_batch` but returns the engine's array-first
    :class:`~paper_2501_17529_b200.engine.BatchOutput` (loadflow count, stage
    timings, report entries as indices) instead of the reference-shaped dict."""
    move, outages, inj = validate_arrays(session, splits, disconnections, injection_sets)
    return session.engine.solve(move.view(np.uint8), outages, inj.view(np.uint8))
