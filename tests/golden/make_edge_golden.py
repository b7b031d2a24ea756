#!/usr/bin/env python3
"""Edge-case golden documents produced by the REFERENCE itself (batchdc_session).

Run in the build container only (imports /root/reference/pkg):

    python tests/golden/make_edge_golden.py

Cases (tests/golden/edges_<name>.npz + .reports.json, listed in manifest_edges.json):
  ragged       disconnection rows with -1 padding anywhere, 0..4 outages, mixed with splits
  outages8     eight simultaneous disconnections (the max_simultaneous_outages cap), MODF
  duplicates   repeated and all-False / all-True candidate rows (first-index winner)
  t1           a single candidate per task
  topk32       topk_per_case = topk_global = 32 (the engine's KMAX)
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "bindings", "src"), REPO]

import batchdc  # noqa: E402
from batchdc import SolveConfig  # noqa: E402
from batchdc_session import session_open, solve_batch  # noqa: E402

GRIDS = os.path.join(HERE, "grids")


def draw(session, grid, n, T, rng, max_d, ragged=True, d_exact=None):
    S, E = session.split_shape
    K = session.n_slots
    eligible = [i for i, s in enumerate(grid.substations) if len(s.branch_elements) >= 2]
    splits = np.zeros((n, S, E), dtype=bool)
    D = max_d + (2 if ragged else 0)
    outages = np.full((n, D), -1, dtype=np.int64)
    # outage candidates: retained branches whose endpoints are not folded (others raise a
    # batch-level ValidationError in the reference)
    base = batchdc.prepare_base_ptdf(grid)
    ok = [k for k in range(grid.n_branches)
          if base.branch_rows[k] >= 0 and base.from_cols[base.branch_rows[k]] >= 0
          and base.to_cols[base.branch_rows[k]] >= 0]
    for i in range(n):
        for si in rng.choice(eligible, size=int(rng.integers(0, min(3, len(eligible)) + 1)), replace=False):
            n_el = len(grid.substations[si].branch_elements)
            bits = rng.integers(0, 2, size=n_el).astype(bool)
            if not bits.any():
                bits[0] = True
            splits[i, si, :n_el] = bits
        d = d_exact if d_exact is not None else int(rng.integers(0, max_d + 1))
        picks = rng.choice(ok, size=d, replace=False)
        slots = np.sort(rng.choice(D, size=d, replace=False)) if ragged else np.arange(d)
        outages[i, slots] = picks
    inj = rng.integers(0, 2, size=(n, T, K)).astype(bool)
    return splits, outages, inj


def run(name, grid_file, cfg, arrays_fn, manifest):
    grid = batchdc.load_grid(os.path.join(GRIDS, grid_file))
    session = session_open(grid, cfg)
    splits, outages, inj = arrays_fn(session, grid)
    out = solve_batch(session, splits, outages, inj)
    np.savez_compressed(os.path.join(HERE, f"edges_{name}.npz"), splits=splits, disconnections=outages,
                        injection_sets=inj, metrics=out["metrics"], best_injection=out["best_injection"],
                        feasible=out["feasible"])
    with open(os.path.join(HERE, f"edges_{name}.reports.json"), "w") as fh:
        json.dump(out["reports"], fh)
    manifest.append({"name": f"edges_{name}", "grid": grid_file, "config": asdict(cfg)})
    print(name, len(splits), "tasks, feasible", int(out["feasible"].sum()))


def main():
    manifest = []
    cfg = SolveConfig()

    def ragged(session, grid):
        return draw(session, grid, 40, 16, np.random.default_rng(1), 4)

    def outages8(session, grid):
        return draw(session, grid, 24, 8, np.random.default_rng(2), 8, ragged=False, d_exact=8)

    def duplicates(session, grid):
        s, d, inj = draw(session, grid, 24, 8, np.random.default_rng(3), 1)
        inj[:, 1] = inj[:, 0]
        inj[:, 3] = inj[:, 0]
        inj[:, 4] = False
        inj[:, 5] = True
        inj[:, 6] = inj[:, 4]
        return s, d, inj

    def t1(session, grid):
        return draw(session, grid, 32, 1, np.random.default_rng(4), 2)

    run("ragged", "case300.json", cfg, ragged, manifest)
    run("outages8", "case300.json", cfg, outages8, manifest)
    run("duplicates", "fixture_b.json", cfg, duplicates, manifest)
    run("t1", "case300.json", cfg, t1, manifest)
    run("topk32", "case300.json", SolveConfig(topk_per_case=32, topk_global=32), ragged, manifest)
    with open(os.path.join(HERE, "manifest_edges.json"), "w") as fh:
        json.dump({"cases": manifest}, fh, indent=1)


if __name__ == "__main__":
    main()
