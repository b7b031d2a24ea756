#!/usr/bin/env python3
"""Generate the golden vectors by running the REFERENCE implementation itself.

Run in the build container only (it imports `/root/reference/pkg`, which does
not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed) under tests/golden/:
  grids/<name>.json            grid documents (reference fixtures a/b/case300
                               copied verbatim; synthetic g14/g118 from
                               paper_2501_17529_b200.synth)
  <case>.npz                   task arrays (splits, disconnections, injection_sets)
                               + reference metrics/best/feasible (+ flows for
                               the small fixtures, + refactorisation-oracle
                               metrics per candidate)
  <case>.reports.json          the reference's per-task result documents
                               (`batchdc_session.solve_batch(...)["reports"]`)
  manifest.json                case list with the SolveConfig used

Tasks are drawn with the reference's own generator (`batchdc.bench.random_tasks`)
and encoded into the session array layout the way the reference's binding
tests do (`pkg/bindings/tests/test_bindings.py:40-56`).
"""

from __future__ import annotations

import json
import os
import shutil
import sys
from dataclasses import asdict

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), os.path.join(REF, "bindings", "src"), REPO]

import batchdc  # noqa: E402
from batchdc import SolveConfig, SplitAction, TopologyTask, candidate_case_flows  # noqa: E402
from batchdc import oracle as ref_oracle  # noqa: E402
from batchdc.bench import random_tasks  # noqa: E402
from batchdc_session import session_open, solve_batch  # noqa: E402

from paper_2501_17529_b200 import synth  # noqa: E402

GRIDS = os.path.join(HERE, "grids")


def encode(session, tasks):
    n = len(tasks)
    S, E = session.split_shape
    splits = np.zeros((n, S, E), dtype=bool)
    d_max = max((len(t.disconnections) for t in tasks), default=0)
    outages = np.full((n, d_max), -1, dtype=np.int64)
    T = len(tasks[0].injection_sets)
    inj = np.zeros((n, T, session.n_slots), dtype=bool)
    for i, task in enumerate(tasks):
        for a in task.splits:
            splits[i, a.substation, : len(a.assignment)] = a.assignment
        for j, k in enumerate(task.disconnections):
            outages[i, j] = k
        rows = [list(r) if len(r) else [False] * session.n_slots for r in task.injection_sets]
        inj[i] = np.array(rows, dtype=bool).reshape(T, session.n_slots)
    return splits, outages, inj


def special_tasks(grid, T):
    """Hand-picked edge cases: identity, degenerate split, all-True, bridge outage."""
    K = len(grid.injection_slots)
    rows = tuple(tuple(bool((t >> s) & 1) for s in range(K)) for t in range(T))
    out = [TopologyTask(injection_sets=rows)]
    for si, sub in enumerate(grid.substations[:3]):
        n = len(sub.branch_elements)
        out.append(TopologyTask(splits=(SplitAction(si, (True,) * n),), injection_sets=rows))
        out.append(
            TopologyTask(
                splits=(SplitAction(si, tuple(i % 2 == 0 for i in range(n))),), injection_sets=rows
            )
        )
    return out


def run_case(name, grid_file, cfg, tasks_fn, flows=False, oracle_metrics=False):
    grid = batchdc.load_grid(os.path.join(GRIDS, grid_file))
    base = batchdc.prepare_base_ptdf(grid)
    session = session_open(grid, cfg)
    tasks = tasks_fn(grid, base)
    splits, outages, inj = encode(session, tasks)
    out = solve_batch(session, splits, outages, inj)
    arrays = dict(
        splits=splits,
        disconnections=outages,
        injection_sets=inj,
        metrics=out["metrics"],
        best_injection=out["best_injection"],
        feasible=out["feasible"],
    )
    if flows or oracle_metrics:
        om = np.full((len(tasks), inj.shape[1]), np.nan)
        for i, task in enumerate(tasks):
            if not out["feasible"][i]:
                continue
            if flows:
                cf = candidate_case_flows(grid, base, task, cfg)
                arrays[f"n0_{i}"] = cf.n0
                n1 = np.full((len(cf.n1),) + cf.n0.shape, np.nan)
                for c, fl in enumerate(cf.n1):
                    if fl is not None:
                        n1[c] = fl
                arrays[f"n1_{i}"] = n1
            if oracle_metrics:
                setup = ref_oracle.materialize(grid, task)
                res = ref_oracle.oracle_solve(grid, setup)
                om[i] = ref_oracle.oracle_metric(grid, res, cfg.islanding_penalty)
        arrays["oracle_metric"] = om
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    with open(os.path.join(HERE, f"{name}.reports.json"), "w") as fh:
        json.dump(out["reports"], fh)
    print(f"{name}: {len(tasks)} tasks, feasible {int(out['feasible'].sum())}")
    return {"name": name, "grid": grid_file, "config": asdict(cfg)}


def main():
    os.makedirs(GRIDS, exist_ok=True)
    for f in ("fixture_a.json", "fixture_b.json", "case300.json"):
        shutil.copy(os.path.join(REF, "tests", "data", f), os.path.join(GRIDS, f))
    for spec in ("g14", "g118"):
        with open(os.path.join(GRIDS, f"{spec}.json"), "w") as fh:
            json.dump(synth.make_grid_doc(spec, seed=0), fh)

    def rt(n, ti, k, seed, d=0):
        return lambda g, b: random_tasks(g, b, n, ti_size=ti, n_splits=k, seed=seed, n_disconnections=d)

    def combo(*fns):
        return lambda g, b: [t for fn in fns for t in fn(g, b)]

    def spec(ti):
        return lambda g, b: special_tasks(g, ti)

    cases = []
    cases.append(run_case("fixture_a", "fixture_a.json", SolveConfig(),
                          combo(spec(4), rt(24, 4, 2, 78), rt(8, 4, 1, 79, 1)), flows=True, oracle_metrics=True))
    cases.append(run_case("fixture_a_error", "fixture_a.json", SolveConfig(islanding_policy="error"),
                          combo(spec(4), rt(8, 4, 2, 80))))
    cases.append(run_case("fixture_b", "fixture_b.json", SolveConfig(),
                          combo(spec(8), rt(40, 8, 2, 909), rt(24, 8, 2, 910, 1), rt(8, 8, 3, 911, 2)),
                          flows=True, oracle_metrics=True))
    cases.append(run_case("fixture_b_topk", "fixture_b.json", SolveConfig(topk_per_case=3, topk_global=7),
                          combo(rt(16, 6, 2, 77), rt(8, 6, 1, 76, 1))))
    cases.append(run_case("fixture_b_seq", "fixture_b.json", SolveConfig(multi_outage_method="sequential"),
                          combo(rt(16, 4, 1, 75, 2), rt(8, 4, 2, 74, 3))))
    cases.append(run_case("case300", "case300.json", SolveConfig(),
                          combo(spec(16), rt(16, 16, 3, 31), rt(6, 16, 2, 32, 1)), oracle_metrics=True))
    cases.append(run_case("g14", "g14.json", SolveConfig(),
                          combo(spec(16), rt(48, 16, 2, 14), rt(48, 16, 1, 15, 1)), oracle_metrics=True))
    cases.append(run_case("g118", "g118.json", SolveConfig(),
                          combo(spec(64), rt(12, 64, 3, 118), rt(4, 64, 3, 119, 2))))
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"reference": "/root/reference/pkg (batchdc 0.1.0)", "cases": cases}, fh, indent=1)


def grid_sha(doc) -> str:
    import hashlib

    return hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()


def main_large():
    """Round-2 cases (manifest_large.json): the other two evaluation modes on the
    reference fixtures, and reference-run documents at BASELINE.json's larger grid sizes,
    chosen so that every kernel variant the benchmarked configs launch is covered:
      g1k_t128    configs[2] shape: G1k, T=128 (the 16x128 TOP tile / k_pairs variant)
      g3k_r12     configs[3] multi-split: k=8 splits + 4 disconnections (rank 12: the
                  two-K-block tensor-core screening kernel, k_scale_tc<2,2>)
      g10k_t*     configs[4] sweep end points T = 1, 64, 1024
    The synthetic grids are not stored: the test regenerates them from
    paper_2501_17529_b200.synth (seeded) and checks the document's sha256."""
    import tempfile

    def rt(n, ti, k, seed, d=0):
        return lambda g, b: random_tasks(g, b, n, ti_size=ti, n_splits=k, seed=seed, n_disconnections=d)

    def combo(*fns):
        return lambda g, b: [t for fn in fns for t in fn(g, b)]

    cases = []
    cases.append(run_case("fixture_b_sym", "fixture_b.json", SolveConfig(mode="symmetric"),
                          combo(rt(24, 8, 2, 921), rt(8, 8, 2, 922, 1))))
    cases.append(run_case("case300_of", "case300.json", SolveConfig(mode="output_first"),
                          combo(rt(8, 16, 3, 33), rt(4, 16, 2, 34, 1))))
    tmp = tempfile.mkdtemp()
    for name, spec_name, fn in (
        ("g1k_t128", "g1k", combo(rt(32, 128, 3, 1001), rt(8, 128, 3, 1002, 1))),
        ("g3k_r12", "g3k", rt(6, 32, 8, 3001, 4)),
        ("g10k_t1", "g10k", rt(3, 1, 3, 10001)),
        ("g10k_t64", "g10k", rt(3, 64, 3, 10002)),
        ("g10k_t1024", "g10k", rt(2, 1024, 3, 10003)),
    ):
        doc = synth.make_grid_doc(spec_name, seed=0)
        path = os.path.join(tmp, f"{spec_name}.json")
        with open(path, "w") as fh:
            json.dump(doc, fh)
        import time

        t0 = time.time()
        c = run_case(name, path, SolveConfig(), fn)
        c["grid"] = None
        c["synth"] = spec_name
        c["grid_sha256"] = grid_sha(doc)
        c["reference_seconds"] = round(time.time() - t0, 1)
        cases.append(c)
    with open(os.path.join(HERE, "manifest_large.json"), "w") as fh:
        json.dump({"reference": "/root/reference/pkg (batchdc 0.1.0)", "cases": cases}, fh, indent=1)


if __name__ == "__main__":
    if "--large" in sys.argv:
        main_large()
    else:
        main()
