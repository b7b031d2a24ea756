"""Pin the CPU oracle against golden vectors produced by the reference itself.

The golden files (tests/golden/, written by make_golden.py from
/root/reference) hold the reference's per-task result documents, metrics and
winners, the engine flows of `candidate_case_flows` for the small fixtures,
and the refactorisation oracle's per-candidate metrics.  The numpy port must
reproduce the documents exactly (same float bits), and the restated
refactorisation oracle must match the reference's oracle metrics.
"""

import json

import numpy as np
import pytest

from conftest import golden_path, load_case, load_manifest
from oracle import port, refact
from paper_2501_17529_b200 import io as bio
from paper_2501_17529_b200.ptdf import prepare_base_ptdf
from paper_2501_17529_b200.solver import SolveConfig

CASES = load_manifest()
with open(golden_path("manifest_edges.json")) as _fh:
    EDGES = json.load(_fh)["cases"]  # reference-run edge cases (make_edge_golden.py)


def _grid(case):
    return bio.load_grid(golden_path("grids", case["grid"]))


@pytest.mark.parametrize("case", CASES + EDGES, ids=[c["name"] for c in CASES + EDGES])
def test_port_reproduces_reference_documents(case):
    grid = _grid(case)
    base = prepare_base_ptdf(grid)
    cfg = SolveConfig(**case["config"])
    arr, reports = load_case(case["name"])
    res = port.solve_arrays(grid, base, arr["splits"], arr["disconnections"], arr["injection_sets"], cfg)
    assert len(res) == len(reports)
    for i, (r, doc) in enumerate(zip(res, reports)):
        mine = r.to_dict()
        # documents match key for key; floats to 1e-12 (base PTDF is refactorised here)
        assert mine.keys() == doc.keys(), (i, mine, doc)
        assert mine["feasible"] == doc["feasible"]
        assert mine["best_injection"] == doc["best_injection"], (i, mine, doc)
        assert mine.get("diagnostics") == doc.get("diagnostics"), i
        if doc["metric"] is None:
            assert mine["metric"] is None
            continue
        assert abs(mine["metric"] - doc["metric"]) <= 1e-12 * max(1.0, abs(doc["metric"]))
        for key in ("n0_worst", "n1_worst"):
            assert len(mine[key]) == len(doc[key])
            for a, b in zip(mine[key], doc[key]):
                assert a.get("case") == b.get("case") and a["branch"] == b["branch"], (i, key, a, b)
                assert abs(a["flow_mw"] - b["flow_mw"]) <= 1e-9
                assert abs(a["rel_load"] - b["rel_load"]) <= 1e-12


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b"])
def test_port_flows_match_reference_engine_flows(name):
    case = next(c for c in CASES if c["name"] == name)
    grid = _grid(case)
    base = prepare_base_ptdf(grid)
    cfg = SolveConfig(**case["config"])
    arr, _ = load_case(name)
    canons = port.decode_arrays(grid, arr["splits"], arr["disconnections"], arr["injection_sets"])
    checked = 0
    for i, c in enumerate(canons):
        if f"n0_{i}" not in arr:
            continue
        cf = port.case_flows(grid, base, c, cfg)
        assert cf["feasible"]
        np.testing.assert_allclose(cf["n0"], arr[f"n0_{i}"], atol=1e-9)
        ref_n1 = arr[f"n1_{i}"]
        for ci, fl in enumerate(cf["n1"]):
            if fl is None:
                assert np.isnan(ref_n1[ci]).all()
            else:
                np.testing.assert_allclose(fl, ref_n1[ci], atol=1e-9)
        checked += 1
    assert checked > 10


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b", "case300", "g14"])
def test_refactorisation_oracle_matches_reference_oracle(name):
    case = next(c for c in CASES if c["name"] == name)
    grid = _grid(case)
    cfg = SolveConfig(**case["config"])
    arr, _ = load_case(name)
    canons = port.decode_arrays(grid, arr["splits"], arr["disconnections"], arr["injection_sets"])
    om = arr["oracle_metric"]
    n = 0
    for i, c in enumerate(canons):
        if np.isnan(om[i]).all():
            continue
        res = refact.solve(grid, c)
        mine = refact.metric(grid, res, cfg.islanding_penalty)
        np.testing.assert_allclose(mine, om[i], rtol=1e-9, atol=1e-9)
        n += 1
        if n >= 8:
            break
    assert n > 0


def test_golden_known_answers_triangle():
    """Reference known-answer vectors (`tests/test_factors.py:81-134`, `test_oracle.py:24-63`)."""
    from paper_2501_17529_b200.grid import Branch, ContingencyCase, Injection, build_grid
    from paper_2501_17529_b200.ptdf import compute_ptdf

    grid = build_grid(
        ["n0", "n1", "n2"],
        [
            Branch("e01", 0, 1, 10.0, 80.0),
            Branch("e12", 1, 2, 10.0, 80.0),
            Branch("e02", 0, 2, 10.0, 80.0),
        ],
        [Injection("load2", 2, -90.0)],
        slack=0,
        contingencies=[
            ContingencyCase("out_e02", "single_branch", (2,)),
            ContingencyCase("loss_load", "injection", (), 0),
        ],
    )
    p = compute_ptdf(grid)
    np.testing.assert_allclose(
        p.values, [[0, -2 / 3, -1 / 3], [0, 1 / 3, -1 / 3], [0, -1 / 3, -2 / 3]], atol=1e-12
    )
    canon = port.canonical(grid, [], (), [[]])
    res = refact.solve(grid, canon)
    np.testing.assert_allclose(res.n0[:, 0], [30, 30, 60], atol=1e-9)
    np.testing.assert_allclose(res.n1[0][:, 0], [90, 90, 0], atol=1e-9)
    np.testing.assert_allclose(res.n1[1][:, 0], [0, 0, 0], atol=1e-12)
    assert refact.metric(grid, res, 10.0)[0] == pytest.approx(90 / 80, abs=1e-12)
    # the port's LODF path: self factor exactly -1, post-outage flow exactly 0
    cf = port.case_flows(grid, prepare_base_ptdf(grid, fold_static=False), canon, SolveConfig())
    np.testing.assert_allclose(cf["n1"][0][:, 0], [90, 90, 0], atol=1e-9)
    assert cf["n1"][0][2, 0] == 0.0
    r = port.solve_one(grid, prepare_base_ptdf(grid), canon, SolveConfig())
    assert r.metric == pytest.approx(90 / 80, abs=1e-12) and r.best_injection == 0
