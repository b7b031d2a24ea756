"""GPU parity at BASELINE.json's larger sizes and in the reference's other two evaluation
modes, against documents the reference itself produced (tests/golden/make_golden.py
--large, manifest_large.json):

  fixture_b_sym / case300_of   mode="symmetric" / "output_first" (solver.py:777-842)
  g1k_t128                     configs[2] shape (T=128: the 16x128 TOP tile and k_pairs)
  g3k_r12                      configs[3] multi-split, rank k+d = 12 (k_scale_tc<2,2>)
  g10k_t1 / _t64 / _t1024      configs[4] T sweep end points

Contract (same as test_gpu_parity.py): feasibility, reasons and islanded sets exact;
metric within 1e-9 (relative to max(1, metric)); best_injection identical unless the two
candidates tie within FP64 noise (checked with the oracle on exactly those two); report
entries identical up to permutations among loadings tied within 1e-9.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import golden_path, load_case
from oracle import port
from test_gpu_parity import GAP64, _same_entries

pytestmark = pytest.mark.gpu

with open(golden_path("manifest_large.json")) as _fh:
    LARGE = json.load(_fh)["cases"]
with open(golden_path("manifest_edges.json")) as _fh:
    LARGE += json.load(_fh)["cases"]  # edge cases: ragged / 8 outages / duplicates / T=1 / top-k 32


def _grid_source(case):
    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.io import grid_from_dict

    if case.get("synth"):
        doc = synth.make_grid_doc(case["synth"], seed=0)
        sha = hashlib.sha256(json.dumps(doc, sort_keys=True).encode()).hexdigest()
        assert sha == case["grid_sha256"], "synthetic grid generator drifted from the golden run"
        return grid_from_dict(doc)
    return golden_path("grids", case["grid"])


@pytest.fixture(scope="module")
def sessions():
    from paper_2501_17529_b200.session import session_open
    from paper_2501_17529_b200.solver import SolveConfig

    cache = {}

    def get(case):
        key = (case.get("synth") or case["grid"], json.dumps(case["config"], sort_keys=True))
        if key not in cache:
            cache[key] = session_open(_grid_source(case), SolveConfig(**case["config"]))
        return cache[key]

    return get


def _fp64_tie(sess, arr, b, t1, t2):
    """FP64 metrics of candidates t1, t2 of task b by the oracle (only those two rows)."""
    canon = port.decode_arrays(sess.grid, arr["splits"][b:b + 1], arr["disconnections"][b:b + 1],
                               arr["injection_sets"][b:b + 1, [t1, t2]])[0]
    m = port.evaluate(sess.grid, sess.base, canon, sess.config)[0]
    return float(m[0]), float(m[1])


@pytest.mark.parametrize("case", LARGE, ids=[c["name"] for c in LARGE])
def test_large_matches_reference_documents(case, sessions, record_property):
    from paper_2501_17529_b200.session import solve_batch

    sess = sessions(case)
    arr, ref_docs = load_case(case["name"])
    out = solve_batch(sess, arr["splits"], arr["disconnections"], arr["injection_sets"])
    assert isinstance(out["reports"], list)
    assert np.array_equal(out["feasible"], arr["feasible"])
    same = ties = 0
    for b, doc in enumerate(ref_docs):
        mine = out["reports"][b]
        assert mine["feasible"] == doc["feasible"]
        if not doc["feasible"]:
            assert mine == doc, (b, mine, doc)
            continue
        assert mine.get("diagnostics") == doc.get("diagnostics"), b
        scale = max(1.0, abs(doc["metric"]))
        assert abs(mine["metric"] - doc["metric"]) <= 1e-9 * scale, (b, mine["metric"], doc["metric"])
        if mine["best_injection"] == doc["best_injection"]:
            same += 1
            _same_entries(mine["n0_worst"], doc["n0_worst"], ("n0", b))
            _same_entries(mine["n1_worst"], doc["n1_worst"], ("n1", b))
        else:
            ma, mb = _fp64_tie(sess, arr, b, mine["best_injection"], doc["best_injection"])
            assert abs(ma - mb) <= GAP64 * scale, (b, mine["best_injection"], doc["best_injection"], ma, mb)
            ties += 1
    # every disagreement is an FP64-noise tie (asserted above); the agreement rate is recorded
    n_feas = int(arr["feasible"].sum())
    record_property("winner_agreement", f"{same}/{n_feas} ({ties} FP64 ties)")
    print(f"{case['name']}: best_injection identical on {same}/{n_feas} feasible tasks, {ties} FP64 ties")


@pytest.mark.parametrize("name", ["fixture_b_sym", "case300_of"])
def test_modes_are_bit_identical(name, sessions):
    """metric_first (screened), symmetric and output_first (every pair evaluated) give
    bit-identical results through the engine, as the reference's three modes do."""
    from dataclasses import replace

    from paper_2501_17529_b200.engine import Engine

    case = next(c for c in LARGE if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    args = (arr["splits"], arr["disconnections"], arr["injection_sets"])
    outs = {}
    for mode in ("metric_first", "symmetric", "output_first"):
        eng = Engine(sess.grid, sess.base, replace(sess.config, mode=mode))
        assert eng.screen == (mode == "metric_first")
        outs[mode] = eng.solve(*args)
    ref = outs["metric_first"]
    for mode in ("symmetric", "output_first"):
        o = outs[mode]
        assert np.array_equal(o.best, ref.best)
        assert np.array_equal(o.metric, ref.metric, equal_nan=True)
        assert o.reports() == ref.reports()
        assert o.loadflows == ref.loadflows
        assert o.n1_pairs >= ref.n1_pairs


def test_candidate_case_flows_library_entry_point(sessions):
    """batchdc.candidate_case_flows (solver.py:919-958) through the device probe: the same
    CaseFlows fields, flows at the reference fixtures' 1e-9 tolerance."""
    from conftest import load_manifest
    from paper_2501_17529_b200.solver import CaseFlows, SplitAction, TopologyTask, candidate_case_flows

    case = next(c for c in load_manifest() if c["name"] == "fixture_b")
    sess = sessions(case)
    arr, _ = load_case("fixture_b")
    grid = sess.grid
    checked = 0
    for b in range(arr["splits"].shape[0]):
        splits = tuple(
            SplitAction(si, tuple(bool(x) for x in arr["splits"][b, si, : len(s.branch_elements)]))
            for si, s in enumerate(grid.substations) if arr["splits"][b, si].any()
        )
        d = tuple(int(k) for k in arr["disconnections"][b] if k >= 0)
        rows = tuple(tuple(bool(x) for x in r) for r in arr["injection_sets"][b])
        cf = candidate_case_flows(grid, sess.base, TopologyTask(splits, d, rows), sess.config)
        assert isinstance(cf, CaseFlows)
        canon = port.decode_arrays(grid, arr["splits"][b:b + 1], arr["disconnections"][b:b + 1],
                                   arr["injection_sets"][b:b + 1])[0]
        ref = port.case_flows(grid, sess.base, canon, sess.config)
        assert cf.feasible == ref["feasible"]
        if not cf.feasible:
            assert cf.reason == ref["reason"]
            continue
        assert np.array_equal(cf.row_branches, sess.base.row_branches)
        np.testing.assert_allclose(cf.n0, ref["n0"], atol=1e-9)
        assert len(cf.n1) == len(ref["n1"])
        for a, e in zip(cf.n1, ref["n1"]):
            assert (a is None) == (e is None)
            if a is not None:
                np.testing.assert_allclose(a, e, atol=1e-9)
        if f"n0_{b}" in arr:
            np.testing.assert_allclose(cf.n0, arr[f"n0_{b}"], atol=1e-9)
        checked += 1
    assert checked > 10


def test_concurrent_batches_equal_serial(sessions):
    """Concurrent solve_batch calls on one session equal the serial results
    (bindings/tests/test_bindings.py:191-203): four threads, each its own batch."""
    from concurrent.futures import ThreadPoolExecutor

    from conftest import load_manifest
    from paper_2501_17529_b200.session import solve_batch

    case = next(c for c in load_manifest() if c["name"] == "g118")
    sess = sessions(case)
    arr, _ = load_case("g118")
    arr = {k: np.asarray(arr[k]) for k in ("splits", "disconnections", "injection_sets")}  # npz reads are not thread-safe
    n = arr["splits"].shape[0]
    parts = [slice(i * n // 4, (i + 1) * n // 4) for i in range(4)]

    def run(sl):
        return solve_batch(sess, arr["splits"][sl], arr["disconnections"][sl], arr["injection_sets"][sl])

    serial = [run(sl) for sl in parts]
    for _ in range(3):
        with ThreadPoolExecutor(4) as pool:
            conc = list(pool.map(run, parts))
        for a, c in zip(serial, conc):
            assert np.array_equal(a["best_injection"], c["best_injection"])
            assert np.array_equal(a["metrics"], c["metrics"], equal_nan=True)
            assert a["reports"] == c["reports"]


def test_two_sessions_in_one_process(sessions):
    """A second session (other grid, other kernels' shared-memory opt-ins) in the same
    process: each keeps giving its own results (launcher opt-ins are per device)."""
    from conftest import load_manifest
    from paper_2501_17529_b200.session import solve_batch

    cases = {c["name"]: c for c in load_manifest()}
    a = sessions(cases["g118"])
    b = sessions(cases["fixture_b"])
    arr_a, docs_a = load_case("g118")
    arr_b, docs_b = load_case("fixture_b")
    for _ in range(2):
        oa = solve_batch(a, arr_a["splits"], arr_a["disconnections"], arr_a["injection_sets"])
        ob = solve_batch(b, arr_b["splits"], arr_b["disconnections"], arr_b["injection_sets"])
        assert [d["feasible"] for d in oa["reports"]] == [d["feasible"] for d in docs_a]
        assert [d["feasible"] for d in ob["reports"]] == [d["feasible"] for d in docs_b]
        for m, d in zip(oa["metrics"], docs_a):
            if d["feasible"]:
                assert abs(m - d["metric"]) <= 1e-9 * max(1.0, abs(d["metric"]))


def test_multi_device_sessions():
    """One session per visible device in one process (skipped with fewer than two)."""
    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.engine import device_count
    from paper_2501_17529_b200.session import session_open, solve_batch_output

    n = device_count()
    if n < 2:
        pytest.skip("needs two CUDA devices")
    grid = synth.make_grid("g118", seed=0)
    splits, discos, inj = synth.random_task_arrays(grid, 64, 16, 3, seed=3)
    outs = [solve_batch_output(session_open(grid, device=d), splits, discos, inj) for d in range(2)]
    assert np.array_equal(outs[0].best, outs[1].best)
    assert np.array_equal(outs[0].metric, outs[1].metric, equal_nan=True)


def test_folded_endpoint_disconnection_raises():
    """Disconnecting a branch whose endpoint column is folded into the static column is a
    batch-level ValidationError in the reference (compute_modf, factors.py:391-392;
    lodf_column :345-346), raised before any device work -- and never an out-of-bounds
    column read on the device."""
    from dataclasses import replace

    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.errors import ValidationError
    from paper_2501_17529_b200.session import session_open, solve_batch

    grid = synth.make_grid("g1k", seed=0)
    folded = np.flatnonzero(synth.folded_branches(grid))
    assert len(folded)
    sess = session_open(grid)
    splits, discos, inj = synth.random_task_arrays(grid, 3, 4, 2, seed=9, n_disconnections=1)
    discos = discos.copy()
    discos[1, 0] = folded[0]
    with pytest.raises(ValidationError, match="outage branch endpoint column folded"):
        solve_batch(sess, splits, discos, inj)
    seq = session_open(grid, replace(sess.config, multi_outage_method="sequential"))
    with pytest.raises(ValidationError, match="endpoint column folded, cannot outage"):
        solve_batch(seq, splits, discos, inj)


def test_empty_batch():
    """B = 0 returns empty arrays and an empty report list, as the reference's session does."""
    from paper_2501_17529_b200.session import session_open, solve_batch

    sess = session_open(golden_path("grids", "fixture_b.json"))
    S, E = sess.split_shape
    out = solve_batch(sess, np.zeros((0, S, E), bool), np.zeros((0, 0), np.int64),
                      np.zeros((0, 3, sess.n_slots), bool))
    assert out["metrics"].shape == (0,) and out["metrics"].dtype == np.float64
    assert out["best_injection"].shape == (0,) and out["best_injection"].dtype == np.int64
    assert out["feasible"].shape == (0,) and out["feasible"].dtype == bool
    assert out["reports"] == []
