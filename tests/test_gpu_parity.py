"""GPU parity: the CUDA engine (through the C ABI) against the reference's golden
documents and the CPU oracle, on the same seeded inputs.

Tolerance contract:
  * feasibility, infeasibility reasons and islanded case sets: exact;
  * metric: within 1e-9 of the reference (FP64: every candidate in the FP32
    near-tie band of the minimum is re-scored in FP64, k_rescore);
  * best_injection: identical whenever the reference's best-vs-runner-up gap
    exceeds GAP64 = 1e-12 x max(1, metric), i.e. the FP64 noise between two
    implementations; otherwise the engine's pick must be metric-minimal within
    that noise (the reference's own rule, test_solver.py:244-246, at FP64);
  * report: identical (case, branch) entries and order, flows/loadings within
    1e-9, except permutations among entries whose loadings differ by < 1e-9;
  * per-candidate FP32 screening metrics within TAU of the FP64 oracle.
"""

import json

import numpy as np
import pytest

from conftest import golden_path, load_case, load_manifest
from oracle import port

pytestmark = pytest.mark.gpu

TAU = 1e-5
GAP64 = 1e-12  # FP64 noise between the engine's low-rank flows and the reference's
CASES = load_manifest()


@pytest.fixture(scope="module")
def sessions():
    from paper_2501_17529_b200.session import session_open
    from paper_2501_17529_b200.solver import SolveConfig

    cache = {}

    def get(case):
        key = case["name"]
        if key not in cache:
            cache[key] = session_open(golden_path("grids", case["grid"]), SolveConfig(**case["config"]))
        return cache[key]

    return get


def _same_entries(mine, ref, key, tie=1e-9):
    """Same entries in the same order, up to permutations among numerically tied
    loadings (|delta rel| <= tie), including ties straddling the top-k cut."""
    assert len(mine) == len(ref), (key, mine, ref)
    for a, b in zip(mine, ref):
        assert abs(a["rel_load"] - b["rel_load"]) <= tie, (key, a, b)
    ident = lambda e: (e.get("case"), e["branch"])
    ref_by = {ident(e): e for e in ref}
    for a in mine:
        b = ref_by.get(ident(a))
        if b is None:
            assert abs(a["rel_load"] - ref[-1]["rel_load"]) <= tie, (key, a, ref)
            continue
        assert abs(a["rel_load"] - b["rel_load"]) <= tie, (key, a, b)
        assert abs(a["flow_mw"] - b["flow_mw"]) <= 1e-7 * max(1.0, abs(b["flow_mw"])), (key, a, b)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_engine_matches_reference_documents(case, sessions):
    from paper_2501_17529_b200.session import solve_batch

    sess = sessions(case)
    arr, ref_docs = load_case(case["name"])
    out = solve_batch(sess, arr["splits"], arr["disconnections"], arr["injection_sets"])
    canons = port.decode_arrays(sess.grid, arr["splits"], arr["disconnections"], arr["injection_sets"])
    assert np.array_equal(out["feasible"], arr["feasible"])
    n_exact = 0
    for b, doc in enumerate(ref_docs):
        mine = out["reports"][b]
        assert mine["feasible"] == doc["feasible"]
        if not doc["feasible"]:
            assert mine == doc, (b, mine, doc)
            assert np.isnan(out["metrics"][b]) and out["best_injection"][b] == -1
            continue
        assert mine.get("diagnostics") == doc.get("diagnostics"), b
        ev = port.evaluate(sess.grid, sess.base, canons[b], sess.config)
        metrics = ev[0]
        # the FP64 re-score of the near-tie band makes the winner the first FP64 argmin:
        # identical to the reference's whenever the reference's best-vs-runner-up gap is
        # above FP64 noise (distinct-flow candidates), metric-minimal at that noise otherwise
        scale = max(1.0, abs(doc["metric"]))
        order = np.sort(metrics)
        gap = order[1] - order[0] if len(order) > 1 else np.inf
        if gap > GAP64 * scale:
            assert mine["best_injection"] == doc["best_injection"], (b, gap)
        assert metrics[mine["best_injection"]] <= metrics.min() + GAP64 * scale, b
        assert abs(mine["metric"] - doc["metric"]) <= 1e-9 * scale, b
        if mine["best_injection"] == doc["best_injection"]:
            n_exact += 1
            _same_entries(mine["n0_worst"], doc["n0_worst"], ("n0", b))
            _same_entries(mine["n1_worst"], doc["n1_worst"], ("n1", b))
        else:
            _, _, n0e, n1e, _ = port.evaluate(sess.grid, sess.base, canons[b], sess.config, mine["best_injection"])
            _same_entries(mine["n0_worst"], [{"branch": x[0], "flow_mw": x[1], "rel_load": x[2]} for x in n0e], ("n0*", b))
            _same_entries(
                mine["n1_worst"],
                [{"case": x[0], "branch": x[1], "flow_mw": x[2], "rel_load": x[3]} for x in n1e],
                ("n1*", b),
            )
    assert n_exact >= 1 or not arr["feasible"].any()


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b", "case300", "g14", "g118"])
def test_candidate_screening_metrics_within_tolerance(name, sessions):
    case = next(c for c in CASES if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    out = sess.engine.solve(arr["splits"], arr["disconnections"], arr["injection_sets"], want_candidates=True)
    canons = port.decode_arrays(sess.grid, arr["splits"], arr["disconnections"], arr["injection_sets"])
    worst = 0.0
    for b, c in enumerate(canons):
        ev = port.evaluate(sess.grid, sess.base, c, sess.config)
        if ev is None:
            assert not out.feasible[b]
            continue
        mine = out.cand_metric[b].astype(np.float64)
        if ev[4]:
            mine = np.maximum(mine, sess.config.islanding_penalty)
        worst = max(worst, float(np.max(np.abs(mine - ev[0]))))
    assert worst <= TAU, worst


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b"])
def test_device_flows_match_reference_flows(name, sessions):
    """candidate_case_flows parity: every flow vector at 1e-9 (reference fixture tolerance)."""
    case = next(c for c in CASES if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    checked = 0
    for b in range(arr["splits"].shape[0]):
        if f"n0_{b}" not in arr:
            continue
        st, _, n0, n1, ok = sess.engine.probe_flows(arr["splits"][b], arr["disconnections"][b], arr["injection_sets"][b])
        assert st == 0
        np.testing.assert_allclose(n0, arr[f"n0_{b}"], atol=1e-9)
        ref = arr[f"n1_{b}"]
        for ci in range(ref.shape[0]):
            if np.isnan(ref[ci]).all():
                assert not ok[ci]
            else:
                assert ok[ci]
                np.testing.assert_allclose(n1[ci], ref[ci], atol=1e-9)
        checked += 1
    assert checked > 10


def test_exact_zero_outaged_flows_and_self_factor(sessions):
    """Post-outage flow of the outaged branch is exactly 0 (test_acceptance.py:308-349)."""
    case = next(c for c in CASES if c["name"] == "fixture_b")
    sess = sessions(case)
    arr, _ = load_case("fixture_b")
    grid = sess.grid
    for b in range(0, arr["splits"].shape[0], 7):
        st, _, n0, n1, ok = sess.engine.probe_flows(arr["splits"][b], arr["disconnections"][b], arr["injection_sets"][b])
        if st != 0:
            continue
        for ci, c in enumerate(grid.contingencies):
            if c.kind == "injection" or not ok[ci]:
                continue
            for k in c.branches:
                assert np.all(n1[ci][sess.base.branch_rows[k]] == 0.0)
        for k in arr["disconnections"][b]:
            if k >= 0:
                assert np.all(n0[sess.base.branch_rows[k]] == 0.0)


def test_library_solve_batch_matches_session(sessions):
    from paper_2501_17529_b200 import io as bio
    from paper_2501_17529_b200.solver import TopologyTask, SplitAction, solve_batch

    case = next(c for c in CASES if c["name"] == "fixture_b")
    sess = sessions(case)
    arr, ref_docs = load_case("fixture_b")
    grid = sess.grid
    tasks = []
    for b in range(20):
        splits = tuple(
            SplitAction(si, tuple(bool(x) for x in arr["splits"][b, si, : len(s.branch_elements)]))
            for si, s in enumerate(grid.substations)
            if arr["splits"][b, si].any()
        )
        d = tuple(int(k) for k in arr["disconnections"][b] if k >= 0)
        rows = tuple(tuple(bool(x) for x in r) for r in arr["injection_sets"][b][: 1 + b % 4])
        tasks.append(TopologyTask(splits, d, rows))
    res = solve_batch(grid, sess.base, tasks, sess.config)
    for b, (t, r) in enumerate(zip(tasks, res)):
        doc = bio.result_to_dict(r)
        c = port.canonical(grid, [(s.substation, s.assignment) for s in t.splits], t.disconnections, t.injection_sets)
        pr = port.solve_one(grid, sess.base, c, sess.config)
        assert doc["feasible"] == pr.feasible
        if pr.feasible:
            assert abs(doc["metric"] - pr.metric) <= TAU
            assert doc["best_injection"] < len(t.injection_sets)


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b", "case300", "g14", "g118"])
def test_dominance_screen_is_exact(name, sessions):
    """The device dominance screen (solver.py:798-822) never changes a result."""
    case = next(c for c in CASES if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    eng = sess.engine
    outs = {}
    for flag in (True, False):
        eng.screen = flag
        outs[flag] = eng.solve(arr["splits"], arr["disconnections"], arr["injection_sets"], want_candidates=True)
    eng.screen = True
    on, off = outs[True], outs[False]
    assert np.array_equal(on.best, off.best)
    assert np.array_equal(on.metric, off.metric, equal_nan=True)
    assert on.reports() == off.reports()
    pen = sess.config.islanding_penalty
    for b in range(len(on.best)):
        if not on.feasible[b]:
            continue
        a, c = on.cand_metric[b], off.cand_metric[b]
        if on.n_islanded[b] > 0:
            a, c = np.maximum(a, pen), np.maximum(c, pen)
        assert np.array_equal(a, c), b
    assert on.n1_pairs <= off.n1_pairs


@pytest.mark.parametrize("name", ["fixture_b", "g118"])
def test_wave_split_is_invisible(name, sessions):
    """Splitting a batch into many waves (workspace reuse, double-buffered host
    staging) gives bit-identical results to a single wave."""
    case = next(c for c in CASES if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    eng = sess.engine
    args = (arr["splits"], arr["disconnections"], arr["injection_sets"])
    try:
        eng.set_wave(0)
        one = eng.solve(*args, want_candidates=True)
        eng.set_wave(3)
        many = eng.solve(*args, want_candidates=True)
    finally:
        eng.set_wave(0)
    assert many.waves > 2 and one.waves == 1
    assert np.array_equal(one.best, many.best)
    assert np.array_equal(one.metric, many.metric, equal_nan=True)
    assert np.array_equal(one.feasible, many.feasible)
    assert np.array_equal(one.cand_metric, many.cand_metric)
    assert one.reports() == many.reports()
    assert one.loadflows == many.loadflows and one.n1_pairs == many.n1_pairs


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b", "case300", "g118"])
def test_report_select_variants_agree(name, sessions, monkeypatch):
    """The warp-per-task winner-report selection (small grids) and the CTA-per-task one
    (large grids, forced here with BDC_RSEL_CTA=1) give bit-identical results, and so do
    the report sweep's one-case and four-case warp variants (BDC_RSWEEP_CQ) and the two
    FP64 re-score variants (BDC_RESCORE_NT, BDC_RESCORE_FULL)."""
    case = next(c for c in CASES if c["name"] == name)
    sess = sessions(case)
    arr, _ = load_case(name)
    eng = sess.engine
    args = (arr["splits"], arr["disconnections"], arr["injection_sets"])
    warp = eng.solve(*args)
    monkeypatch.setenv("BDC_RSEL_CTA", "1")
    cta = eng.solve(*args)
    monkeypatch.delenv("BDC_RSEL_CTA")
    assert np.array_equal(warp.best, cta.best)
    assert np.array_equal(warp.metric, cta.metric, equal_nan=True)
    assert warp.reports() == cta.reports()
    # the FP64 near-tie re-score: 2- vs 8-warp CTAs, hot elements vs every row of every class
    for env in (("BDC_RESCORE_NT", "256"), ("BDC_RESCORE_FULL", "1")):
        monkeypatch.setenv(*env)
        alt = eng.solve(*args)
        monkeypatch.delenv(env[0])
        assert np.array_equal(warp.best, alt.best), env
        assert np.array_equal(warp.metric, alt.metric, equal_nan=True), env
    # k_scale_tc with task groups rasterised fastest (the large-grid order): same bounds
    monkeypatch.setenv("BDC_SCALE_RASTER", "1")
    ras = eng.solve(*args)
    monkeypatch.delenv("BDC_SCALE_RASTER")
    assert np.array_equal(warp.best, ras.best)
    assert np.array_equal(warp.metric, ras.metric, equal_nan=True)
    assert warp.n1_pairs == ras.n1_pairs
    # prefix-shared split chains (k_update's memo) forced on: copied splits, same bits
    monkeypatch.setenv("BDC_PREFIX", "1")
    pfx = eng.solve(*args)
    monkeypatch.delenv("BDC_PREFIX")
    assert np.array_equal(warp.best, pfx.best)
    assert np.array_equal(warp.metric, pfx.metric, equal_nan=True)
    assert warp.reports() == pfx.reports()
    # the multi/injection dominance screen (k_oscreen + k_oexact) forced on
    monkeypatch.setenv("BDC_OSCREEN", "1")
    osc = eng.solve(*args)
    # ... with the side stream forced on and off (k_terms, k_other next to / on the solve stream)
    monkeypatch.setenv("BDC_SIDE", "1")
    osc2 = eng.solve(*args)
    monkeypatch.setenv("BDC_SIDE", "0")
    osc1 = eng.solve(*args)
    monkeypatch.delenv("BDC_OSCREEN")
    assert np.array_equal(warp.best, osc.best)
    assert np.array_equal(warp.metric, osc.metric, equal_nan=True)
    assert warp.reports() == osc.reports()
    assert np.array_equal(osc1.metric, osc.metric, equal_nan=True)
    assert osc1.reports() == osc.reports() and osc1.n1_pairs == osc.n1_pairs
    assert np.array_equal(osc2.metric, osc.metric, equal_nan=True)
    assert osc2.reports() == osc.reports() and osc2.n1_pairs == osc.n1_pairs
    # one stream for everything, and the side stream next to the N-0 contraction / TOP path
    ser = eng.solve(*args)
    monkeypatch.setenv("BDC_SIDE", "1")
    sid = eng.solve(*args)
    monkeypatch.delenv("BDC_SIDE")
    assert np.array_equal(warp.metric, sid.metric, equal_nan=True)
    assert warp.reports() == sid.reports()
    assert warp.n1_pairs == sid.n1_pairs and warp.loadflows == sid.loadflows
    assert np.array_equal(warp.best, ser.best)
    assert np.array_equal(warp.metric, ser.metric, equal_nan=True)
    assert warp.reports() == ser.reports()
    assert warp.n1_pairs == ser.n1_pairs and warp.loadflows == ser.loadflows
    monkeypatch.setenv("BDC_RSWEEP_NT", "256")  # one-chunk sweep with 256- instead of 128-thread CTAs
    nt = eng.solve(*args)
    monkeypatch.delenv("BDC_RSWEEP_NT")
    assert np.array_equal(warp.metric, nt.metric, equal_nan=True)
    assert warp.reports() == nt.reports()
    monkeypatch.setenv("BDC_RSWEEP_WIDE", "1")  # 160-case sweep tiles (batches >= 1024 tasks)
    wide = eng.solve(*args)
    monkeypatch.delenv("BDC_RSWEEP_WIDE")
    assert np.array_equal(warp.metric, wide.metric, equal_nan=True)
    assert warp.reports() == wide.reports()
    for cq in ("1", "4"):
        monkeypatch.setenv("BDC_RSWEEP_CQ", cq)
        alt = eng.solve(*args)
        monkeypatch.delenv("BDC_RSWEEP_CQ")
        assert np.array_equal(warp.metric, alt.metric, equal_nan=True)
        assert warp.reports() == alt.reports()


@pytest.mark.parametrize("name,T,k,d", [("g1k", 72, 3, 1), ("g3k", 16, 6, 0)])
def test_large_grid_matches_oracle(name, T, k, d):
    """Paper-scale synthetic grids exercise the large-grid kernel variants (CTA top-k and
    report selection, multi-chunk report sweep, many tensor-core case tiles, the
    warp-per-case multi/injection stream at G1k's 11 cases x 72 candidates) against the
    CPU oracle: feasibility and reasons exact, metric within TAU, winner metric-minimal."""
    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.session import session_open, solve_batch_output

    grid = synth.make_grid(name, seed=0)
    sess = session_open(grid)
    splits, discos, inj = synth.random_task_arrays(grid, 6, T, k, seed=11, n_disconnections=d)
    out = solve_batch_output(sess, splits, discos, inj)
    ref = port.solve_arrays(grid, sess.base, splits, discos, inj, sess.config)
    for b, r in enumerate(ref):
        assert bool(out.feasible[b]) == r.feasible, (b, r.reason)
        if not r.feasible:
            assert out.reason(b) == r.reason
            continue
        assert abs(out.metric[b] - r.metric) <= TAU, (b, out.metric[b], r.metric)
        if int(out.best[b]) != r.best_injection:
            continue  # a tie within TAU: the metric check above is the contract
        doc = out.report(b)
        assert len(doc["n1_worst"]) == len(r.n1_worst)
        for a, e in zip(doc["n1_worst"], r.n1_worst):
            assert abs(a["rel_load"] - e[3]) <= 1e-6, (b, a, e)
