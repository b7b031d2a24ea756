"""Device-side task generation (taskgen.random_tasks_device, csrc/bdc_gen.cu) against the
reference generator's rules (batchdc.bench.random_tasks, src/batchdc/bench.py:33-91):
distinct eligible substations, non-empty assignment bits, distinct disconnections,
uniform injection bits, every returned task feasible at N-0 -- and the engine's results
on drawn tasks against the CPU oracle."""

import numpy as np
import pytest

from oracle import port

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def g118():
    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.session import session_open

    grid = synth.make_grid("g118", seed=0)
    return session_open(grid)


def _draw(sess, B, T, k, d, seed):
    from paper_2501_17529_b200.taskgen import random_tasks_device, to_host

    s, dc, inj, draws = random_tasks_device(sess, B, T, k, seed, n_disconnections=d)
    return to_host(s, dc, inj) + (draws,)


@pytest.mark.parametrize("k,d", [(3, 0), (2, 1), (1, 2)])
def test_drawn_tasks_follow_the_reference_rules(g118, k, d):
    from paper_2501_17529_b200.synth import _feasible_mask

    sess = g118
    grid = sess.grid
    splits, discos, inj, draws = _draw(sess, 4096, 16, k, d, seed=11)
    counts = np.array([len(s.branch_elements) for s in grid.substations])
    eligible = counts >= 2
    moved = splits.any(axis=2)
    assert (moved.sum(axis=1) == min(k, int(eligible.sum()))).all()
    assert not (moved & ~eligible[None, :]).any()
    width = splits.shape[2]
    valid = np.arange(width)[None, :] < counts[:, None]
    assert not (splits & ~valid[None]).any(), "bits beyond a substation's elements"
    if d:
        assert (discos >= 0).all() and (discos < grid.n_branches).all()
        srt = np.sort(discos, axis=1)
        assert not (srt[:, 1:] == srt[:, :-1]).any(), "repeated disconnection"
    assert inj.shape == (4096, 16, len(grid.injection_slots))
    # acceptance: every returned task is feasible at N-0 (the host graph test agrees)
    assert _feasible_mask(grid, splits, discos).all()
    assert draws >= 1


def test_drawn_distribution_is_uniform(g118):
    sess = g118
    grid = sess.grid
    splits, _, inj, _ = _draw(sess, 16384, 32, 1, 0, seed=3)
    counts = np.array([len(s.branch_elements) for s in grid.substations])
    elig = np.flatnonzero(counts >= 2)
    freq = splits.any(axis=2)[:, elig].sum(axis=0) / 16384.0
    # one split per task: each eligible substation with probability ~1/|eligible|
    # (rejections remove a few draws, so the tolerance is loose)
    assert np.allclose(freq, 1.0 / len(elig), atol=0.05), freq
    assert abs(inj.mean() - 0.5) < 0.01
    # assignment bits: uniform over the non-empty patterns of each substation
    for si in elig[:3]:
        rows = splits[:, si, : counts[si]][splits[:, si].any(axis=1)]
        assert abs(rows.mean() - 0.5 * 2 ** counts[si] / (2 ** counts[si] - 1)) < 0.05


def test_draws_are_deterministic_per_seed(g118):
    a = _draw(g118, 512, 8, 3, 1, seed=5)
    b = _draw(g118, 512, 8, 3, 1, seed=5)
    c = _draw(g118, 512, 8, 3, 1, seed=6)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)
    assert not np.array_equal(a[0], c[0])


def test_engine_on_drawn_tasks_matches_oracle(g118):
    """The drawn batch through the session API against the CPU oracle: feasibility and
    reasons exact, metric within 1e-9 where the winner agrees, winner agreement up to
    FP64 ties."""
    from paper_2501_17529_b200.session import solve_batch_output

    sess = g118
    splits, discos, inj, _ = _draw(sess, 48, 16, 3, 1, seed=21)
    out = solve_batch_output(sess, splits, discos, inj)
    ref = port.solve_arrays(sess.grid, sess.base, splits, discos, inj, sess.config)
    for b, r in enumerate(ref):
        assert bool(out.feasible[b]) == r.feasible, b
        if not r.feasible:
            assert out.reason(b) == r.reason
            continue
        scale = max(1.0, abs(r.metric))
        if int(out.best[b]) == r.best_injection:
            assert abs(out.metric[b] - r.metric) <= 1e-9 * scale
        else:
            canon = port.decode_arrays(sess.grid, splits[b:b + 1], discos[b:b + 1],
                                       inj[b:b + 1, [int(out.best[b]), r.best_injection]])[0]
            m = port.evaluate(sess.grid, sess.base, canon, sess.config)[0]
            assert abs(float(m[0]) - float(m[1])) <= 1e-12 * scale
