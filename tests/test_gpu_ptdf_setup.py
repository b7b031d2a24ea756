"""GPU base-PTDF setup: the SPD solve of compute_ptdf
(factors.py:161-216) as blocked FP64 potrf + potrs on the device (bdc_spd_solve),
against the host scipy path the reference uses -- values to rounding, the engine's
results on a GPU-built base equal to the reference documents, singular systems raising
the reference's SingularSystem."""

import numpy as np
import pytest

from conftest import golden_path, load_case, load_manifest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["fixture_a", "fixture_b", "case300", "g118", "g1k"])
def test_device_ptdf_equals_host(name):
    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.io import load_grid
    from paper_2501_17529_b200.ptdf import prepare_base_ptdf

    grid = synth.make_grid(name, seed=0) if name.startswith("g") else load_grid(golden_path("grids", f"{name}.json"))
    host = prepare_base_ptdf(grid)
    dev = prepare_base_ptdf(grid, device=0)
    assert dev.values.shape == host.values.shape
    scale = max(1.0, float(np.abs(host.values).max()))
    assert np.abs(dev.values - host.values).max() <= 1e-11 * scale
    assert np.array_equal(dev.from_cols, host.from_cols) and np.array_equal(dev.to_cols, host.to_cols)
    assert dev.static_col == host.static_col


def test_engine_on_device_built_base_matches_reference():
    from paper_2501_17529_b200.session import session_open, solve_batch

    case = next(c for c in load_manifest() if c["name"] == "g118")
    from test_gpu_large import _grid_source  # same synthetic-grid pinning

    sess = session_open(_grid_source(case), base_setup="gpu")
    arr, docs = load_case("g118")
    out = solve_batch(sess, arr["splits"], arr["disconnections"], arr["injection_sets"])
    for mine, doc in zip(out["reports"], docs):
        assert mine["feasible"] == doc["feasible"]
        if doc["feasible"]:
            assert abs(mine["metric"] - doc["metric"]) <= 1e-9 * max(1.0, abs(doc["metric"]))


def test_singular_susceptance_matrix_raises():
    from paper_2501_17529_b200.errors import SingularSystem
    from paper_2501_17529_b200.ptdf import _spd_solve_device

    lap = np.array([[1.0, -1.0, 0.0], [-1.0, 1.0, 0.0], [0.0, 0.0, 2.0]])  # not positive definite
    with pytest.raises(SingularSystem, match="factorization failed"):
        _spd_solve_device(lap, np.eye(3), 0)
    spd = np.array([[4.0, 1.0], [1.0, 3.0]])
    x = _spd_solve_device(spd, np.eye(2), 0)
    assert np.allclose(x, np.linalg.inv(spd), atol=1e-14)
