"""CPU-only checks: the C-ABI library, host-side validation, task generation.

No compute call reaches the device here (there is no GPU in the build
container); the device paths are covered by the `-m gpu` tests.
"""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, golden_path
from oracle import port, refact
from paper_2501_17529_b200 import synth
from paper_2501_17529_b200.errors import DisconnectedTopology, EngineUnavailable, ParseError, ValidationError
from paper_2501_17529_b200.io import grid_to_dict, load_grid
from paper_2501_17529_b200.ptdf import prepare_base_ptdf
from paper_2501_17529_b200.session import SolverSession, session_open, validate_arrays
from paper_2501_17529_b200.solver import SolveConfig, SplitAction, TopologyTask, canonicalize_task


def _header_symbols():
    with open(os.path.join(REPO, "include", "bdc.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(bdc_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2501_17529_b200 import build, engine

    if not os.path.exists(build.TARGET):
        pytest.skip("libbdc.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(build.TARGET)
    syms = _header_symbols()
    assert len(syms) >= 8
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(engine.EXPORTS)
    lib.bdc_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.bdc_version()


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of BdcGrid/BdcConfig/BdcBatch have the C layout: a probe compiled
    with gcc against include/bdc.h prints sizeof and every field's offsetof."""
    import shutil
    import subprocess

    from paper_2501_17529_b200 import engine

    # 13 int32 + 31 pointers, padded to 8
    assert ctypes.sizeof(engine._Grid) == 13 * 4 + 4 + 31 * 8
    assert ctypes.sizeof(engine._Config) == 32
    assert engine._Batch.stage_ms.offset % 4 == 0
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    structs = {"BdcGrid": engine._Grid, "BdcConfig": engine._Config, "BdcBatch": engine._Batch}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "bdc.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f in cls._fields_:
            lines.append(f'printf("{cname}.{f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines.append("return 0;}")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run([cc, "-I", os.path.join(REPO, "include"), "-o", str(exe), str(src)], check=True)
    got = dict(ln.split() for ln in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.splitlines())
    for cname, cls in structs.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f in cls._fields_:
            assert int(got[f"{cname}.{f[0]}"]) == getattr(cls, f[0]).offset, (cname, f[0])


def _fake_session(path):
    grid = load_grid(path)
    return SolverSession(
        grid=grid,
        base=prepare_base_ptdf(grid),
        config=SolveConfig(),
        element_counts=tuple(len(s.branch_elements) for s in grid.substations),
        engine=None,
    )


def test_session_validation_messages():
    """Same checks and messages as the reference binding (test_bindings.py:206-278)."""
    session = _fake_session(golden_path("grids", "fixture_b.json"))
    n_slots = session.n_slots
    S, E = session.split_shape
    good = np.zeros((2, 1, n_slots), dtype=bool)
    with pytest.raises(ValidationError, match="slot bits"):
        validate_arrays(session, None, None, np.zeros((2, 1, n_slots + 1), dtype=bool))
    with pytest.raises(ValidationError, match="3-dimensional"):
        validate_arrays(session, None, None, np.zeros((2, n_slots), dtype=bool))
    with pytest.raises(ValidationError, match="candidate row"):
        validate_arrays(session, None, None, np.zeros((2, 0, n_slots), dtype=bool))
    with pytest.raises(ValidationError, match="must be boolean"):
        validate_arrays(session, None, None, np.zeros((2, 1, n_slots)))
    with pytest.raises(ValidationError, match="does not match"):
        validate_arrays(session, np.zeros((2, S + 1, E), dtype=bool), None, good)
    with pytest.raises(ValidationError, match="does not match"):
        validate_arrays(session, np.zeros((3, S, E), dtype=bool), None, good)
    with pytest.raises(ValidationError, match="integer"):
        validate_arrays(session, None, np.zeros((2, 1)), good)
    with pytest.raises(ValidationError, match="shape"):
        validate_arrays(session, None, np.zeros(2, dtype=np.int64), good)
    bad = np.full((2, 1), -1, dtype=np.int64)
    bad[1, 0] = session.n_branches
    with pytest.raises(ValidationError, match="indices"):
        validate_arrays(session, None, bad, good)
    dup = np.array([[3, 3], [1, -1]], dtype=np.int64)
    with pytest.raises(ValidationError, match="duplicate"):
        validate_arrays(session, None, dup, good)
    ok = np.array([[-1, -1], [1, -1]], dtype=np.int64)
    validate_arrays(session, None, ok, good)


def test_split_bits_past_width_rejected():
    doc = {
        "nodes": [{"id": f"n{i}"} for i in range(6)],
        "branches": [
            {"id": f"r{i}", "from": f"n{i}", "to": f"n{(i + 1) % 6}", "susceptance": 2.0, "rating": 100.0}
            for i in range(6)
        ]
        + [
            {"id": "c0", "from": "n1", "to": "n4", "susceptance": 1.5, "rating": 100.0},
            {"id": "c1", "from": "n0", "to": "n3", "susceptance": 1.0, "rating": 100.0},
        ],
        "injections": [{"id": "g0", "node": "n4", "p_mw": 50.0}, {"id": "l0", "node": "n2", "p_mw": -50.0}],
        "slack": "n0",
        "substations": [
            {"node": "n1", "branch_elements": ["r0", "r1", "c0"], "injection_elements": []},
            {"node": "n3", "branch_elements": ["r2", "r3"], "injection_elements": []},
        ],
        "contingencies": [],
    }
    from paper_2501_17529_b200.io import grid_from_dict

    grid = grid_from_dict(doc)
    s = SolverSession(grid, prepare_base_ptdf(grid), SolveConfig(), (3, 2), None)
    assert s.split_shape == (2, 3)
    splits = np.zeros((1, 2, 3), dtype=bool)
    splits[0, 1, 2] = True
    with pytest.raises(ValidationError, match="substation 1"):
        validate_arrays(s, splits, None, np.zeros((1, 1, 0), dtype=bool))


def test_open_sources_and_errors():
    with pytest.raises(FileNotFoundError):
        session_open(golden_path("grids", "no_such_grid.json"))
    with pytest.raises(ParseError, match="missing"):
        session_open({})
    with pytest.raises(ValidationError, match="grid source"):
        session_open(42)


def test_no_cpu_fallback_without_device():
    """The solve path fails loudly when no GPU (or no library) is present."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    grid = load_grid(golden_path("grids", "fixture_b.json"))
    with pytest.raises(EngineUnavailable):
        session_open(grid)


def test_canonicalize_rules():
    grid = load_grid(golden_path("grids", "fixture_b.json"))
    t = TopologyTask(
        splits=(
            SplitAction(2, (True, False, False)),
            SplitAction(0, (False, False, False)),
            SplitAction(1, (False, True, False)),
        ),
        injection_sets=((),),
    )
    c = canonicalize_task(grid, t)
    assert [s.substation for s in c.splits] == [1, 2]
    assert c.injection_sets == ((False, False, False),)
    with pytest.raises(ValidationError, match="out of range"):
        canonicalize_task(grid, TopologyTask(splits=(SplitAction(9, (True,)),)))
    with pytest.raises(ValidationError, match="twice"):
        canonicalize_task(grid, TopologyTask(splits=(SplitAction(1, (True, False, False)), SplitAction(1, (False, True, False)))))
    with pytest.raises(ValidationError, match="bits"):
        canonicalize_task(grid, TopologyTask(splits=(SplitAction(1, (True,)),)))
    with pytest.raises(ValidationError, match="duplicate"):
        canonicalize_task(grid, TopologyTask(disconnections=(3, 3)))
    with pytest.raises(ValidationError, match="injection set"):
        canonicalize_task(grid, TopologyTask(injection_sets=((True,),)))
    with pytest.raises(ValidationError, match="at least one"):
        canonicalize_task(grid, TopologyTask(injection_sets=()))


def test_solve_config_validation():
    for bad in (
        {"mode": "fastest"},
        {"islanding_policy": "ignore"},
        {"multi_outage_method": "magic"},
        {"topk_per_case": 0},
        {"topk_global": 0},
        {"workers": 0},
        {"max_simultaneous_outages": 0},
        {"islanding_penalty": 0.0},
    ):
        with pytest.raises(ValidationError):
            SolveConfig(**bad).validate()
    SolveConfig().validate()


@pytest.mark.parametrize("spec", ["g14", "g118"])
def test_task_generator_feasibility_matches_oracle(spec):
    """Vectorised N-0 acceptance == the refactorisation oracle's connectivity test."""
    grid = synth.make_grid(spec)
    s, d, i = synth.random_task_arrays(grid, 200, 2, 3, seed=3, n_disconnections=2, reject_infeasible=False)
    mask = synth._feasible_mask(grid, s, d)
    canons = port.decode_arrays(grid, s, d, i)
    for b, c in enumerate(canons):
        degenerate = any(all(bits) for _si, bits in c.splits)
        try:
            refact.materialize(grid, c)
            connected = True
        except DisconnectedTopology:
            connected = False
        assert mask[b] == (connected and not degenerate), b
    assert 0 < mask.sum() < len(mask)


def test_synthetic_grid_shapes():
    g = synth.make_grid("g1k")
    assert g.n_nodes == 1000 and g.n_branches == 1370
    assert len(g.substations) == 50 and len(g.injection_slots) == 72
    assert all(len(s.branch_elements) == 5 for s in g.substations)
