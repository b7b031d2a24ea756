"""Stub-branch replacement (grid.replace_stub_branches) against documents produced by the
reference's own batchdc.replace_stub_branches (tests/golden/make_stub_golden.py), plus the
reference's unit cases (pkg/tests/test_grid.py:193-250) restated."""

import glob
import json
import os

import pytest

from conftest import golden_path

STUBS = sorted(glob.glob(golden_path("stubs", "*.json")))


@pytest.mark.parametrize("path", STUBS, ids=[os.path.basename(p)[:-5] for p in STUBS])
def test_matches_reference_documents(path):
    from paper_2501_17529_b200.grid import replace_stub_branches
    from paper_2501_17529_b200.io import grid_from_dict, grid_to_dict

    with open(path) as fh:
        doc = json.load(fh)
    out = replace_stub_branches(grid_from_dict(doc["input"]))
    assert json.loads(json.dumps(grid_to_dict(out), sort_keys=True)) == doc["expected"]


def _tri(extra_branches, injections, slack=0, cases=()):
    from paper_2501_17529_b200.grid import Branch, Grid, SplittableSubstation

    top = max([2] + [max(b.from_node, b.to_node) for b in extra_branches])
    names = ["a", "b", "c", "x", "y"][: top + 1]
    br = (Branch("ab", 0, 1, 1.0, 10.0), Branch("bc", 1, 2, 1.0, 10.0), Branch("ac", 0, 2, 1.0, 10.0))
    g = Grid(node_ids=tuple(names), branches=br + tuple(extra_branches), injections=tuple(injections), slack=slack,
             substations=(SplittableSubstation(1, branch_elements=(0, 1)),), contingencies=tuple(cases))
    g.validate()
    return g


def test_hanging_load_collapses_onto_the_substation():
    from paper_2501_17529_b200.grid import Branch, Injection, replace_stub_branches

    g = _tri((Branch("bx", 1, 3, 1.0, 10.0), Branch("xy", 3, 4, 1.0, 10.0)),
             (Injection("g", 0, 5.0), Injection("l", 4, -5.0)))
    r = replace_stub_branches(g)
    assert r.n_nodes == 3 and r.n_branches == 3
    assert {i.id: r.node_ids[i.node] for i in r.injections} == {"g": "a", "l": "b"}
    assert r.injection_index["l"] in r.substations[0].injection_elements


def test_named_or_slack_side_stubs_stay():
    from paper_2501_17529_b200.grid import Branch, ContingencyCase, Injection, replace_stub_branches

    named = _tri((Branch("bx", 1, 3, 1.0, 10.0),), (Injection("l", 3, -5.0),),
                 cases=(ContingencyCase("n1_bx", "single_branch", branches=(3,)),))
    assert replace_stub_branches(named).n_nodes == 4
    slack = _tri((Branch("bx", 1, 3, 1.0, 10.0),), (), slack=3)
    assert replace_stub_branches(slack).n_nodes == 4


def test_parallel_branches_are_not_bridges():
    from paper_2501_17529_b200.grid import Branch, branch_bridges

    g = _tri((Branch("bx", 1, 3, 1.0, 10.0), Branch("bx2", 1, 3, 1.0, 10.0)), ())
    assert branch_bridges(g) == frozenset()
