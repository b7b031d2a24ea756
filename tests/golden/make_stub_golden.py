#!/usr/bin/env python3
"""Golden documents for stub-branch replacement, produced by the
REFERENCE's own batchdc.replace_stub_branches (src/batchdc/grid.py:437-560).

Run in the build container only (imports /root/reference/pkg):

    python tests/golden/make_stub_golden.py

Input grids are the reference fixtures and a synthetic G118 grid with radial
appendages grafted on (chains and small trees hanging off substation nodes and off
ordinary nodes, carrying loads / generators / monitored and unmonitored branches; some
appendages are referenced by a contingency or hold the slack, so they must stay).
Writes tests/golden/stubs/<name>.json = {"input": grid doc, "expected": grid doc}.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/pkg"
sys.path[:0] = [os.path.join(REF, "src"), REPO]

from batchdc import replace_stub_branches  # noqa: E402
from batchdc.io import grid_from_dict, grid_to_dict  # noqa: E402

from paper_2501_17529_b200 import synth  # noqa: E402

OUT = os.path.join(HERE, "stubs")


def graft(doc: dict, seed: int, n_app: int, referenced: int = 1, slack_side: bool = False) -> dict:
    """Attach n_app radial appendages to `doc` (a grid document)."""
    rng = np.random.default_rng(seed)
    doc = json.loads(json.dumps(doc))
    nodes = [n["id"] for n in doc["nodes"]]
    subs = [s["node"] for s in doc["substations"]]
    anchors = subs + [nodes[i] for i in rng.choice(len(nodes), size=min(4, len(nodes)), replace=False)]
    for a in range(n_app):
        at = anchors[a % len(anchors)]
        depth = int(rng.integers(1, 4))
        prev = at
        chain = []
        for d in range(depth):
            nid = f"stub{a}_{d}"
            doc["nodes"].append({"id": nid})
            bid = f"sb{a}_{d}"
            doc["branches"].append({"id": bid, "from": prev, "to": nid,
                                    "susceptance": float(np.round(rng.uniform(2.0, 20.0), 4)),
                                    "rating": float(np.round(rng.uniform(30.0, 120.0), 1)),
                                    "monitored": bool(rng.random() < 0.7)})
            chain.append(bid)
            if rng.random() < 0.6:
                doc["injections"].append({"id": f"sl{a}_{d}", "node": nid,
                                          "p_mw": -float(np.round(rng.uniform(5.0, 40.0), 2))})
            if rng.random() < 0.2:
                doc["injections"].append({"id": f"sg{a}_{d}", "node": nid,
                                          "p_mw": float(np.round(rng.uniform(5.0, 30.0), 2))})
            # a side branch (small tree) now and then
            if rng.random() < 0.3:
                tid = f"stub{a}_{d}t"
                doc["nodes"].append({"id": tid})
                doc["branches"].append({"id": f"sb{a}_{d}t", "from": nid, "to": tid, "susceptance": 7.5,
                                        "rating": 50.0, "monitored": True})
                doc["injections"].append({"id": f"st{a}_{d}", "node": tid, "p_mw": -3.0})
            prev = nid
        if a < referenced:
            doc["contingencies"].append({"id": f"n1_{chain[-1]}", "kind": "single_branch", "branches": [chain[-1]]})
    if slack_side:
        doc["slack"] = f"stub{n_app - 1}_0"
    return doc


def main():
    os.makedirs(OUT, exist_ok=True)
    bases = {}
    for name in ("fixture_a", "fixture_b", "case300"):
        with open(os.path.join(HERE, "grids", f"{name}.json")) as fh:
            bases[name] = json.load(fh)
    bases["g118"] = synth.make_grid_doc("g118", seed=0)
    cases = [
        ("fixture_a_stubs", "fixture_a", dict(seed=1, n_app=4)),
        ("fixture_b_stubs", "fixture_b", dict(seed=2, n_app=6, referenced=2)),
        ("case300_stubs", "case300", dict(seed=3, n_app=10, referenced=3)),
        ("g118_stubs", "g118", dict(seed=4, n_app=12, referenced=2)),
        ("g118_slack_side", "g118", dict(seed=5, n_app=5, referenced=0, slack_side=True)),
    ]
    for name, base, kw in cases:
        doc = graft(bases[base], **kw)
        grid = grid_from_dict(doc)
        grid.validate()
        out = replace_stub_branches(grid)
        with open(os.path.join(OUT, f"{name}.json"), "w") as fh:
            json.dump({"input": doc, "expected": grid_to_dict(out)}, fh, sort_keys=True)
        print(name, grid.n_nodes, "->", out.n_nodes, "nodes,", grid.n_branches, "->", out.n_branches, "branches")


if __name__ == "__main__":
    main()
