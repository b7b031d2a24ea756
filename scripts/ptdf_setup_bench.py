"""Base-PTDF setup time, host scipy SPD solve vs the device (bdc_spd_solve), per grid.
    python scripts/ptdf_setup_bench.py [g1k g3k g10k]"""
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_2501_17529_b200 import synth  # noqa: E402
from paper_2501_17529_b200.ptdf import compute_ptdf  # noqa: E402

rows = []
for spec in sys.argv[1:] or ["g1k", "g3k", "g10k"]:
    grid = synth.make_grid(spec, seed=0)
    compute_ptdf(synth.make_grid("g14", seed=0), device=0)  # warm the context
    t0 = time.perf_counter()
    dev = compute_ptdf(grid, device=0)
    t_dev = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = compute_ptdf(grid)
    t_host = time.perf_counter() - t0
    err = float(np.abs(dev.values - host.values).max())
    n = grid.n_nodes - 1
    rows.append({"grid": spec, "nodes": grid.n_nodes, "rows": int(host.values.shape[0]), "host_s": t_host,
                 "device_s": t_dev, "speedup": t_host / t_dev, "max_abs_diff": err,
                 "potrf_flops": n ** 3 / 3, "potrs_flops": 2.0 * n * n * host.values.shape[0]})
    print(json.dumps(rows[-1]), flush=True)
os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
with open(os.path.join(REPO, "gpurun_out", "ptdf_setup.json"), "w") as fh:
    json.dump(rows, fh, indent=1)
