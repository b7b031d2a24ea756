"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the engine on tiny batches, each variant once.
    compute-sanitizer --tool racecheck python scripts/sanitize.py
"""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_2501_17529_b200 import synth  # noqa: E402
from paper_2501_17529_b200.session import session_open, solve_batch_output  # noqa: E402


def run(spec, B, T, k, d, seed=1):
    grid = synth.make_grid(spec, seed=0)
    sess = session_open(grid)
    s, dd, inj = synth.random_task_arrays(grid, B, T, k, seed=seed, n_disconnections=d)
    out = solve_batch_output(sess, s, dd, inj)
    print(spec, B, T, k, d, "feasible", int(out.feasible.sum()), "launches", out.kernel_launches, flush=True)
    sess.engine.probe_flows(s[0], dd[0], inj[0])


run("g14", 16, 16, 2, 1)
run("g118", 24, 64, 3, 1)       # TOP tile 16 x 64, warp report select, one-chunk sweep
run("g118", 8, 128, 3, 0)       # 16 x 128 TOP tile (T >= 96)
run("g1k", 4, 32, 3, 1)         # CTA report select, multi-chunk sweep, k_other_w
run("g3k", 2, 16, 8, 4)         # rank 12: k_scale_tc<2,2>, four-case sweep
