"""Near-tie band statistics of the FP64 winner re-score (k_rescore), per bench config.

    python scripts/rescore_diag.py [g118 g1k g3k g10k]

Prints, per config: tasks, tasks with more than one candidate in the band, band size
distribution, distinct FP32 values inside the band, candidates re-scored, winners changed,
and the select-stage time.
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from bench import WORKLOADS, make_workload  # noqa: E402
from paper_2501_17529_b200.engine import STAGES  # noqa: E402
from paper_2501_17529_b200.session import session_open  # noqa: E402

EPS = 6.103515625e-05


def main(names):
    for name in names:
        spec, tasks, T, k, d = WORKLOADS[name]
        tasks = min(tasks, 8192)
        grid, s, dd, inj = make_workload(name, 0, tasks, T)
        sess = session_open(grid)
        out = sess.engine.solve(s, dd, inj, want_candidates=True)
        out = sess.engine.solve(s, dd, inj, want_candidates=True)
        cm = out.cand_metric.astype(np.float64)
        fe = out.feasible.astype(bool)
        pen = out.n_islanded > 0
        v = np.where(pen[:, None], np.maximum(cm, sess.config.islanding_penalty), cm)
        vmin = v.min(axis=1)
        hi = vmin + 2 * EPS * np.maximum(1.0, vmin)
        band = (v <= hi[:, None]) & fe[:, None]
        bs = band.sum(axis=1)[fe]
        distinct = np.array([len(np.unique(v[b][band[b]])) for b in np.flatnonzero(fe)])
        st = dict(zip(STAGES, out.stage_ms))
        print(f"{name}: tasks={tasks} feasible={fe.sum()} pen={int((pen & fe).sum())} "
              f"band>1={int((bs > 1).sum())} band mean={bs.mean():.1f} p50={np.median(bs):.0f} "
              f"p90={np.percentile(bs, 90):.0f} max={bs.max()} distinct mean={distinct.mean():.1f} "
              f"max={distinct.max()} rescore_stats={out.rescore_stats.tolist()} "
              f"select_ms={st['select']:.2f} report_ms={st['report']:.2f}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["g118", "g1k", "g3k", "g10k"])
