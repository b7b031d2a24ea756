"""Where the e2e (host arrays in/out) time goes, per phase (run under gpurun)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_2501_17529_b200.session import session_open, validate_arrays
from paper_2501_17529_b200.engine import BatchOutput

cfg = sys.argv[1] if len(sys.argv) > 1 else "g118"
grid, splits, discos, inj = bench.make_workload(cfg, 0)
sess = session_open(grid)
eng = sess.engine
ps = torch.from_numpy(splits).pin_memory().numpy()
pd = torch.from_numpy(discos).pin_memory().numpy()
pi = torch.from_numpy(inj).pin_memory().numpy()
for it in range(4):
    t = [time.perf_counter()]
    mv, o, ij = validate_arrays(sess, ps, pd, pi); t.append(time.perf_counter())
    mr = eng.check_batch(mv.view(np.uint8), o); t.append(time.perf_counter())
    out = eng.solve(mv.view(np.uint8), o, ij.view(np.uint8), max_rank=mr); t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"{cfg} it{it}: validate {d[0]:.2f} ms, scan {d[1]:.2f} ms, solve {d[2]:.2f} ms; device stages {sum(out.stage_ms):.2f} ms {[round(x,2) for x in out.stage_ms]}")
B = inj.shape[0]
for name in ("alloc",):
    t0 = time.perf_counter(); BatchOutput(eng, B, inj.shape[1], 10, 5, mv, o, ij, False); print("BatchOutput alloc", (time.perf_counter()-t0)*1e3, "ms")
