import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2501_17529_b200.session import session_open, solve_batch_output
cfg = sys.argv[1] if len(sys.argv) > 1 else "g118"
grid, s, d, i = bench.make_workload(cfg, 0)
sess = session_open(grid)
ps = torch.from_numpy(s).pin_memory().numpy(); pd = torch.from_numpy(d).pin_memory().numpy(); pi = torch.from_numpy(i).pin_memory().numpy()
for cap in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "16384", "8192", "0"])]:
    sess.engine.set_wave(cap)
    solve_batch_output(sess, ps, pd, pi)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter(); o = solve_batch_output(sess, ps, pd, pi); ts.append(time.perf_counter() - t0)
    print("cap", cap, "e2e ms", [round(x*1e3, 2) for x in ts], "lf/s %.3e" % (o.loadflows / np.median(ts)), "dev", round(sum(o.stage_ms), 2), [round(x, 2) for x in o.stage_ms])
