#!/usr/bin/env python3
"""BASELINE configs[4]: the ~10k-bus grid with 1..1024 injection candidates per topology.

Runs bench.py once per candidate count and tabulates the device stages: the per-topology
update (split chain, case factors) and the tensor-core screening scales do not depend on T,
the N-0 contraction, the N-1 sweep and the multi/injection cases grow with T -- the
crossover is where the T-proportional stages overtake the per-topology ones.
    python scripts/tsweep.py [--config g10k] [--tasks 64] [--out gpurun_out/tsweep_g10k.json]
"""
import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="g10k")
    ap.add_argument("--tasks", type=int, default=64)
    ap.add_argument("--ts", default="1,2,4,8,16,32,64,128,256,512,1024")
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "tsweep_g10k.json"))
    args = ap.parse_args()
    rows = []
    for T in [int(x) for x in args.ts.split(",")]:
        cmd = [sys.executable, os.path.join(REPO, "bench.py"), "--config", args.config, "--tasks", str(args.tasks),
               "--candidates", str(T), "--steps", "3", "--warmup", "3", "--no-cpu", "--check", "0"]
        p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ""
        try:
            d = json.loads(line)
        except ValueError:
            print(T, "FAILED", p.stderr[-800:])
            continue
        st = d["stage_ms_per_step"]
        per_topo = st["update"] + st["scale"] + st["topk"]
        per_cand = st["n0"] + st["top"] + st["screen"] + st["other_n1"]
        # the dense injection contraction the north star names, (R x C) . (C x T) per
        # topology, at the tensor-core peak (TF32 = BF16 / 2, MEASURED_PEAKS.json), against
        # the measured low-rank N-0 stage (k_n0: f0 + B'' y_t, inner dimension k+d)
        cfg = d["config"]
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
            os.path.join(REPO, "MEASURED_PEAKS.json")) else {"bf16_tflops": 1670.9}
        dense_flops = 2.0 * cfg["rows"] * (cfg["rows"] / 1.37) * T * args.tasks  # C = nodes ~ R / 1.37
        dense_ms = dense_flops / (peaks["bf16_tflops"] / 2 * 1e12) * 1e3
        rows.append({"T": T, "lf_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                     "per_topology_ms": per_topo, "per_candidate_ms": per_cand, "report_ms": st["report"],
                     "n0_ms": st["n0"], "dense_gemm_ms_at_tf32_peak": dense_ms,
                     "stages": st, "skipped_frac": d["screen"]["skipped_frac"]})
        print(f"T={T:5d} {d['value']:.3e} lf/s  step {d['ms_per_step']:.2f} ms  per-topology {per_topo:.2f} ms  "
              f"per-candidate {per_cand:.2f} ms  report {st['report']:.2f} ms  n0 {st['n0']:.3f} ms  "
              f"dense GEMM at TF32 peak {dense_ms:.3f} ms", flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump({"config": args.config, "tasks": args.tasks, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
