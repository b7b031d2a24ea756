#!/usr/bin/env python3
"""Throughput benchmark: DC loadflows/s of the batched topology screen on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config g118] [--impl ours|reference]

One step = one ``bdc_solve`` over one batch of synthetic topology tasks (the
BASELINE config: by default configs[1], a 118-bus-sized synthetic grid,
65,536 topologies x 64 injection candidates, k=3 busbar splits, full N-1).
A loadflow is one flow vector (topology, injection candidate, case), counted
exactly as the reference counts it: T * (1 + feasible cases) per feasible
task (`solver.py:881-883`).

Reported (one JSON line on rank 0):
  value     whole-job loadflows/s with inputs resident in HBM, device-timed with
            CUDA events on the solve stream, L2 flushed between steps, max over ranks;
            with N > 1 ranks the step includes the NCCL all-gather of every rank's
            per-topology results (parallel.all_gather_device)
  e2e       the same metric through the public API with host (pinned) inputs and
            host outputs, copies inside the timed region (wall clock): the session's
            solve_batch_output at N = 1, parallel.solve_shard (solve + all-gather) at N > 1
  roofline  the longest device stage against its bound (stages_roofline lists all:
            HBM bytes, tcgen05 TF32 flops, FP32 lane-ops, FP64 ops)
  parity_sample  --check n tasks of the timed batch re-solved by the CPU oracle port
            (checker only): feasibility, winner agreement, metric difference
  cpu_baseline  the CPU oracle port (reference algorithm, metric_first, plus the
            symmetric brute-force mode) on the host cores, bounded sample of the same
            workload (rank 0, N=1 only)

`--gpus N` outside torchrun launches N ranks itself (torch.distributed.run, 127.0.0.1).
`--impl reference` times the reference algorithm on the CPU instead (the oracle
port, all host cores).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (grid spec, tasks per GPU per step, candidates, splits, disconnections)
    "g14": ("g14", 1024, 16, 2, 0),
    "g118": ("g118", 65536, 64, 3, 0),
    "g1k": ("g1k", 8192, 128, 3, 0),
    "g3k": ("g3k", 1024, 32, 8, 0),
    "g10k": ("g10k", 64, 64, 3, 0),
    # BASELINE configs[2] (config C): 10^6 topologies x 128 over 8 GPUs, 125,000 per GPU,
    # drawn on the device (taskgen.random_tasks_device)
    "g1k_c": ("g1k", 125000, 128, 3, 0),
}
DEVICE_TASKS = {"g1k_c"}
DESCR = {
    "g14": "IEEE-14-sized synthetic grid, 1024 topologies x 16 injections, 2 splits, full N-1",
    "g118": "IEEE-118-sized synthetic grid, 65536 topologies x 64 injections, 3 splits, full N-1",
    "g1k": "1000-bus synthetic grid, topologies x 128 injections, 3 splits, full N-1",
    "g3k": "3000-bus synthetic grid, multi-split (k=8) topologies x 32 injections, full N-1",
    "g10k": "10k-bus synthetic grid, topologies x 64 injections, 3 splits, full N-1",
    "g1k_c": "1000-bus synthetic grid, 10^6 topologies over 8 GPUs (125,000 per GPU) x 128 injections, "
    "3 splits, full N-1, tasks drawn on the device",
}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 50 ms during the timed region."""

    Q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True,
            )
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def ready(self, timeout: float = 3.0) -> None:
        """Wait until nvidia-smi streams (its start-up takes a while), then drop what came
        before, so the samples cover the timed region."""
        t0 = time.perf_counter()
        while self.proc is not None and not self.lines and time.perf_counter() - t0 < timeout:
            time.sleep(0.01)
        self.lines.clear()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        # a timed region shorter than the sampling period: the first sample right after it
        after = False
        t0 = time.perf_counter()
        while not self.lines and time.perf_counter() - t0 < 0.5:
            after = True
            time.sleep(0.005)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[6]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        out = {
            "sm_mhz": statistics.median(sm) if sm else None,
            "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons),
            "samples": len(sm),
            "power_w_max": max(power) if power else None,
        }
        if after and sm:
            out["note"] = "timed region shorter than the 50 ms sampling period: first sample right after it"
        return out


def make_workload(name, rank, n_tasks=None, n_cand=None):
    from paper_2501_17529_b200 import synth

    spec, tasks, T, k, d = WORKLOADS[name]
    if n_tasks is not None:
        tasks = n_tasks
    if n_cand:
        T = n_cand
    grid = synth.make_grid(spec, seed=0)
    splits, discos, inj = synth.random_task_arrays(grid, tasks, T, k, seed=1000 + rank, n_disconnections=d)
    return grid, splits, discos, inj


# ---------------------------------------------------------------------------- CPU legs
def _port_worker(args):
    grid_doc, splits, discos, inj = args[:4]
    mode = args[4] if len(args) > 4 else "metric_first"
    from oracle import port
    from paper_2501_17529_b200.io import grid_from_dict
    from paper_2501_17529_b200.ptdf import prepare_base_ptdf
    from paper_2501_17529_b200.solver import SolveConfig

    grid = grid_from_dict(grid_doc)
    base = prepare_base_ptdf(grid)
    cfg = SolveConfig(mode=mode)
    canons = port.decode_arrays(grid, splits, discos, inj)
    t0 = time.perf_counter()
    lf = 0
    for c in canons:
        r = port.solve_one(grid, base, c, cfg)
        if r.feasible:
            lf += c.rows.shape[0] * (1 + r.n_feasible_cases)
    return lf, time.perf_counter() - t0, len(canons)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_port_rate(name, budget_s=12.0, cores=None, rank=0, mode="metric_first"):
    """The reference algorithm (oracle port, `mode`) on host cores; solve-only time."""
    import multiprocessing as mp

    from paper_2501_17529_b200 import synth
    from paper_2501_17529_b200.io import grid_to_dict

    spec, _tasks, T, k, d = WORKLOADS[name]
    cores = cores or os.cpu_count() or 1
    grid = synth.make_grid(spec, seed=0)
    doc = grid_to_dict(grid)
    # calibrate the per-task cost on one core, then size the sample to ~budget_s
    s, dd, i = synth.random_task_arrays(grid, 4, T, k, seed=77 + rank, n_disconnections=d)
    lf0, t_0, n0 = _port_worker((doc, s, dd, i, mode))
    per_task = max(t_0 / n0, 1e-4)
    n_total = int(max(cores, min(200000, budget_s * cores / per_task)))
    per = (n_total + cores - 1) // cores
    s, dd, i = synth.random_task_arrays(grid, per * cores, T, k, seed=99 + rank, n_disconnections=d)
    jobs = [(doc, s[c * per:(c + 1) * per], dd[c * per:(c + 1) * per], i[c * per:(c + 1) * per], mode)
            for c in range(cores)]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        res = pool.map(_port_worker, jobs)
    lf = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {
        "value": lf / wall,
        "unit": "loadflows/s",
        "cores": cores,
        "kind": "port",
        "sample": f"{per * cores} tasks of the {name} workload ({T} candidates, k={k}), {mode}, "
        f"{cores} processes x {per} tasks, solve-only wall {wall:.1f}s",
        "loadflows": lf,
        "cpu_model": cpu_model(),
        "mode": mode,
    }


def _check_worker(args):
    """Checker (test infrastructure): the oracle port on a few tasks of the timed batch."""
    grid_doc, splits, discos, inj, mine = args
    from oracle import port
    from paper_2501_17529_b200.io import grid_from_dict
    from paper_2501_17529_b200.ptdf import prepare_base_ptdf
    from paper_2501_17529_b200.solver import SolveConfig

    grid = grid_from_dict(grid_doc)
    base = prepare_base_ptdf(grid)
    cfg = SolveConfig(mode="metric_first")
    out = []
    for b, r in enumerate(port.solve_arrays(grid, base, splits, discos, inj, cfg)):
        tie = None
        if r.feasible and int(mine[b]) != r.best_injection:
            canon = port.decode_arrays(grid, splits[b:b + 1], discos[b:b + 1],
                                       inj[b:b + 1, [int(mine[b]), r.best_injection]])[0]
            m = port.evaluate(grid, base, canon, cfg)[0]
            tie = abs(float(m[0]) - float(m[1]))
        out.append((r.feasible, r.metric if r.feasible else float("nan"), r.best_injection if r.feasible else -1, tie))
    return out


def parity_sample(grid, splits, discos, inj, metric, best, feasible, n, cores=None):
    """Re-solve the first n tasks of the timed batch with the CPU oracle port and compare:
    feasibility, |metric - oracle| and best_injection agreement (a disagreement must be an
    FP64 tie of the two candidates, |m_a - m_b| <= 1e-12 max(1, metric))."""
    import multiprocessing as mp

    from paper_2501_17529_b200.io import grid_to_dict

    n = min(n, splits.shape[0])
    cores = max(1, min(cores or os.cpu_count() or 1, n))
    doc = grid_to_dict(grid)
    per = (n + cores - 1) // cores
    jobs = [(doc, splits[a:a + per], discos[a:a + per], inj[a:a + per], best[a:a + per]) for a in range(0, n, per)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(jobs)) as pool:
        res = [x for part in pool.map(_check_worker, jobs) for x in part]
    feas_ok = all(bool(feasible[b]) == res[b][0] for b in range(n))
    same = ties = bad = 0
    dmax = 0.0
    for b, (f, m, bi, tie) in enumerate(res):
        if not f:
            continue
        scale = max(1.0, abs(m))
        if int(best[b]) == bi:
            same += 1
            dmax = max(dmax, abs(float(metric[b]) - m) / scale)
        elif tie is not None and tie <= 1e-12 * scale:
            ties += 1
            dmax = max(dmax, abs(float(metric[b]) - m) / scale)
        else:
            bad += 1
    nf = sum(1 for r in res if r[0])
    return {
        "tasks": n,
        "feasible_match": feas_ok,
        "winner_identical": same,
        "winner_fp64_ties": ties,
        "winner_mismatch": bad,
        "feasible_tasks": nf,
        "max_rel_metric_diff": dmax,
        "oracle": "oracle/port.py (reference algorithm restated, metric_first), checker only",
        "wall_s": round(time.perf_counter() - t0, 1),
    }


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    steps = []
    last = None
    for it in range(args.warmup + args.steps):
        r = cpu_port_rate(args.config, budget_s=args.cpu_budget, rank=it)
        if it >= args.warmup:
            steps.append(r)
        last = r
    lf = sum(r["loadflows"] for r in steps)
    val = statistics.mean(r["value"] for r in steps)
    spec, tasks, T, k, d = WORKLOADS[args.config]
    line = {
        "impl": "reference",
        "metric": "DC loadflows/sec (topo x inj x N-1)",
        "value": val,
        "unit": "loadflows/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": None,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (scaled make_fixtures recipe, random_tasks semantics)",
        "config": {"workload": DESCR[args.config], "grid": spec, "candidates": T, "splits": k},
        "cpu_baseline": {k2: last[k2] for k2 in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": val, "unit": "loadflows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line["cpu_baseline"]["value"] = val
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- rooflines
def stage_rooflines(tb, splits, discos, fe, T, evaluated, stage_ms, report_cases, rescore_classes):
    """Algorithmic work of each device stage over its live
    CUDA-event time, against its bound: HBM bytes, tcgen05 TF32 flops, FP32 lane-ops or
    FP64 ops."""
    peaks, src = _peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    hbm = float(peaks.get("hbm_gbs", 6650.0)) * 1e9
    tf32 = float(peaks.get("bf16_tflops", 2250.0)) * 1e12 / 2.0  # dense TF32 = BF16 / 2
    alu = 148 * 128 * sm_mhz * 1e6
    f64 = 148 * 64 * sm_mhz * 1e6  # FP64 CUDA-core rate: half the FP32 lanes (B200 nominal)
    R, M, N1, C0 = tb.R, tb.M, tb.N1, tb.C0
    sp = splits.view(np.uint8).reshape(splits.shape[0], tb.S, -1).astype(bool)
    moved = sp.any(axis=2)                                   # (B, S) split substations
    k = moved.sum(axis=1)
    d = (discos >= 0).sum(axis=1) if discos.size else np.zeros(len(k), dtype=np.int64)
    r = (k + d)[fe].astype(np.float64)
    rbar = float(r.mean()) if len(r) else 0.0
    e_sum = (moved * np.asarray(tb.sub_count)[None, :]).sum(axis=1)[fe].astype(np.float64)
    kf, df = k[fe].astype(np.float64), d[fe].astype(np.float64)
    # every single case's outaged row monitored: s(c, t) is read from n0s, s32 is not written
    s_mon = bool(N1 == 0 or np.all(np.asarray(tb.row_mon_pos)[np.asarray(tb.sc_row)] >= 0))
    # update: touched FP64 rows / columns of P0 and the factors written (SURVEY 8(d) stage 1)
    upd = float((8 * (e_sum * C0 + (e_sum + kf) * R) + 8 * df * (C0 + 2 * R) + 4 * (R + C0 + N1) * r).sum())
    # N-0: n0/rating written (FP32; + s32 when an outaged row is unmonitored), B''/rating
    # (FP32 + FP64 copies) written, B'' and Y read
    n0w = M + (0 if s_mon else N1)
    n0b = float((4.0 * n0w * T + 12.0 * r * M + 8.0 * r * (R + T)).sum())
    # screening scales: the rank-r product per (monitored row, case) on the tensor cores
    scl = float((2.0 * M * N1 * r).sum())
    # N-1 single-branch: FFMA + FMNMX per monitored row of every evaluated (case, candidate)
    n1 = 2.0 * M * evaluated
    # winner report: per listed single case and monitored row, the rank-r D'' entry, the
    # LODF scale, the flow FMA and |F|/rating (r + 3 FP64 ops), plus the N-0 column (R r)
    rep = float(report_cases) * M * (rbar + 3.0) + float(len(r)) * R * rbar
    # FP64 re-score: per y-class the N-0 column on monitored rows (M r) and the one relevant
    # single case measured per class (M (2r + 3))
    rsc = float(rescore_classes) * M * (3.0 * rbar + 3.0)
    out = []

    def add(kernel, stage_keys, bound, work, peak, unit, what):
        ms = sum(stage_ms.get(s, 0.0) for s in stage_keys)
        if ms <= 0:
            return
        ach = work / (ms / 1e3)
        div = 1e9 if unit in ("GB/s", "Gop/s") else 1e12
        out.append({"kernel": kernel, "bound": bound, "achieved": ach / div, "peak": peak / div, "unit": unit,
                    "frac": ach / peak, "kernel_ms_per_step": ms, "work": what})

    add("k_update (split chain, outages, case factors; FP64)", ["update"], "hbm", upd, hbm, "GB/s",
        "8*sum_j(|E_j| C + (|E_j|+1) R) + 8 d (C + 2R) + 4 (R + C + N1)(k+d) bytes per task")
    add("k_n0 (N-0 contraction + screening data)", ["n0"], "hbm", n0b, hbm, "GB/s",
        f"4 {'M' if s_mon else '(M + N1)'} T + 12 (k+d) M + 8 (k+d)(R + T) bytes per task"
        + (" (s32 not written: every outaged row monitored)" if s_mon else ""))
    add("k_scale_tc (screening scales, tcgen05 TF32)", ["scale"], "tensor", scl, tf32, "TFLOP/s",
        f"2 M N1 (k+d) flops per task; peak = dense TF32 = BF16/2 ({src} MEASURED_PEAKS.json)")
    add("k_top + k_live + k_pairs (single-branch N-1, FFMA2/FMNMX3)", ["top", "screen"], "alu", n1, alu, "Gop/s",
        f"2 lane-ops (FFMA + FMNMX) per monitored row per evaluated (case, candidate); "
        f"peak = 148 SMs x 128 lanes x {sm_mhz:.0f} MHz")
    add("k_rsel + k_rsweep + k_rmerge (winner report, FP64)", ["report"], "fp64", rep, f64, "Gop/s",
        "listed cases x M x (k+d+3) + R (k+d) FP64 ops per task; peak = 148 SMs x 64 FP64 lanes x "
        f"{sm_mhz:.0f} MHz (nominal B200 FP64 = FP32 / 2)")
    add("k_select + k_rescore (first FP64 argmin of the near-tie band)", ["select"], "fp64", rsc, f64, "Gop/s",
        "y-classes x M x (3 (k+d) + 3) FP64 ops (N-0 column + one relevant single case per class)")
    return out


# ---------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    from paper_2501_17529_b200 import parallel
    from paper_2501_17529_b200.engine import STAGES
    from paper_2501_17529_b200.session import session_open, solve_batch_output

    spec, tasks, T, k, d = WORKLOADS[args.config]
    if args.tasks:
        tasks = args.tasks
    if args.candidates:
        T = args.candidates
    # the job's batch is ws * tasks topologies; this rank's shard (parallel.shard_range of
    # the concatenation) is drawn with its own seed, on the host (the reference's
    # generator semantics) or on the device (taskgen, bdc_draw_tasks)
    from paper_2501_17529_b200 import synth

    grid = synth.make_grid(spec, seed=0)
    sess = session_open(grid, device=local)
    eng = sess.engine
    eng.screen = not args.no_screen
    device_tasks = args.device_tasks or args.config in DEVICE_TASKS
    gen_s = None
    if device_tasks:
        from paper_2501_17529_b200.taskgen import random_tasks_device, to_host

        torch.cuda.synchronize()
        g0 = time.perf_counter()
        t_spl, t_dis, t_inj, draws = random_tasks_device(sess, tasks, T, k, 1000 + rank, n_disconnections=d)
        torch.cuda.synchronize()
        gen_s = time.perf_counter() - g0
        splits, discos, inj = to_host(t_spl, t_dis, t_inj)
    else:
        splits, discos, inj = synth.random_task_arrays(grid, tasks, T, k, seed=1000 + rank, n_disconnections=d)
        t_spl = torch.from_numpy(splits.view(np.uint8)).to(dev)
        t_dis = torch.from_numpy(discos).to(dev)
        t_inj = torch.from_numpy(inj.view(np.uint8)).to(dev)
    max_rank = eng.check_batch(splits.view(np.uint8), discos)
    B = splits.shape[0]
    kg = sess.config.topk_global
    ncw = max(1, (len(grid.contingencies) + 31) // 32)
    outs = {
        "metric": torch.empty(B, dtype=torch.float64, device=dev),
        "best": torch.empty(B, dtype=torch.int64, device=dev),
        "feasible": torch.empty(B, dtype=torch.uint8, device=dev),
        "status": torch.empty(B, dtype=torch.int32, device=dev),
        "status_arg": torch.empty(B, dtype=torch.int32, device=dev),
        "n_islanded": torch.empty(B, dtype=torch.int32, device=dev),
        "islanded_bits": torch.empty(B, ncw, dtype=torch.int32, device=dev),
        "n0_count": torch.empty(B, dtype=torch.int32, device=dev),
        "n0_pos": torch.empty(B, kg, dtype=torch.int32, device=dev),
        "n0_flow": torch.empty(B, kg, dtype=torch.float64, device=dev),
        "n0_rel": torch.empty(B, kg, dtype=torch.float64, device=dev),
        "n1_count": torch.empty(B, dtype=torch.int32, device=dev),
        "n1_case": torch.empty(B, kg, dtype=torch.int32, device=dev),
        "n1_pos": torch.empty(B, kg, dtype=torch.int32, device=dev),
        "n1_flow": torch.empty(B, kg, dtype=torch.float64, device=dev),
        "n1_rel": torch.empty(B, kg, dtype=torch.float64, device=dev),
    }
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    gathered = {}

    def step():
        r = eng.solve_device(t_spl, t_dis, t_inj, outs, stream.cuda_stream, max_rank)
        if ws > 1:
            # the per-topology results of every rank, all-gathered in HBM (NCCL over NVLink)
            gathered.update(parallel.all_gather_device(outs))
        return r

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    clocks.ready()
    elapsed_ms = 0.0
    pairs_eval = 0
    report_cases = 0
    rescore = [0, 0, 0]
    split_shared = 0
    lf_total = 0
    stage = [0.0] * len(STAGES)
    launches = 0
    waves = 0
    for _ in range(args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        st, wv, nl, lf = step()
        e1.record(stream)
        torch.cuda.synchronize()
        elapsed_ms += e0.elapsed_time(e1)
        lf_total += lf
        stage = [a + b for a, b in zip(stage, st)]
        launches += nl
        waves = wv
        pairs_eval += eng.last_pairs
        report_cases += eng.last_report_cases
        rescore = [a + b for a, b in zip(rescore, eng.last_rescore)]
        split_shared += eng.last_split_shared
    torch.cuda.synchronize()
    clk = clocks.stop()
    if ws > 1:
        dist.barrier()
        tt = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        lt = torch.tensor([lf_total], dtype=torch.float64, device=dev)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        elapsed_max, lf_all = float(tt.item()), float(lt.item())
    else:
        elapsed_max, lf_all = elapsed_ms, float(lf_total)
    value = lf_all / (elapsed_max / 1e3)
    # the timed batch's results (this rank's shard) for the parity sample
    res_metric = outs["metric"].cpu().numpy()
    res_best = outs["best"].cpu().numpy()
    res_feas = outs["feasible"].cpu().numpy().astype(bool)

    # ---- e2e: host pinned inputs -> public session API -> host outputs, wall clock
    pin_s = torch.from_numpy(splits).pin_memory().numpy()
    pin_d = torch.from_numpy(discos).pin_memory().numpy()
    pin_i = torch.from_numpy(inj).pin_memory().numpy()
    solver = parallel.engine_solver(sess)

    def e2e_call():
        if ws > 1:  # shard solve + all-gather of the results (parallel.solve_shard)
            full = parallel.solve_shard(pin_s, pin_d, pin_i, ws * B, solver, device=dev)
            return full["loadflows"], None
        o = solve_batch_output(sess, pin_s, pin_d, pin_i)
        return o.loadflows, o

    e2e_call()  # warm
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e2e_s = 0.0
    e2e_lf = 0
    n_e2e = max(1, min(args.steps, 3))
    out = None
    for _ in range(n_e2e):
        t0 = time.perf_counter()
        lf_i, o = e2e_call()
        e2e_s += time.perf_counter() - t0
        e2e_lf += lf_i
        out = o or out
    if ws > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())  # e2e_lf is already the job-wide total (solve_shard)
    e2e_val = e2e_lf / e2e_s
    h2d = splits.nbytes + discos.nbytes + inj.nbytes
    # report loadings (n0_rel, n1_rel) are recomputed on the host as |flow| / rating
    res_names = ("metric", "best", "feasible", "status", "status_arg", "n_islanded", "islanded_bits",
                 "n0_count", "n0_pos", "n0_flow", "n1_count", "n1_case", "n1_pos", "n1_flow")
    d2h = sum(int(outs[n].numel() * outs[n].element_size()) for n in res_names)
    if ws > 1:
        # solve_shard: the local results go up for the gather and the full batch comes back
        fields = parallel.RESULT_FIELDS
        local_bytes = sum(int(outs[n].numel() * outs[n].element_size()) for n in fields)
        h2d += local_bytes
        d2h = local_bytes + ws * local_bytes

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return

    # ---- per-stage rooflines, kernel times live from the engine's CUDA events
    tb = eng.tables
    fe = res_feas
    single_orders = set(int(x) for x in tb.sc_order)
    isl_single = np.zeros(B, dtype=np.int64)
    if out is None:
        out = solve_batch_output(sess, pin_s, pin_d, pin_i)
    for b in np.flatnonzero(out.n_islanded > 0):
        isl_single[b] = sum(1 for o in out.islanded_orders(int(b)) if o in single_orders)
    pairs = float(((tb.N1 - isl_single) * fe).sum()) * T  # feasible (case, candidate) pairs per step
    evaluated = pairs_eval / args.steps  # pairs the N-1 kernels actually evaluated (screen on)
    stage_ms = {n: v / args.steps for n, v in zip(STAGES, stage)}
    roof = stage_rooflines(tb, splits, discos, fe, T, evaluated, stage_ms, report_cases / args.steps,
                           rescore[0] / args.steps)
    dom = max(roof, key=lambda r: r["kernel_ms_per_step"])  # the longest stage with a roofline
    # DRAM bytes per launch (ncu --set full, per task, scaled to this launch size) of every
    # stage's kernels, where profiles/kernel_traffic.json has them for this config
    tj = {}
    tp = os.path.join(REPO, "profiles", "kernel_traffic.json")
    if os.path.exists(tp):
        try:
            with open(tp) as fh:
                tj = json.load(fh).get(args.config, {})
        except (OSError, ValueError):
            tj = {}
    for r in roof:
        per_task = tj.get(r["kernel"].split()[0])
        r["traffic"] = per_task * B / max(1, waves) if per_task else None
    roofline = dict(dom)
    step_ms = elapsed_max / args.steps
    line = {
        "metric": "DC loadflows/sec (topo x inj x N-1)",
        "value": value,
        "unit": "loadflows/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32 N-1 scan / f64 updates, winner (FP64 argmin of the near-tie band) and report",
        "data": "synthetic (scaled make_fixtures recipe, random_tasks semantics, seeded per rank)",
        "config": {
            "workload": DESCR[args.config],
            "grid": spec,
            "tasks_per_gpu": int(B),
            "tasks_total": int(B) * ws,
            "candidates": T,
            "splits": k,
            "disconnections": d,
            "rows": tb.R,
            "monitored": tb.M,
            "cases": len(grid.contingencies),
            "parallelism": f"topology-sharded dp{ws}"
            + (" (no collective in the solve; per-topology results all-gathered over NCCL inside the timed step)" if ws > 1 else ""),
            "l2": "flushed between steps (256 MB write, outside the timed events)",
        },
        "e2e": {"value": e2e_val, "unit": "loadflows/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "how": ("session API solve_batch_output" if ws == 1 else "parallel.solve_shard (session engine + all-gather)")
                + ", pinned host arrays in, host arrays out, wall clock, max over ranks"},
        "roofline": roofline,
        "stages_roofline": roof,
        "stage_ms_per_step": stage_ms,
        "screen": {
            "enabled": bool(eng.screen),
            "pairs_total": pairs,
            "pairs_evaluated": evaluated,
            "skipped_frac": (1.0 - evaluated / pairs) if pairs else 0.0,
            "report_cases_per_task": report_cases / args.steps / max(1, B),
            "note": "exact dominance screen of the reference's metric_first mode (solver.py:798-822); "
            "the metric is unchanged, skipped pairs are provably dominated",
        },
        "rescore": {
            "classes_per_step": rescore[0] / args.steps,
            "winners_replaced_per_step": rescore[1] / args.steps,
            "tasks_with_band_per_step": rescore[2] / args.steps,
            "note": "FP64 re-score of every candidate within 2 RESCORE_EPS of the FP32 minimum, grouped by "
            "bitwise-equal rank coefficients (k_rescore); best_injection = first FP64 argmin",
        },
        "tasks": {"generated_on": "device (taskgen.random_tasks_device, bdc_draw_tasks)" if device_tasks else
                  "host (synth.random_task_arrays)", "generate_s": gen_s},
        "split_chain": {
            "applications_per_step": float(((np.asarray(splits).reshape(B, -1, splits.shape[-1]).any(axis=2)).sum())),
            "shared_per_step": split_shared / args.steps,
            "note": "split applications copied from another task of the wave with the same canonical prefix "
            "(k_update prefix memo, levels < 2; tree.py:50-113) instead of computed",
        },
        "gpu_launches": int(launches),
        "clocks": clk,
        "loadflows_per_step": lf_all / args.steps,
        "feasible_tasks": int(fe.sum()),
    }
    if args.check < 0:
        args.check = {"g14": 64, "g118": 64, "g1k": 32, "g1k_c": 32, "g3k": 16, "g10k": 4}.get(args.config, 8)
    if args.check > 0:
        try:
            line["parity_sample"] = parity_sample(grid, splits, discos, inj, res_metric, res_best, res_feas, args.check)
        except Exception as exc:  # reported, never fatal
            line["parity_sample"] = {"error": str(exc)}
    if ws == 1 and not args.no_cpu:
        try:
            cb = cpu_port_rate(args.config, budget_s=args.cpu_budget)
            line["cpu_baseline"] = {k2: cb[k2] for k2 in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
            sym = cpu_port_rate(args.config, budget_s=args.cpu_budget / 2, mode="symmetric")
            line["cpu_baseline"]["symmetric"] = {
                "value": sym["value"], "sample": sym["sample"],
                "note": "the reference's brute-force-equivalent mode (every pair evaluated)"}
        except Exception as exc:  # the baseline is reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "loadflows/s", "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def _self_launch(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: launch N ranks (one per GPU)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="g118", choices=sorted(WORKLOADS))
    ap.add_argument("--tasks", type=int, default=0, help="override tasks per GPU per step")
    ap.add_argument("--candidates", type=int, default=0, help="override injection candidates per task")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-screen", action="store_true", help="brute-force every (case, candidate) pair")
    ap.add_argument("--device-tasks", action="store_true", help="draw the tasks on the GPU (taskgen)")
    ap.add_argument("--check", type=int, default=-1,
                    help="re-solve this many tasks of the timed batch with the CPU oracle (parity_sample); "
                    "0 = off, -1 = by grid size (64 at G14/G118 ... 4 at G10k)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
