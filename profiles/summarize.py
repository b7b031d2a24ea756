#!/usr/bin/env python3
"""Summarise ncu captures (run here, on the CPU box, on reports brought back in gpurun_out/).

    python profiles/summarize.py gpurun_out/prof_k_single_g1k_r1.ncu-rep [...] > profiles/xxx.md
    python profiles/summarize.py --launches gpurun_out/launches_g118_r1.csv

Prints the metrics the roofline and the optimisation notes rely on: duration,
DRAM bytes, issue/pipe utilisation, occupancy, top stall reasons.
"""

import csv
import io
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(path):
    h, units, data = raw(path)
    print(f"### {path.split('/')[-1]}\n")
    for d in data:
        name = d[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"kernel `{name[:90]}`\n")
        print("| metric | value |\n|---|---|")
        for k, label in KEYS:
            if k in h:
                i = h.index(k)
                print(f"| {label} | {d[i]} {units[i]} |")
        st = [(h[i], d[i]) for i in range(len(h))
              if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:5]
        print("| top stalls (per issue) | " + ", ".join(
            f"{a.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')} {float(b):.2f}"
            for a, b in st) + " |\n")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault(d["Kernel Name"].split("(")[0][:60], []).append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    print(f"### launch list {path.split('/')[-1]} (ncu, cold-cache, serialised)\n")
    print("| kernel | launches | mean us | share |\n|---|---|---|---|")
    for k, v in agg.items():
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")
    print()


def source(path, top=25):
    """Top CUDA source lines by warp-stall samples, per captured kernel
    (needs -lineinfo at compile time and --import-source on at capture)."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    per_fn = OrderedDict()
    fn, fpath, hdr = "?", "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path":
            fpath = r[1].split("/")[-1]
            continue
        if r[0] == "Function Name":
            fn = r[1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or r[2] != "-":
            continue  # SASS rows carry an address; line aggregates carry "-"
        try:
            v = float(r[4] or 0)
        except ValueError:
            continue
        if v > 0:
            per_fn.setdefault(fn, []).append((v, f"{fpath}:{r[0]}", r[1].strip()[:100]))
    for fn, data in per_fn.items():
        tot = sum(d[0] for d in data) or 1.0
        print(f"#### hot source lines of `{fn[:110]}` ({path.split('/')[-1]}, share of warp-stall samples)\n")
        print("| share | line | source |\n|---|---|---|")
        for v, ln, src in sorted(data, key=lambda x: -x[0])[:top]:
            print(f"| {v / tot * 100:.1f}% | {ln} | `{src.replace('|', '/')}` |")
        print()


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--source":
        for p in args[1:]:
            source(p)
    elif args and args[0] == "--launches":
        for p in args[1:]:
            launches(p)
    else:
        for p in args:
            summarize(p)
