"""Build libbdc.so in-tree for sm_100a (nvcc; no JIT cache, so it travels with the repo)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = ["bdc_update.cu", "bdc_single.cu", "bdc_scale.cu", "bdc_flows.cu", "bdc_report.cu", "bdc_gen.cu",
           "bdc_chol.cu", "bdc_capi.cu"]
TARGET = os.path.join(HERE, "libbdc.so")
FLAGS = [
    "-std=c++17",
    "-O3",
    "-lineinfo",
    "-gencode",
    "arch=compute_100a,code=sm_100a",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-O3",
]
OBJDIR = os.path.join(HERE, "build")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not os.path.exists(TARGET):
        return True
    t = os.path.getmtime(TARGET)
    deps = [os.path.join(HERE, "csrc", s) for s in SOURCES + ["bdc_device.cuh"]]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "bdc.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return TARGET
    # one nvcc per translation unit, in parallel, then one link
    os.makedirs(OBJDIR, exist_ok=True)
    procs = []
    objs = []
    headers = [os.path.join(HERE, "csrc", "bdc_device.cuh"), os.path.join(os.path.dirname(HERE), "include", "bdc.h")]
    hdr_t = max(os.path.getmtime(h) for h in headers)
    for src in SOURCES:
        obj = os.path.join(OBJDIR, src.replace(".cu", ".o"))
        path = os.path.join(HERE, "csrc", src)
        objs.append(obj)
        # incremental unless forced: a unit is rebuilt when it or a shared header is newer
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(path), hdr_t):
            continue
        cmd = [nvcc()] + FLAGS + ["-c", "-o", obj, path]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed on {failed}")
    tmp = TARGET + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp] + objs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, TARGET)
    return TARGET


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
