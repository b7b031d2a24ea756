#!/bin/bash
# Round check under gpurun: parity tests, smoke, default bench (with CPU baseline), short benches.
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench_default.json
tail -c 3000 gpurun_out/bench_default.json
bash scripts/gpu_test_bench.sh "${1:-g1k g3k}" skip
