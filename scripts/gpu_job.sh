set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
cat MEASURED_PEAKS.json 2>/dev/null; mkdir -p gpurun_out; cp MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py 2>&1 | tail -2 > gpurun_out/bench_g118.log
timeout 600 python bench.py --config g1k --no-cpu 2>&1 | tail -2 > gpurun_out/bench_g1k.log
timeout 600 python bench.py --config g3k --no-cpu 2>&1 | tail -2 > gpurun_out/bench_g3k.log
cat gpurun_out/bench_*.log
