set -u
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash scripts/gpu_test_bench.sh "g3k" skip
