set -u
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_test_bench.sh "g118 g1k g3k" skip
bash scripts/launches.sh tp g118 g1k g3k 2>&1 | grep -E "k_top<|k_pairs|launch list"
