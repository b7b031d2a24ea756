set -u
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
bash scripts/gpu_test_bench.sh "g118 g1k g3k g10k" skip
bash scripts/launches.sh sc g118 g3k 2>&1 | grep -E "k_scale|launch list"
