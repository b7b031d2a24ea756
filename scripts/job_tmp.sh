set -u
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
bash scripts/gpu_test_bench.sh "g118 g1k" skip
bash scripts/launches.sh rs4 g118 2>&1 | grep -E "k_rs|launch list"
