timeout 180 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
bash scripts/gpu_test_bench.sh "g118 g1k g3k" skip
bash scripts/launches.sh tc1 g118 g1k g3k
