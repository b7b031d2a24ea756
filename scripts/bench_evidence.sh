#!/bin/bash
# Light round evidence in one GPU call: GPU tests, bench lines of every config (G118 with
# the CPU baseline) and ncu launch lists of G118 / G1k (no --set full captures).
#   usage: bash scripts/bench_evidence.sh <tag>
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT/tmp
S=$OUT/summary_${TAG}.md; : > $S
timeout 500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for C in g118 g1k g3k g14 g10k g1k_c; do
  if [ $C = g118 ]; then timeout 900 python bench.py --config $C 2>&1 | tail -1 > $OUT/bench_${C}_${TAG}.json
  else timeout 900 python bench.py --config $C --no-cpu 2>&1 | tail -1 > $OUT/bench_${C}_${TAG}.json; fi
  python -c "
import json; d=json.load(open('$OUT/bench_${C}_${TAG}.json')); print('$C', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], round(d['ms_per_step'],2), d['roofline']['kernel'][:20], round(d['roofline']['frac'],4), d['clocks'])"
done
declare -A TASKS=([g118]=16384 [g1k]=2048)
for CFG in g118 g1k; do
  N=${TASKS[$CFG]}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu \
      > $OUT/tmp/l_${CFG}.log 2>&1
  python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv >> $S
done
rm -rf $OUT/tmp
