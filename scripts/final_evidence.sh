#!/bin/bash
# Round evidence in one GPU call: GPU tests, bench lines of every config (G118 with the CPU
# baseline), ncu launch lists, and --set full captures of every kernel behind a roofline
# stage plus the report kernels, summarised on the box.  1 GPU.
#   usage: bash scripts/final_evidence.sh <tag>
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT/tmp
S=$OUT/summary_${TAG}.md; : > $S
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for C in g118 g1k g3k g14 g10k g1k_c; do
  if [ $C = g118 ]; then timeout 900 python bench.py --config $C 2>&1 | tail -1 > $OUT/bench_${C}_${TAG}.json
  else timeout 900 python bench.py --config $C --no-cpu 2>&1 | tail -1 > $OUT/bench_${C}_${TAG}.json; fi
  python -c "
import json; d=json.load(open('$OUT/bench_${C}_${TAG}.json')); print('$C', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], round(d['ms_per_step'],2), d['roofline']['kernel'][:20], round(d['roofline']['frac'],4), d.get('cpu_baseline',{}).get('value'))"
done
# brute force (every (case, candidate) pair; BASELINE.md 3 / VERDICT r1 item 3)
for C in g118 g1k; do
  timeout 900 python bench.py --config $C --no-cpu --no-screen --check 8 2>&1 | tail -1 > $OUT/bench_${C}_noscreen_${TAG}.json
  python -c "
import json; d=json.load(open('$OUT/bench_${C}_noscreen_${TAG}.json')); print('$C no-screen', '%.3e'%d['value'], round(d['ms_per_step'],2))"
done
declare -A TASKS=([g14]=1024 [g118]=16384 [g1k]=2048 [g3k]=512)
for CFG in g14 g118 g1k g3k; do
  N=${TASKS[$CFG]}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu \
      > $OUT/tmp/l_${CFG}.log 2>&1
  python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv >> $S
done
cap() {  # cap <kernel regex> <config>
  local K=$1 CFG=$2 N=${TASKS[$2]}
  local R=$OUT/tmp/p
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 1 -c 1 \
      -o $R -f python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu > $OUT/tmp/n.log 2>&1
  echo "#### capture $K $CFG ($N tasks)" >> $S
  python profiles/summarize.py $R.ncu-rep >> $S
  python profiles/summarize.py --source $R.ncu-rep >> $S 2>&1
}
for CFG in g118 g1k g3k; do
  for K in "k_update" "k_terms" "k_n0" "k_scale_tc" "^k_top$" "k_live" "k_pairs" "k_oscreen" "k_other" "k_rescore" "k_oexact" "k_rsel" "k_rsweep"; do
    cap "$K" $CFG
  done
done
rm -rf $OUT/tmp
du -sh $OUT
