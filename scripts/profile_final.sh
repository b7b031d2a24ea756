#!/bin/bash
# Round evidence: ncu launch lists of every config and --set full captures of the main
# kernels, summarised on the box (gpurun brings back <= 64 MiB).  1 GPU.
#   usage: bash scripts/profile_final.sh <tag>
set -u
TAG=$1
OUT=gpurun_out; mkdir -p $OUT/tmp
declare -A TASKS=([g14]=1024 [g118]=16384 [g1k]=2048 [g3k]=512 [g10k]=16)
for CFG in g14 g118 g1k g3k; do
  N=${TASKS[$CFG]}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu \
      > $OUT/tmp/l_${CFG}.log 2>&1
  python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv >> $OUT/summary_${TAG}.md
done
cap() {  # cap <kernel regex> <config> <keep 0|1>
  local K=$1 CFG=$2 KEEP=$3 N=${TASKS[$2]}
  local R=$OUT/tmp/prof_${K}_${CFG}_${TAG}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 \
      -o $R -f python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu > $OUT/tmp/n.log 2>&1
  echo "#### capture $K $CFG ($N tasks)" >> $OUT/summary_${TAG}.md
  python profiles/summarize.py $R.ncu-rep >> $OUT/summary_${TAG}.md
  python profiles/summarize.py --source $R.ncu-rep >> $OUT/summary_${TAG}.md 2>&1
  if [ "$KEEP" = 1 ]; then mv $R.ncu-rep $OUT/; fi
}
cap k_scale_tc g1k 1
cap k_scale_tc g3k 0
cap "k_update" g118 0
cap "k_terms" g118 0
cap "k_n0" g118 0
cap "^k_top$" g1k 1
cap "^k_top$" g118 0
cap "k_pairs" g118 0
cap "k_live" g1k 0
cap "k_other" g1k 0
cap "k_rsel_w" g118 0
cap "k_rsweep" g118 0
cap "k_rsweep" g1k 0
cap "k_update" g1k 0
cap "k_n0" g1k 0
rm -rf $OUT/tmp
du -sh $OUT; ls -la $OUT | tail -20
