#!/bin/bash
# ncu launch lists + --set full captures of the engine kernels, summarised ON the
# box (gpurun only brings back <= 64 MiB).  Run under gpurun, 1 GPU.
#   usage: bash scripts/profile_job.sh <tag> <keep-regex> <full-configs> [launch-list configs...]
set -u
TAG=$1; KEEP=$2; FULL=$3; shift 3
CFGS=${@:-g118 g1k g3k}
OUT=gpurun_out; mkdir -p $OUT/tmp
declare -A TASKS=([g14]=1024 [g118]=16384 [g1k]=2048 [g3k]=512 [g10k]=32)
for CFG in $CFGS; do
  N=${TASKS[$CFG]}
  CMD="python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_${TAG}.csv $CMD > $OUT/tmp/ncu_launch_${CFG}.log 2>&1
  python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv >> $OUT/summary_${TAG}.md
  echo " $FULL " | grep -q " $CFG " || continue
  for K in k_single k_scale k_update k_n0 k_other k_rsel k_rsweep; do
    R=$OUT/tmp/prof_${K}_${CFG}_${TAG}
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 3 \
        -o $R -f $CMD > $OUT/tmp/ncu_${K}_${CFG}.log 2>&1
    python profiles/summarize.py $R.ncu-rep >> $OUT/summary_${TAG}.md
    python profiles/summarize.py --source $R.ncu-rep >> $OUT/summary_${TAG}.md 2>&1
    if echo "${K}_${CFG}" | grep -Eq "$KEEP"; then mv $R.ncu-rep $OUT/; fi
  done
done
rm -rf $OUT/tmp
du -sh $OUT; ls -la $OUT
