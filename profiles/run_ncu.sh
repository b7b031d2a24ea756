#!/bin/bash
# Profiling recipe (run under gpurun on one B200): launch list of one bench
# command + one `ncu --set full` capture of each engine kernel.
#   usage: bash profiles/run_ncu.sh <config> <tasks> <tag>
set -u
CFG=${1:-g118}; TASKS=${2:-16384}; TAG=${3:-r1}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --config $CFG --tasks $TASKS --steps 2 --warmup 1 --no-cpu"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
    --log-file $OUT/launches_${CFG}_${TAG}.csv $CMD > $OUT/ncu_launch_${CFG}_${TAG}.log 2>&1
for K in k_single k_update k_report k_other; do
  ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
      -o $OUT/prof_${K}_${CFG}_${TAG} -f $CMD > $OUT/ncu_${K}_${CFG}_${TAG}.log 2>&1
done
ls $OUT
