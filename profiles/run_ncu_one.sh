#!/bin/bash
# One `ncu --set full` capture of one kernel of one bench config (run under gpurun).
#   usage: bash profiles/run_ncu_one.sh <kernel-regex> <config> <tasks> <tag>
set -u
K=$1; CFG=$2; TASKS=$3; TAG=$4
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof_${K}_${CFG}_${TAG} -f \
    python bench.py --config $CFG --tasks $TASKS --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_${K}_${CFG}_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_${K}_${CFG}_${TAG}.log
