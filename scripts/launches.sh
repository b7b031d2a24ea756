#!/bin/bash
# ncu launch lists (per-kernel device time, serialised) for the given configs.
#   usage: bash scripts/launches.sh <tag> <configs...>
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
declare -A TASKS=([g14]=1024 [g118]=16384 [g1k]=2048 [g3k]=512 [g10k]=32)
for CFG in "$@"; do
  N=${TASKS[$CFG]}
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
  python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv
done
