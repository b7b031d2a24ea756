#!/bin/bash
# One kernel, one config: launch list + --set full capture summarised on the box.
#   usage: bash scripts/ncu_one.sh <tag> <kernel-regex> <config> [tasks]
set -u
TAG=$1; K=$2; CFG=$3; N=${4:-2048}
OUT=gpurun_out; mkdir -p $OUT/tmp
CMD="python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_${CFG}_${TAG}.csv $CMD > $OUT/tmp/l.log 2>&1
python profiles/summarize.py --launches $OUT/launches_${CFG}_${TAG}.csv >> $OUT/summary_${TAG}.md
for KK in $K; do
  R=$OUT/tmp/prof_${KK}_${CFG}_${TAG}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KK -s 1 -c 1 \
      -o $R -f $CMD > $OUT/tmp/n.log 2>&1
  python profiles/summarize.py $R.ncu-rep >> $OUT/summary_${TAG}.md
  python profiles/summarize.py --source $R.ncu-rep >> $OUT/summary_${TAG}.md 2>&1
  mv $R.ncu-rep $OUT/ 2>/dev/null
done
rm -rf $OUT/tmp; ls -la $OUT | tail -5
