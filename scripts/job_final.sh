set -u
mkdir -p gpurun_out/tmp
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for C in g118 g1k g3k g14 g10k; do
  if [ $C = g118 ]; then timeout 900 python bench.py --config $C 2>&1 | tail -1 > gpurun_out/bench_${C}_r1g.json
  else timeout 900 python bench.py --config $C --no-cpu 2>&1 | tail -1 > gpurun_out/bench_${C}_r1g.json; fi
  python -c "
import json; d=json.load(open('gpurun_out/bench_${C}_r1g.json')); print('$C', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], round(d['ms_per_step'],2), d['roofline']['kernel'][:20], round(d['roofline']['frac'],4), d.get('cpu_baseline',{}).get('value'))"
done
declare -A TASKS=([g14]=1024 [g118]=16384 [g1k]=2048 [g3k]=512)
cap() {
  local K=$1 CFG=$2 N=${TASKS[$2]}
  local R=gpurun_out/tmp/p_${CFG}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 1 -c 1 \
      -o $R -f python bench.py --config $CFG --tasks $N --steps 1 --warmup 1 --no-cpu > gpurun_out/tmp/n.log 2>&1
  echo "#### capture $K $CFG ($N tasks)" >> gpurun_out/summary_r1g_b.md
  python profiles/summarize.py $R.ncu-rep >> gpurun_out/summary_r1g_b.md
  python profiles/summarize.py --source $R.ncu-rep >> gpurun_out/summary_r1g_b.md 2>&1
}
cap "^k_top$" g118
cap "^k_top$" g1k
cap "^k_top$" g3k
cap "k_scale_tc" g118
cap "k_live" g118
cap "k_pairs" g1k
cap "k_pairs" g3k
cap "k_terms" g1k
cap "k_update" g3k
cap "k_terms" g3k
cap "k_n0" g3k
rm -rf gpurun_out/tmp
