#!/bin/bash
# One GPU call during development: the GPU tests (optionally a -k filter), then bench lines
# of the given configs with the stage breakdown.   usage: bash scripts/quick_gpu.sh "<pytest -k expr or ->" cfg...
K=$1; shift
mkdir -p gpurun_out
if [ "$K" != "-" ]; then
  if [ "$K" = "all" ]; then timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
  else timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -4; fi
fi
for C in "$@"; do
  timeout 300 python bench.py --config $C --no-cpu 2>&1 | tail -1 > gpurun_out/q_$C.json
  python -c "
import json; d=json.load(open('gpurun_out/q_$C.json')); print('$C', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stage_ms_per_step'].items()}, d.get('parity_sample'))" 2>&1 | tail -2
done
