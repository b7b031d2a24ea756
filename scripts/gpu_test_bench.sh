#!/bin/bash
# parity tests + short benches (run under gpurun)
#   usage: bash scripts/gpu_test_bench.sh "<configs>" [pytest -k expr]
set -u
CFGS=${1:-g1k}
mkdir -p gpurun_out
[ "${2:-}" = skip ] || timeout 900 python -m pytest tests -m gpu -x -q ${2:+-k "$2"} 2>&1 | tail -15
for C in $CFGS; do
  timeout 600 python bench.py --config $C --no-cpu --check ${CHECK:-0} --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_$C.json
  python - "$C" <<'PY'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{c}.json").read())
except Exception as e:
    print(c, "FAILED", open(f"gpurun_out/bench_{c}.json").read()[-2000:]); sys.exit()
st = {k: round(v, 2) for k, v in d["stage_ms_per_step"].items()}
print(c, f"value={d['value']:.3e} e2e={d['e2e']['value']:.3e} ms/step={d['ms_per_step']:.2f} roof={d['roofline']['kernel'].split()[0]} frac={d['roofline']['frac']:.3f} skip={d['screen']['skipped_frac']:.3f} rcases={d['screen'].get('report_cases_per_task', -1):.1f}", st)
print("   fracs", {r['kernel'].split()[0]: round(r['frac'], 3) for r in d['stages_roofline']}, d.get('parity_sample', ''))
PY
done
