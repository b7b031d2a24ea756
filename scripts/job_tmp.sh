BDC_PTOP=16 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for C in g118 g1k g3k; do
for P in 0 8 16 32; do
BDC_PTOP=$P timeout 600 python bench.py --config $C --no-cpu --steps 3 --warmup 3 2>&1 | tail -1 > gpurun_out/b.json
python -c "
import json; d=json.load(open('gpurun_out/b.json')); st={k: round(v,2) for k,v in d['stage_ms_per_step'].items()}
print('$C $P', '%.3e'%d['value'], round(d['ms_per_step'],2), 'skip=%.3f'%d['screen']['skipped_frac'], st)"
done; done
