# bench.py on every BASELINE config (run under gpurun): one JSON line each.
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for c in c1 c5 c3 c4; do
  timeout 1500 python bench.py --config $c --steps 2 --warmup 3 > gpurun_out/bench_$c.log 2>&1
  tail -1 gpurun_out/bench_$c.log >> gpurun_out/configs.jsonl
  python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1])
  print('$c', d['value'], d['unit'], 'e2e', d['e2e']['value'], 'ms/step', d['ms_per_step'], 'its', d['config'].get('batch_iterations'), 'cpu', (d.get('cpu_baseline') or {}).get('value'), 'frac', (d.get('roofline') or {}).get('frac'))
except Exception as e: print('$c failed', e)
"
done
