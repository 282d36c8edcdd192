# Session-7 bench lines for every config on one B200 (current build).
mkdir -p gpurun_out
for c in c1 c2 c3 c5 udf bvh march modes; do
  timeout 900 python bench.py --config $c > gpurun_out/all7_$c.json 2> gpurun_out/all7_$c.err; echo "$c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/all7_$c.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}
print('$c', d['metric'], round(d['value']/1e6,3), 'M', d['unit'], 'ms', round(d['ms_per_step'],3), 'frac', r.get('frac'), 'e2e', (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1
done
