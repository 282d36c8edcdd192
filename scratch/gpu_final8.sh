# Session-7 end state: smoke, default bench (c4), c5/udf/c3 lines.
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f8_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/f8_smoke.log
timeout 600 python bench.py > gpurun_out/f8_c4.json 2> gpurun_out/f8_c4.err; echo "c4 rc=$?"
for c in c3 c5 udf; do timeout 600 python bench.py --config $c > gpurun_out/f8_$c.json 2> gpurun_out/f8_$c.err; echo "$c rc=$?"; done
for c in c4 c3 c5 udf; do python -c "
import json; d=json.loads(open('gpurun_out/f8_$c.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$c', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), 'ms e2e', round(d['e2e']['value']/1e6,3), 'mlp', round(r['achieved']), round(r['frac'],3), 'cmp', (r.get('compaction') or {}).get('ms'), d['gpu_launches'], d['clocks'])"; done
