# Session-7 validation on one B200: GPU tests, smoke, default bench, reference
# arm, and the c4 pilot-balanced split (pilot time + per-rank rows).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/f7_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f7_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/f7_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/f7_smoke.log
timeout 600 python bench.py > gpurun_out/f7_bench.json 2> gpurun_out/f7_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/f7_ref.json 2> gpurun_out/f7_ref.err; echo "ref rc=$?"
timeout 400 python scratch/rank_balance.py c4 2 pilot > gpurun_out/f7_c4_pilot.log 2>&1; echo "balance rc=$?"; grep pilot gpurun_out/f7_c4_pilot.log | head -1
python -c "
import json; d=json.loads(open('gpurun_out/f7_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print('c4', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms e2e', round(d['e2e']['value']/1e6,2), 'mlp', round(r['achieved']), round(r['frac'],3), d['clocks'])
d=json.loads(open('gpurun_out/f7_ref.json').read().strip().splitlines()[-1]); print('ref', d['value'], d['cpu_baseline']['cores'])"
