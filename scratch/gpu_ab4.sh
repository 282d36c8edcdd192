mkdir -p gpurun_out
for rep in 1 2; do
  DDF_SPLIT2=1 timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/split2 /'
  timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/split4 /'
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu8.log
for v in split2 split4; do
  if [ $v = split2 ]; then export DDF_SPLIT2=1; else unset DDF_SPLIT2; fi
  timeout 600 python bench.py --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab4_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab4_c4_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$v c4', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms', 'mlp', round(r['achieved']), d['clocks']['sm_mhz'])"
done
