mkdir -p gpurun_out
OLD=$PWD/scratch/oldlib/libddf_b200.so
for rep in 1 2; do
  DDF_B200_LIB=$OLD timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/old /'
  timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/new /'
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu12.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu12.log
for lib in old new old new; do
  if [ $lib = old ]; then export DDF_B200_LIB=$OLD; else unset DDF_B200_LIB; fi
  timeout 600 python bench.py --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab8_c4_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab8_c4_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib c4', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms', 'mlp', round(r['achieved']), {k: round(v['tflops']) for k, v in r.items() if isinstance(v, dict) and v.get('tflops')}, d['clocks']['sm_mhz'])"
done
