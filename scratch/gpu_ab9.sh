# A/B: production lib vs the DDF_EXP_NOBIAS timing build (bias add dropped;
# the configs' biases are zero, so results are unchanged)
mkdir -p gpurun_out
EXP=$PWD/scratch/explib/libddf_b200.so
for rep in 1 2; do
  timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/base /'
  DDF_B200_LIB=$EXP timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/nobias /'
done
for lib in base exp base exp; do
  if [ $lib = exp ]; then export DDF_B200_LIB=$EXP; else unset DDF_B200_LIB; fi
  timeout 600 python bench.py --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab9_c4_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab9_c4_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib c4', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms', 'mlp', round(r['achieved']), {k: round(v['tflops']) for k, v in r.items() if isinstance(v, dict) and v.get('tflops')}, d['clocks']['sm_mhz'])"
done
