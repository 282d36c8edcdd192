# A/B on one box: scratch/oldlib (HEAD before the change) vs the in-tree build
mkdir -p gpurun_out
OLD=$PWD/scratch/oldlib/libddf_b200.so
for rep in 1 2; do
  DDF_B200_LIB=$OLD timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 2097152 | sed 's/^/old /'
  timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 2097152 | sed 's/^/new /'
done
STATS=1 timeout 120 python scratch/smem_exp.py "(65,)+(512,)*8+(1,)" 2097152
for lib in old new; do
  if [ $lib = old ]; then export DDF_B200_LIB=$OLD; else unset DDF_B200_LIB; fi
  timeout 600 python bench.py --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab_c4_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab_c4_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib c4', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms', 'fwd', round(r['forward']['tflops']), 'grad', round(r['gradient']['tflops']), 'fused', round(r['fused_trace_gradient']['tflops']), d['clocks']['sm_mhz'])"
done
