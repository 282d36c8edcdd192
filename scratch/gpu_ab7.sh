mkdir -p gpurun_out
OLD=$PWD/scratch/oldlib/libddf_b200.so
for rep in 1 2; do
  DDF_B200_LIB=$OLD timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/old /'
  timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 4194304 | sed 's/^/new /'
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu11.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu11.log
for cfg in c4 c3; do
for lib in old new; do
  if [ $lib = old ]; then export DDF_B200_LIB=$OLD; else unset DDF_B200_LIB; fi
  timeout 600 python bench.py --config $cfg --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab7_${cfg}_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab7_${cfg}_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib $cfg', round(d['value']/1e6,2), 'M', round(d['ms_per_step'],1), 'ms', 'mlp', round(r['achieved']), d['clocks']['sm_mhz'])"
done; done
export DDF_B200_LIB=$OLD
for k in TraceGradOp GradOutOp; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_kernel<.*$k" -s 3 -c 1 -o gpurun_out/c4_$k python bench.py --steps 1 --warmup 0 --cpu-baseline 0 --no-e2e > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
