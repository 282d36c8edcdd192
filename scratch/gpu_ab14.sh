# Bucketed scan over all objects at once: GPU tests, then A/B against the previous build
# (scratch/oldlib) on the 8-object scene (c5).
mkdir -p gpurun_out
OLD=$PWD/scratch/oldlib/libddf_b200.so
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab14_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/ab14_pytest.log
for cfg in c5; do
for lib in old new old new; do
  if [ $lib = old ]; then export DDF_B200_LIB=$OLD; else unset DDF_B200_LIB; fi
  timeout 600 python bench.py --config $cfg --cpu-baseline 0 --no-e2e --steps 3 > gpurun_out/ab14_${cfg}_$lib.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ab14_${cfg}_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib $cfg', round(d['value']/1e6,3), 'M', round(d['ms_per_step'],2), 'ms', 'compaction_ms', round(r.get('compaction_ms') or 0, 2), 'launches', d['gpu_launches'], d['clocks']['sm_mhz'])"
done
done
unset DDF_B200_LIB
