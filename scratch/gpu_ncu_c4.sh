# ncu evidence for the c4 hot kernels; only text exports come back (reps are large)
mkdir -p gpurun_out
# (bench line: run separately)
for ks in TraceGradOp:7 GradOutOp:8 TraceStepOp:45; do k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_kernel<.*$k" -s $skip -c 1 -f -o /tmp/c4_$k python bench.py --steps 1 --warmup 0 --cpu-baseline 0 --no-e2e > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
  ncu -i /tmp/c4_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv 2>/dev/null
  ncu -i /tmp/c4_$k.ncu-rep --page details --csv > gpurun_out/ncu_${k}_details.csv 2>/dev/null
  ncu -i /tmp/c4_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${k}_sass.csv 2>/dev/null
  gzip -f gpurun_out/ncu_${k}_sass.csv
done
ls -la gpurun_out
