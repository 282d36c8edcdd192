mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final_c4_ref.json 2> gpurun_out/final_c4_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v11.csv python bench.py --steps 1 --warmup 3 --cpu-baseline 0 --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
for k in TraceGradOp GradOutOp TraceStepOp; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel<.*$k" -s 3 -c 1 -o gpurun_out/c4_$k python bench.py --steps 1 --warmup 0 --cpu-baseline 0 --no-e2e > gpurun_out/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
