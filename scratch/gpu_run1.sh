set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
timeout 600 python bench.py --config c2 --precision fp32 > gpurun_out/bench_c2_fp32.json 2> gpurun_out/bench_c2_fp32.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c2_fp32_launches.csv python bench.py --config c2 --precision fp32 --steps 1 --warmup 3 --cpu-baseline 0 --no-e2e > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
