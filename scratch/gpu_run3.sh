mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_fused.py tests/test_gpu_bf16_scene.py -x -q > gpurun_out/pytest_fused.log 2>&1; echo "fused rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --cpu-baseline 0 > gpurun_out/bench_c4_fused.json 2> gpurun_out/bench_c4_fused.err; echo "bench rc=$?"
timeout 600 python bench.py --config c3 --cpu-baseline 0 > gpurun_out/bench_c3_fused.json 2> gpurun_out/bench_c3_fused.err; echo "bench c3 rc=$?"
