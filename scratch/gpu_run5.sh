mkdir -p gpurun_out
timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 2097152 > gpurun_out/micro5.log 2>&1; echo "micro rc=$?"
cat gpurun_out/micro5.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --cpu-baseline 0 > gpurun_out/bench_c4_v10.json 2> gpurun_out/bench_c4_v10.err; echo "bench rc=$?"
timeout 600 python bench.py --config c3 --cpu-baseline 0 > gpurun_out/bench_c3_v10.json 2> gpurun_out/bench_c3_v10.err; echo "bench c3 rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/bench_c4_v10.json", "gpurun_out/bench_c3_v10.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f, d["value"], d["ms_per_step"], r["achieved"], r.get("forward", {}).get("tflops"), r.get("gradient", {}).get("tflops"), r.get("fused_trace_gradient", {}).get("tflops"), d["clocks"])
    except Exception as e: print(f, e)
PY
