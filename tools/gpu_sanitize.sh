#!/bin/bash
# One compute-sanitizer tool per gpurun call (B200_PROFILING.md), on the small
# parity tests that reach every engine (FFMA, 3xTF32, quad / ping-pong / pair
# bf16), the wavefront kernels and the look-back compaction:
#   gpurun --timeout 3000 -- 'bash tools/gpu_sanitize.sh memcheck|racecheck|synccheck'
TOOL=${1:-memcheck}
OUT=gpurun_out/sanitize_$TOOL.txt
mkdir -p gpurun_out
SEL="tests/test_gpu_parity.py tests/test_gpu_x3.py tests/test_gpu_fused.py tests/test_known_answers.py"
python -m pytest $SEL -m gpu -x -q > gpurun_out/sanitize_plain_$TOOL.txt 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/sanitize_plain_$TOOL.txt; exit 1; }
tail -1 gpurun_out/sanitize_plain_$TOOL.txt
timeout 2700 compute-sanitizer --tool $TOOL --target-processes all --error-exitcode 99 --log-file $OUT \
    python -m pytest $SEL -m gpu -x -q > gpurun_out/sanitize_${TOOL}_pytest.txt 2>&1
echo "compute-sanitizer $TOOL rc=$?"
tail -2 gpurun_out/sanitize_${TOOL}_pytest.txt
grep -c "=========" $OUT; tail -5 $OUT
