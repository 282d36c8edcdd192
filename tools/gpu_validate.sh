#!/bin/bash
# One gpurun call: GPU tests, smoke, the default bench line and the other
# configs, then (only after the plain runs exited 0) the ncu launch list and
# one --set full capture of each MLP class of the c4 render.
#   gpurun --timeout 3000 -- 'bash tools/gpu_validate.sh <tag> [ncu]'
set -u
TAG=${1:-r2}
WANT_NCU=${2:-}
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests -m gpu -x -q > $OUT/${TAG}_gputest.txt 2>&1; echo "pytest rc=$?" | tee -a $OUT/${TAG}_gputest.txt
tail -3 $OUT/${TAG}_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $OUT/${TAG}_smoke.txt
python bench.py > $OUT/${TAG}_c4_bench.json 2> $OUT/${TAG}_c4_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_c4_reference_arm.json 2>/dev/null; echo "ref rc=$?"
for c in c1 c3 c5; do
  python bench.py --config $c > $OUT/${TAG}_${c}_bench.json 2> $OUT/${TAG}_${c}_bench.err; echo "$c rc=$?"
done
python bench.py --config c1 --precision bf16 > $OUT/${TAG}_c1_bf16_bench.json 2>/dev/null; echo "c1 bf16 rc=$?"
for c in c2 udf; do
  python bench.py --config $c > $OUT/${TAG}_${c}_bench.json 2> $OUT/${TAG}_${c}_bench.err; echo "$c rc=$?"
done
if [ -n "$WANT_NCU" ]; then
  CMD="python bench.py --steps 1 --warmup 0 --cpu-baseline 0 --no-e2e"
  $CMD > $OUT/${TAG}_ncu_plain.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -s 400 -c 400 --csv \
      --log-file $OUT/${TAG}_c4_launches.csv $CMD > $OUT/${TAG}_ncu_launches.log 2>&1
  echo "ncu launches rc=$?"
  for KS in TraceGradOp:7 GradOutOp:8 TraceStepOp:45; do
    K=${KS%%:*}; SKIP=${KS##*:}
    ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
        -k regex:"mlp.*_kernel<.*$K" -s $SKIP -c 1 -o $OUT/${TAG}_ncu_$K -f $CMD > $OUT/${TAG}_ncu_$K.log 2>&1
    echo "ncu $K rc=$?"
    ncu -i $OUT/${TAG}_ncu_$K.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${K}_raw.csv 2>/dev/null
    rm -f $OUT/${TAG}_ncu_$K.ncu-rep   # gpurun_out/ comes back only under 64 MiB: keep the exports
  done
  # the narrow engines: quad (c1 bf16), two-tile 3xTF32 (c1 fp32), ping-pong (c5 forward / gradient)
  MIC="python tools/mlp_micro.py (5,128,128,128,128,1) 4194304"
  $MIC bf16 > $OUT/${TAG}_ncu_micro_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_quad_kernel<.*RawForwardOp" \
      -s 2 -c 1 -o $OUT/${TAG}_ncu_quad -f $MIC bf16 > $OUT/${TAG}_ncu_quad.log 2>&1
  echo "ncu quad rc=$?"
  $MIC fp32 >> $OUT/${TAG}_ncu_micro_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_x3pp_kernel<.*RawForwardOp" \
      -s 2 -c 1 -o $OUT/${TAG}_ncu_x3pp -f $MIC fp32 > $OUT/${TAG}_ncu_x3pp.log 2>&1
  echo "ncu x3pp rc=$?"
  C5="python bench.py --config c5 --steps 1 --warmup 0 --cpu-baseline 0 --no-e2e"
  $C5 > $OUT/${TAG}_ncu_c5_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_pp_kernel<.*TraceStepOp" \
      -s 4 -c 1 -o $OUT/${TAG}_ncu_pp_fwd -f $C5 > $OUT/${TAG}_ncu_pp_fwd.log 2>&1
  echo "ncu pp fwd rc=$?"
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"mlp_pp_kernel<.*GradOutOp" \
      -s 2 -c 1 -o $OUT/${TAG}_ncu_pp_grad -f $C5 > $OUT/${TAG}_ncu_pp_grad.log 2>&1
  echo "ncu pp grad rc=$?"
  for K in quad x3pp pp_fwd pp_grad; do
    ncu -i $OUT/${TAG}_ncu_$K.ncu-rep --page raw --csv > $OUT/${TAG}_ncu_${K}_raw.csv 2>/dev/null
    rm -f $OUT/${TAG}_ncu_$K.ncu-rep
  done
fi
