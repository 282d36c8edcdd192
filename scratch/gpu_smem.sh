mkdir -p gpurun_out
test -f scratch/statslib/libddf_b200.so || { echo no statslib; exit 1; }
for d in 0 128; do
  STATS=1 DDF_DEBUG_UMMA=$d timeout 120 python scratch/smem_exp.py "(65,)+(512,)*8+(1,)" 2097152 >> gpurun_out/smem_exp2.log 2>&1
  STATS=1 DDF_DEBUG_UMMA=$d timeout 120 python scratch/smem_exp.py "(5,)+(256,)*8+(1,)" 2097152 >> gpurun_out/smem_exp2.log 2>&1
done
cat gpurun_out/smem_exp2.log
