mkdir -p gpurun_out
timeout 120 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 2097152 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mlp_kernel -s 1 -c 1 -o gpurun_out/mlp512_fwd_v2 python scratch/mlp_micro.py "(65,)+(512,)*8+(1,)" 2097152 > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_src.log
