C="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
export IABN_FUSED_K=8
timeout 300 $C > gpurun_out/plain.log 2>&1 && IABN_FUSED_NBUF=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof_bwd_k8nb1 $C > gpurun_out/ncu_full.log 2>&1
IABN_FUSED_NBUF=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 1 -o gpurun_out/prof_fwd_k8nb2 $C > gpurun_out/ncu_full2.log 2>&1
echo done
