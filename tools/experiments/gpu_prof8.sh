C="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
export IABN_FUSED_NBUF=3
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 6 -c 2 -o gpurun_out/prof_ws2 $C > gpurun_out/ncu_full.log 2>&1
echo done
