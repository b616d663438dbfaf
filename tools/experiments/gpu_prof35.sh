C="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain35.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof35_bwd $C > gpurun_out/ncu35.log 2>&1
echo done
