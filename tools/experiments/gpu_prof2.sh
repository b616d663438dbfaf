timeout 600 python -m pytest tests -m "gpu and not slow" -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $B > gpurun_out/b_default.log 2>&1
IABN_FUSED_SMEM_KB=200 timeout 300 $B > gpurun_out/b_kb200.log 2>&1
C="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $C --schedule streaming > gpurun_out/plain_s.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_stream.csv $C --schedule streaming > gpurun_out/ncu_launch_s.log 2>&1
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 6 -c 2 -o gpurun_out/prof_persist $C > gpurun_out/ncu_full.log 2>&1
echo done
