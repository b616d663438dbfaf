# streaming statistics / gradient-sum kernels: plane cursor, batched raw loads
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --schedule streaming"
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline --schedule streaming"
timeout 300 $B > gpurun_out/e46.log 2>&1
timeout 300 $B --config r50s3 > gpurun_out/e46_r50.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l46.csv $C > /dev/null 2>&1
echo done
