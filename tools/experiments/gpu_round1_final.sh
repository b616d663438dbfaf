# round-1 measurement set: tests, bench (default), launch list, full ncu of both fused kernels
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests_all.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_all.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/smi_before.csv
IABN_VERBOSE=1 timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; echo rc=$? >> gpurun_out/bench_final.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $C > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 2 -c 2 -o gpurun_out/prof_final $C > gpurun_out/ncu_full.log 2>&1
echo done
