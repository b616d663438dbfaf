B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for kb in 40 56 100 200; do IABN_FUSED_SMEM_KB=$kb timeout 300 $B > gpurun_out/sweep_kb$kb.log 2>&1; done
timeout 300 $B --schedule streaming > gpurun_out/sweep_stream.log 2>&1
timeout 300 $B --config r50s3 > gpurun_out/sweep_r50.log 2>&1
timeout 300 $B --config r50s3 --schedule streaming > gpurun_out/sweep_r50_stream.log 2>&1
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $C > gpurun_out/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv $C > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_ -s 6 -c 2 -o gpurun_out/prof_fused $C > gpurun_out/ncu_full.log 2>&1
echo done
