C="python bench.py --config r50s3 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 300 $C > gpurun_out/e74_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l74.csv $C > /dev/null 2>&1
timeout 300 nsys --version > /dev/null 2>&1 || true
echo done
