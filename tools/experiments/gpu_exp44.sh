# streaming kernels: loads in flight (unroll) and split target
C="python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --schedule streaming"
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline --schedule streaming"
L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
for v in main su8 tw4 su8tw4; do
  if [ $v != main ]; then cp tools/libiabn_$v.so $L; fi
  timeout 300 $B > gpurun_out/e44_$v.log 2>&1
  timeout 300 $B --config r50s3 > gpurun_out/e44_r50_$v.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l44_$v.csv $C > /dev/null 2>&1
  cp /tmp/main.so $L
done
echo done
