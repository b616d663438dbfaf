# warp-count variants (reduce R, apply A, min CTAs/SM for the register cap)
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
for v in main au8 ru16 r4ru8 ord0 au3 r3a4m1; do
  if [ $v != main ]; then cp tools/libiabn_$v.so $L; fi
  timeout 300 $B > gpurun_out/e42_$v.log 2>&1
  timeout 300 $B --config r50s3 > gpurun_out/e42_r50_$v.log 2>&1
  cp /tmp/main.so $L
done
echo done
