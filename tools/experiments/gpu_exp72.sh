L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline"
for v in main trig; do
  if [ $v != main ]; then cp tools/libiabn_$v.so $L; fi
  timeout 300 $B > gpurun_out/e72_$v.log 2>&1
  timeout 300 $B --config r50s3 > gpurun_out/e72_r50_$v.log 2>&1
  for cfg in "densenet264 bf16 NHWC" "rx101 bf16 NCHW" "rx101 f32 NCHW"; do
    set -- $cfg
    timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw72_${v}_$1_$2_$3.json 2> gpurun_out/sw72_${v}_$1_$2_$3.err
  done
  cp /tmp/main.so $L
done
IABN_NVCC_EXTRA=-DIABN_PDL_TRIGGER=1 true
echo done
