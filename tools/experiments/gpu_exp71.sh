L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
for v in main nm3 nm4; do
  if [ $v != main ]; then cp tools/libiabn_$v.so $L; fi
  for cfg in "densenet264 bf16 NHWC" "rx101 f32 NHWC"; do
    set -- $cfg
    timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw71_${v}_$1_$2_$3.json 2> gpurun_out/sw71_${v}_$1_$2_$3.err
  done
  cp /tmp/main.so $L
done
echo done
