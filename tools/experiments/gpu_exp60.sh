# small layers: more CTAs per SM (register cap) and smaller slabs
L=paper_1712_02616_b200/libiabn.so
cp $L /tmp/main.so
B="python bench.py --steps 60 --warmup 5 --e2e-steps 0 --no-cpu-baseline --config r50s3"
timeout 300 $B > gpurun_out/e60_main.log 2>&1
timeout 300 python tools/sweep.py --net rx101 --dtype f32 --layout NCHW > gpurun_out/sw60_main.json 2>&1
for v in m4 m3; do
  cp tools/libiabn_$v.so $L
  for kb in 50 66; do
    IABN_FUSED_SMEM_KB=$kb timeout 300 $B > gpurun_out/e60_${v}_$kb.log 2>&1
    IABN_FUSED_SMEM_KB=$kb timeout 300 python tools/sweep.py --net rx101 --dtype f32 --layout NCHW > gpurun_out/sw60_${v}_$kb.json 2>&1
  done
  cp /tmp/main.so $L
done
echo done
