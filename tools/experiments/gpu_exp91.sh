for m in 1 0; do
for cfg in "rx101 bf16 NCHW" "densenet264 bf16 NCHW" "densenet264 f32 NCHW" "rx101 f32 NCHW"; do
  set -- $cfg
  IABN_FUSED_MIS=$m timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw91_${m}_$1_$2_$3.json 2> gpurun_out/sw91_${m}_$1_$2_$3.err
done; done
echo done
