# whole-network sweeps (cfg3 ResNeXt-101, cfg5 DenseNet-264)
for cfg in "rx101 f32 NCHW" "rx101 bf16 NCHW" "densenet264 f32 NCHW" "densenet264 bf16 NCHW" "densenet264 bf16 NHWC" "rx101 f32 NHWC"; do
  set -- $cfg
  timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw49_$1_$2_$3.json 2> gpurun_out/sw49_$1_$2_$3.err
done
echo done
