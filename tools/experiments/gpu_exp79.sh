timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests.log
for g in 1 0; do
for cfg in "densenet264 bf16 NHWC" "rx101 f32 NHWC"; do
  set -- $cfg
  IABN_GRES=$g timeout 600 python tools/sweep.py --net $1 --dtype $2 --layout $3 > gpurun_out/sw79_${g}_$1_$2_$3.json 2> gpurun_out/sw79_${g}_$1_$2_$3.err
done; done
echo done
