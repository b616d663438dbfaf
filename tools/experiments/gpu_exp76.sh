# one-launch schedule for small layers with a grid sized to the layer
for mode in "0 48 32" "1 4 32" "1 8 16" "1 4 64"; do
  set -- $mode
  for cfg in "densenet264 bf16 NHWC" "rx101 bf16 NCHW"; do
    set -- $mode $cfg
    IABN_COOP=$1 IABN_COOP_MB=$2 IABN_COOP_KB_PER_CTA=$3 timeout 600 python tools/sweep.py --net $4 --dtype $5 --layout $6 > gpurun_out/sw76_$1_$2_$3_$4_$5_$6.json 2> gpurun_out/sw76_$1_$2_$3_$4_$5_$6.err
  done
done
echo done
