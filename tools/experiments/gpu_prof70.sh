timeout 600 ncu --set full --clock-control none -k regex:"stats_nhwc|fwd_apply_nhwc|bwd_reduce_nhwc|bwd_apply_nhwc" -s 4 -c 4 -o gpurun_out/prof70_nhwc python tools/layer_probe.py 32 128 3136 bf16 NHWC > gpurun_out/ncu70.log 2>&1
echo done
