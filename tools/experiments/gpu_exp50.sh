# per-kernel times of small / misaligned / NHWC layers
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
i=0
for s in "32 512 196 bf16 NCHW" "32 512 196 f32 NCHW" "32 512 196 bf16 NHWC" "32 256 3136 f32 NHWC" "32 1024 49 bf16 NCHW" "32 128 3136 bf16 NCHW"; do
  i=$((i+1))
  timeout 300 ncu $M --log-file gpurun_out/l50_$i.csv python tools/layer_probe.py $s > gpurun_out/l50_$i.log 2>&1
  echo "$i $s" >> gpurun_out/l50_index.txt
done
echo done
