M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
i=0
rm -f gpurun_out/l57_index.txt
for s in "32 512 196 bf16 NCHW" "32 512 196 f32 NCHW" "32 512 196 f32 NCHW 256" "32 128 784 bf16 NHWC"; do
  i=$((i+1))
  timeout 300 ncu $M --log-file gpurun_out/l57_$i.csv python tools/layer_probe.py $s > gpurun_out/l57_$i.log 2>&1
  echo "$i $s" >> gpurun_out/l57_index.txt
done
echo done
