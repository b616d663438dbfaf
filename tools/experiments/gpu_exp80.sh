M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
i=0
rm -f gpurun_out/l80_index.txt
for s in "32 128 196 bf16 NHWC" "32 128 3136 bf16 NHWC" "32 64 3136 bf16 NHWC"; do
 for g in 1 0; do
  i=$((i+1))
  IABN_GRES=$g timeout 300 ncu $M --log-file gpurun_out/l80_$i.csv python tools/layer_probe.py $s > gpurun_out/l80_$i.log 2>&1
  echo "$i gres=$g $s" >> gpurun_out/l80_index.txt
 done
done
IABN_GRES=1 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "grid_resident or offset or stress" > gpurun_out/t80.log 2>&1
IABN_GRES=0 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "stress" > gpurun_out/t80b.log 2>&1
echo done
