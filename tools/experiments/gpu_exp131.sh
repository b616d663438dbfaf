# small NCHW layers (ResNeXt-101 / DenseNet shapes, N=32): cluster size / slab size knobs
SH="512x196,1024x196,256x784,1024x49,2048x49,128x3136"
for dt in bf16 f32; do
for v in "X=1" "IABN_FUSED_K=2" "IABN_FUSED_K=4" "IABN_FUSED_SMALL_KB=25" "IABN_FUSED_SMALL_KB=30 IABN_FUSED_DEEP=0" "IABN_FUSED_DEEP=0"; do
  echo "$dt $v $(env $v timeout 200 python tools/shape_graph.py --layout NCHW --dtype $dt --shapes $SH 2>/dev/null | tail -1)"
done; done
