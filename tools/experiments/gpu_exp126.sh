# phase trace of small layers (producer issue time of a slice with many planes)
for s in 32,512,196,bf16 32,1024,196,bf16 64,1024,196,f32 32,512,784,bf16; do
  echo "##### $s"; IABN_VERBOSE=1 IABN_FUSED_DEBUG=4 timeout 120 python tools/trace_fused.py --shape $s 2>&1 | head -40
done
