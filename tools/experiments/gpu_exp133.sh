# warp split of the fused kernels (reduce, apply warps): 3,4 (default) vs 4,4 / 3,5 / 2,5 / 4,6
SH="512x196,1024x196,256x784,1024x49,128x3136"
W="python bench.py --steps 100 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
R="python bench.py --config r50s3 --e2e-steps 0 --no-cpu-baseline --sync-emulated 0"
p() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["fwd_ms"], d["bwd_ms"])'; }
q() { python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(" ".join("%s:%.1f" % (k, v["us_per_layer"]) for k, v in d.items() if isinstance(v, dict)))'; }
for d in . _w44 _w35 _w25 _w46; do
  cd $d
  echo "$d wrn38 $($W 2>/dev/null | p) r50s3 $($R 2>/dev/null | p)"
  echo "$d bf16 $(timeout 200 python tools/shape_graph.py --layout NCHW --dtype bf16 --shapes $SH 2>/dev/null | q)"
  echo "$d f32  $(timeout 200 python tools/shape_graph.py --layout NCHW --dtype f32 --shapes $SH 2>/dev/null | q)"
  cd $GRAFT_REPO_ROOT
done
