# NHWC reductions: register caps / unroll variants vs the committed build (_base)
for d in _base _nm1 _nm3 _nm3u8; do
  (cd $d && timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$d', d['graph_ms'], d['graph_pct_of_peak'], [ (r['shape'], r['fwd_us'], r['bwd_us']) for r in sorted(d['per_shape'], key=lambda r:-r['share_pct'])[:3]])")
  (cd $d && timeout 600 python tools/sweep.py --net rx101 --dtype f32 --layout NHWC 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$d rx101 f32 NHWC', d['graph_ms'], d['graph_pct_of_peak'])")
done
