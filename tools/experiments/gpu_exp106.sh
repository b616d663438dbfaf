# NHWC reductions: rows per CTA (IABN_NHWC_ROWS) with the register-unbounded kernels
for r in 256 128 64 32; do
  (cd _nm1 && IABN_NHWC_ROWS=$r timeout 600 python tools/sweep.py --net densenet264 --dtype bf16 --layout NHWC 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('rows $r', d['graph_ms'], d['graph_pct_of_peak'], [ (r['shape'], r['fwd_us'], r['bwd_us']) for r in sorted(d['per_shape'], key=lambda r:-r['share_pct'])[:3]])")
  (cd _nm1 && IABN_NHWC_ROWS=$r timeout 600 python tools/sweep.py --net rx101 --dtype f32 --layout NHWC 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('rows $r rx101 f32 NHWC', d['graph_ms'], d['graph_pct_of_peak'])")
done
