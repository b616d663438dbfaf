"""Per-shape device time of the NHWC schedules: streaming and every feasible channel-group
plan (g channels per group, K CTAs per cluster), forward and backward separately, from
CUDA-graph replay over R distinct buffer sets (inputs from HBM, launch cost hidden).

    python tools/nhwc_tune.py --dtype bf16 --shapes 128x49,128x196,... [--N 32] [--gs 8,16,32,64]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
hook = L.lib.iabn_debug_nhwc_plan
hook.argtypes = [ctypes.c_int] * 3
hook.restype = None

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--shapes", default="128x49,128x196,128x784,128x3136,512x196,1024x49,2688x49")
ap.add_argument("--N", type=int, default=32)
ap.add_argument("--gs", default="")
ap.add_argument("--ks", default="1,2,3,4,6,8")
args = ap.parse_args()
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
b = 2 if args.dtype == "bf16" else 4


def time_pass(xs, dzs, g, bt, pass_, flags):
    def seq():
        for x, dz in zip(xs, dzs):
            if pass_ == 0:
                P.forward(x, g, bt, layout="NHWC", out=dz, flags=flags)
            else:
                P.backward(x, dz, g, bt, sv, layout="NHWC", dx=out, flags=flags)
    C = g.numel()
    sv = torch.ones(C, device=dev)
    out = torch.empty_like(xs[0])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        seq()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        seq()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * len(xs)) * 1e3


res = {}
for sh in args.shapes.split(","):
    C, HW = (int(v) for v in sh.split("x"))
    N = args.N
    nbytes = N * C * HW * b
    R = max(2, min(32, (256 << 20) // max(nbytes, 1)))
    xs = [torch.randn((N, HW, C), device=dev).to(dt) for _ in range(R)]
    dzs = [torch.randn((N, HW, C), device=dev).to(dt) for _ in range(R)]
    g, bt = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
    rows = {}
    hook(0, 0, 0)
    rows["streaming"] = [time_pass(xs, dzs, g, bt, p, L.FORCE_STREAMING) for p in (0, 1)]
    rows["auto"] = [time_pass(xs, dzs, g, bt, p, 0) for p in (0, 1)]
    d = L.desc(N, C, HW, L.BF16 if b == 2 else L.F32, L.NHWC)
    gs = [int(v) for v in args.gs.split(",")] if args.gs else \
        [gb // b for gb in (16, 32, 64, 128, 256) if gb // b <= C]
    for gg in gs:
        for K in (int(v) for v in args.ks.split(",")):
            hook(gg, K, 0)
            t = []
            for p in (0, 1):
                s_, k_ = L.query_schedule(d, p)
                t.append(time_pass(xs, dzs, g, bt, p, 0) if (s_ == 4 and k_ == K) else None)
            rows[f"g{gg}_K{K}"] = t
    hook(0, 0, 0)
    best = {p: min((v[p], k) for k, v in rows.items() if v[p] is not None) for p in (0, 1)}
    res[sh] = dict(rows={k: [None if x is None else round(x, 2) for x in v] for k, v in rows.items()},
                   best_fwd=best[0], best_bwd=best[1],
                   pct_best=round(100 * 5 * nbytes / ((best[0][0] + best[1][0]) * 1e-6) / (PEAK * 1e9), 1))
    print(sh, json.dumps(res[sh]["rows"]), "best", best, flush=True)
print(json.dumps(dict(dtype=args.dtype, N=args.N, **res)))
