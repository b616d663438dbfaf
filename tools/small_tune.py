"""Per-shape device time of the register-resident small-layer schedule vs the
channel-resident (or streaming) one, graph replay over R buffer sets.

    python tools/small_tune.py --dtype bf16 --shapes 512x196,1024x49 [--N 32]
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

hook = L.lib.iabn_debug_small
hook.argtypes = [ctypes.c_int]
hook.restype = None
hook_r = L.lib.iabn_debug_small_r
hook_r.argtypes = [ctypes.c_int]
hook_r.restype = None
ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--shapes", default="512x196,1024x196,1024x49,2048x49,128x196,128x49,512x784")
ap.add_argument("--N", type=int, default=32)
args = ap.parse_args()
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
b = 2 if args.dtype == "bf16" else 4


def time_pass(xs, dzs, g, bt, pass_):
    C = g.numel()
    sv = torch.ones(C, device=dev)
    out = torch.empty_like(xs[0])

    def seq():
        for x, dz in zip(xs, dzs):
            if pass_ == 0:
                P.forward(x, g, bt, out=dz)
            else:
                P.backward(x, dz, g, bt, sv, dx=out)
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
    return round(e0.elapsed_time(e1) / (5 * len(xs)) * 1e3, 2)


res = {}
for sh in args.shapes.split(","):
    C, HW = (int(v) for v in sh.split("x"))
    N = args.N
    nbytes = N * C * HW * b
    R = max(2, min(32, (256 << 20) // max(nbytes, 1)))
    xs = [torch.randn((N, C, HW), device=dev).to(dt) for _ in range(R)]
    dzs = [torch.randn((N, C, HW), device=dev).to(dt) for _ in range(R)]
    g, bt = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
    d = L.desc(N, C, HW, L.BF16 if b == 2 else L.F32, L.NCHW)
    rows = {}
    hook(-1)
    rows["channel-resident"] = [time_pass(xs, dzs, g, bt, p) for p in (0, 1)]
    hook(1)
    for r in (4, 8):
        hook_r(r)
        if L.query_schedule(d, 0)[0] == 5:
            rows[f"small_R{r}"] = [time_pass(xs, dzs, g, bt, p) for p in (0, 1)]
    hook_r(0)
    hook(0)
    rows["auto"] = [time_pass(xs, dzs, g, bt, p) for p in (0, 1)]
    res[sh] = rows
    print(sh, json.dumps(rows), flush=True)
print(json.dumps(dict(dtype=args.dtype, N=args.N, **res)))
