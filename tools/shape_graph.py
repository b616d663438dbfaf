"""Device time per layer (forward + backward) of given shapes, from a CUDA graph over
R distinct buffer sets (so inputs come from HBM, not L2), launch costs hidden.

    python tools/shape_graph.py --layout NHWC --dtype bf16 --shapes 64x3136,128x196 [--N 32]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

PEAK_GBS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]

ap = argparse.ArgumentParser()
ap.add_argument("--layout", default="NHWC")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--shapes", default="64x3136,128x3136,128x784,128x196,128x49,512x196")
ap.add_argument("--N", type=int, default=32)
args = ap.parse_args()
dev = torch.device("cuda", 0)
dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
res = {}
for sh in args.shapes.split(","):
    C, HW = (int(v) for v in sh.split("x"))
    N = args.N
    shape = (N, C, HW) if args.layout == "NCHW" else (N, HW, C)
    nbytes = N * C * HW * (2 if dt == torch.bfloat16 else 4)
    R = max(2, min(64, (512 << 20) // max(nbytes, 1)))
    xs = [torch.randn(shape, device=dev).to(dt) for _ in range(R)]
    dzs = [torch.randn(shape, device=dev).to(dt) for _ in range(R)]
    g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)

    def seq():
        for x, dz in zip(xs, dzs):
            z, _, v = P.forward(x, g, b, layout=args.layout)
            P.backward(z, dz, g, b, v, layout=args.layout)

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
    us = e0.elapsed_time(e1) / (5 * R) * 1e3
    res[sh] = dict(us_per_layer=round(us, 2), pct_of_peak=round(100 * 5 * nbytes / (us * 1e-6) / (PEAK_GBS * 1e9), 1))
print(json.dumps(dict(layout=args.layout, dtype=args.dtype, N=args.N, **res)))
