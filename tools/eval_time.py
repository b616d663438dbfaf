"""Graph-replay device time of the eval-mode forward (fixed running statistics, PAPER.md:85:
one read and one write per element) against a torch copy of the same tensor.

    python tools/eval_time.py [--shapes 16x4096x12544:bf16:NCHW,...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="16x4096x12544:bf16:NCHW,64x1024x196:f32:NCHW,"
                "32x512x196:bf16:NCHW,32x128x3136:bf16:NHWC,32x1024x49:bf16:NCHW")
args = ap.parse_args()
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def graph_us(fn, R):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * R) * 1e3


for spec in args.shapes.split(","):
    sh, dts, layout = spec.split(":")
    N, C, HW = (int(v) for v in sh.split("x"))
    dt = torch.bfloat16 if dts == "bf16" else torch.float32
    shape = (N, C, HW) if layout == "NCHW" else (N, HW, C)
    nbytes = N * C * HW * (2 if dts == "bf16" else 4)
    R = max(1, min(16, (1 << 30) // (2 * nbytes)))
    xs = [torch.randn(shape, device="cuda").to(dt) for _ in range(R)]
    os_ = [torch.empty_like(xs[0]) for _ in range(R)]
    g, b = torch.rand(C, device="cuda") + 0.5, torch.zeros(C, device="cuda")
    rm, rv = torch.randn(C, device="cuda"), torch.rand(C, device="cuda") + 0.5
    ev = graph_us(lambda: [P.forward(x, g, b, rm, rv, training=False, out=o, layout=layout)
                           for x, o in zip(xs, os_)], R)
    cp = graph_us(lambda: [o.copy_(x) for x, o in zip(xs, os_)], R)
    print(json.dumps(dict(shape=spec, MB=round(nbytes / 1e6, 1), eval_us=round(ev, 2),
                          copy_us=round(cp, 2), eval_pct=round(100 * 2 * nbytes / (ev * 1e-6) / (PEAK * 1e9), 1))))
