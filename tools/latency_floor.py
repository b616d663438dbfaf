"""Calibration of the per-pass latency floor under CUDA-graph replay: time per launch of
(a) torch's copy_ (one read + one write stream) for tensors of 0.001-26 MB and (b) the
library's forward / backward on a tiny layer, each captured R times back to back on
distinct buffers (the sweep's methodology).

    python tools/latency_floor.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402


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
    for _ in range(10):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (10 * R) * 1e3


out = {}
for mb in (0.001, 0.4, 1.6, 6.4, 12.8, 25.6):
    n = max(1, int(mb * 1e6 / 2))
    R = 64
    src = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(R)]
    dst = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(R)]
    us = graph_us(lambda: [d.copy_(s_) for d, s_ in zip(dst, src)], R)
    out[f"copy_{mb}MB"] = dict(us=round(us, 2), gbs=round(2 * n * 2 / (us * 1e-6) / 1e9, 1))
for shape, dt in (((2, 8, 16), torch.float32), ((32, 512, 196), torch.bfloat16),
                  ((32, 128, 196), torch.bfloat16)):
    R = 32
    xs = [torch.randn(shape, device="cuda").to(dt) for _ in range(R)]
    dzs = [torch.randn(shape, device="cuda").to(dt) for _ in range(R)]
    C = shape[1]
    g, b, sv = (torch.ones(C, device="cuda"), torch.zeros(C, device="cuda"),
                torch.ones(C, device="cuda"))
    f = graph_us(lambda: [P.forward(x, g, b) for x in xs], R)
    bw = graph_us(lambda: [P.backward(x, dz, g, b, sv) for x, dz in zip(xs, dzs)], R)
    out["iabn_%dx%dx%d_%s" % (*shape, str(dt)[6:])] = dict(fwd_us=round(f, 2), bwd_us=round(bw, 2))
print(json.dumps(out, indent=1))
