"""Graph-replay device time of the streaming phases of one NHWC / NCHW layer through the
split-phase C ABI: forward_reduce (statistics + combine), forward_apply (coefficients +
apply), backward_reduce (gradient sums + combine), backward_apply (coefficients + dx),
each over R distinct buffer sets.  Also the torch copy_ of the same bytes.

    python tools/phase_time.py --shape 32x128x3136 --dtype bf16 --layout NHWC
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="32x128x3136")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--layout", default="NHWC")
args = ap.parse_args()
N, C, HW = (int(v) for v in args.shape.split("x"))
dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
shape = (N, C, HW) if args.layout == "NCHW" else (N, HW, C)
E = N * C * HW
b = 2 if args.dtype == "bf16" else 4
R = max(2, min(16, (512 << 20) // (E * b * 3)))
xs = [torch.randn(shape, device="cuda").to(dt) for _ in range(R)]
dzs = [torch.randn(shape, device="cuda").to(dt) for _ in range(R)]
outs = [torch.empty_like(xs[0]) for _ in range(R)]
g, bt = torch.rand(C, device="cuda") + 0.5, torch.zeros(C, device="cuda")
sv = torch.ones(C, device="cuda")
sts = [P.forward_reduce(x, layout=args.layout) for x in xs]
sums = [P.backward_reduce(x, dz, g, bt, layout=args.layout) for x, dz in zip(xs, dzs)]


def graph_us(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / (10 * R) * 1e3, 2)


res = dict(shape=args.shape, dtype=args.dtype, layout=args.layout, MB=round(E * b / 1e6, 2))
res["fwd_reduce"] = graph_us(lambda: [P.forward_reduce(x, layout=args.layout) for x in xs])
res["fwd_apply"] = graph_us(lambda: [P.forward_apply(x, st, g, bt, out=o, layout=args.layout)
                                     for x, st, o in zip(xs, sts, outs)])
res["fwd_whole"] = graph_us(lambda: [P.forward(x, g, bt, out=o, layout=args.layout)
                                     for x, o in zip(xs, outs)])
res["bwd_reduce"] = graph_us(lambda: [P.backward_reduce(x, dz, g, bt, layout=args.layout)
                                      for x, dz in zip(xs, dzs)])
res["bwd_apply"] = graph_us(lambda: [P.backward_apply(x, dz, sm, None, g, bt, sv, dx=o,
                                                      layout=args.layout)
                                     for x, dz, sm, o in zip(xs, dzs, sums, outs)])
res["bwd_whole"] = graph_us(lambda: [P.backward(x, dz, g, bt, sv, dx=o, layout=args.layout)
                                     for x, dz, o in zip(xs, dzs, outs)])
res["copy"] = graph_us(lambda: [o.copy_(x) for x, o in zip(xs, outs)])
res["read_sum"] = graph_us(lambda: [x.sum() for x in xs])
print(json.dumps(res))
