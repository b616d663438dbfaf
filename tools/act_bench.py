"""Device time of BN + sigmoid / tanh (streaming, kernels_act.cuh) next to BN + leaky ReLU
(automatic schedule) on the same fp32 tensor, forward and backward, from CUDA-graph replay
over R distinct buffer sets (inputs from HBM).  Bytes: algorithmic 2 E b forward,
3 E b backward (read x / write z; read z, dz / write dx); the streaming schedule moves
3 E b + 5 E b.

    python tools/act_bench.py [--shapes 32x256x3136,32x1024x196] [--layout NCHW]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="32x256x3136,32x512x784,32x1024x196,32x2048x49")
ap.add_argument("--layout", default="NCHW")
args = ap.parse_args()
dev = torch.device("cuda", 0)


def time_pass(seq):
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
    return e0.elapsed_time(e1) / 5


out = {}
for sh in args.shapes.split(","):
    N, C, HW = (int(v) for v in sh.split("x"))
    shape = (N, C, HW) if args.layout == "NCHW" else (N, HW, C)
    E = N * C * HW
    R = max(2, min(16, (1 << 30) // (E * 4)))
    xs = [torch.randn(shape, device=dev) for _ in range(R)]
    dzs = [torch.randn(shape, device=dev) for _ in range(R)]
    dxs = [torch.empty(shape, device=dev) for _ in range(R)]
    g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
    sv = torch.ones(C, device=dev)
    row = {}
    for act in ("leaky_relu", "sigmoid", "tanh"):
        tf = time_pass(lambda: [P.forward(x, g, b, out=dz, layout=args.layout, activation=act)
                                for x, dz in zip(xs, dzs)]) / R
        tb = time_pass(lambda: [P.backward(x, dz, g, b, sv, dx=dx, layout=args.layout,
                                           activation=act)
                                for x, dz, dx in zip(xs, dzs, dxs)]) / R
        row[act] = dict(fwd_us=round(tf * 1e3, 1), bwd_us=round(tb * 1e3, 1),
                        alg_frac=round(5 * E * 4 / ((tf + tb) * 1e-3) / (PEAK * 1e9), 3),
                        moved_frac=round(8 * E * 4 / ((tf + tb) * 1e-3) / (PEAK * 1e9), 3))
    out[sh] = row
    print(sh, json.dumps(row), flush=True)
print(json.dumps(dict(layout=args.layout, peak_gbs=PEAK, shapes=out)))
