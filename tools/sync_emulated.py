"""Synchronized InPlace-ABN on one GPU: the fused-collective kernels
over G virtual ranks (iabn_{forward,backward}_sync_emulated: one cooperative launch,
the ranks' channel records exchanged through the peer-record protocol) against the
same tensor through (a) the plain channel-resident kernels (G = 1, no exchange) and
(b) the streaming schedule the reduce / ncclAllReduce / apply sync path runs (its
kernels only: the all-reduce itself is not part of a one-GPU run).  Device time per
pass with CUDA events, L2 flushed before every timed pass; GB/s for the
channel-resident bytes (2 E b forward, 3 E b backward) and as % of the measured peak.

    python tools/sync_emulated.py [--cfg wrn38|r50s3] [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402

CFGS = {"wrn38": (16, 4096, 112 * 112, torch.bfloat16),
        "r50s3": (64, 1024, 14 * 14, torch.float32),
        "rx101_14": (256, 1024, 14 * 14, torch.bfloat16)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", choices=sorted(CFGS), default="wrn38")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--G", default="1,2,4,8")
    args = ap.parse_args()
    N, C, HW, dt = CFGS[args.cfg]
    dev = torch.device("cuda", 0)
    peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    g = torch.rand(C, device=dev) + 0.5
    b = torch.rand(C, device=dev) - 0.5
    x0 = torch.randn(N, C, HW, device=dev).to(dt)
    dz0 = torch.randn(N, C, HW, device=dev).to(dt)
    x, dz, dx = x0.clone(), dz0.clone(), torch.empty_like(dz0)
    flush = torch.empty(2 * 126 * 2**20 // 4, device=dev)
    E, eb = x.numel(), x.element_size()

    def timeit(fn):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(args.iters):
            flush.add_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        ts.sort()
        return ts[len(ts) // 2]

    rows = []
    state = {}

    def fwd_emu(G):
        def f():
            _, _, state["sv"] = P.forward_sync_emulated(x, G, g, b)
        return f

    def bwd_emu(G):
        def f():
            P.backward_sync_emulated(x, dz, G, g, b, state["sv"], dx=dx)
        return f

    def fwd_plain(flags):
        def f():
            _, _, state["sv"] = P.forward(x, g, b, flags=flags)
        return f

    def bwd_plain(flags):
        def f():
            P.backward(x, dz, g, b, state["sv"], dx=dx, flags=flags)
        return f

    variants = [("fused, no exchange", fwd_plain(L.FORCE_FUSED), bwd_plain(L.FORCE_FUSED), 1)]
    for G in [int(v) for v in args.G.split(",")]:
        if N % G == 0:
            variants.append((f"fused-collective sync, G={G}", fwd_emu(G), bwd_emu(G), G))
    variants.append(("streaming (reduce/all-reduce/apply kernels)", fwd_plain(L.FORCE_STREAMING),
                     bwd_plain(L.FORCE_STREAMING), 1))
    for name, f, bw, G in variants:
        x.copy_(x0)
        try:
            tf = timeit(f)
            tb = timeit(bw)
        except Exception as e:  # a schedule override that does not fit this variant
            print(json.dumps(dict(variant=name, G=G, error=str(e)[:120])), flush=True)
            continue
        gf, gb = 2 * E * eb / tf / 1e9, 3 * E * eb / tb / 1e9
        tot = 5 * E * eb / (tf + tb) / 1e9
        rows.append(dict(variant=name, G=G, fwd_us=round(tf * 1e6, 1), bwd_us=round(tb * 1e6, 1),
                         fwd_gbps=round(gf), bwd_gbps=round(gb), fwd_bwd_gbps=round(tot),
                         pct_of_peak=round(100 * tot / peak, 1)))
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps(dict(cfg=args.cfg, shape=[N, C, HW], dtype=str(dt), peak_gbps=peak,
                          bytes="5*E*b (channel-resident minimum)", rows=rows)))


if __name__ == "__main__":
    main()
