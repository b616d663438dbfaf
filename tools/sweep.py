"""Whole-network layer sweeps of the BN+Act hot path:
every pre-activation BN+Act layer of ResNeXt-101 32x4d or DenseNet-264 at 224^2,
N images per GPU, forward in network order then backward in reverse, each layer
with its own buffers (the working set is far larger than L2).  Reports the
whole sequence's device time (CUDA events), eagerly launched and replayed from a
CUDA graph, and per-shape device times.  Experiments / evidence for profiles/;
not part of the bench contract.

    python tools/sweep.py --net rx101 --dtype f32 [--layout NCHW] [--N 32] [--reps 5]
"""
import argparse
import ctypes
import json
import os
import sys
from collections import OrderedDict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth_inputs as S  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402


densenet264_layers = S.densenet264_layers
rx101_layers = S.rx101_layers


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", choices=["rx101", "densenet264"], default="rx101")
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    ap.add_argument("--layout", choices=["NCHW", "NHWC"], default="NCHW")
    ap.add_argument("--N", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--flags", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    layers = rx101_layers() if args.net == "rx101" else densenet264_layers()
    out_of_place = args.net == "densenet264"  # BN reads the shared concatenated buffer
    tdt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    ldt = L.F32 if args.dtype == "f32" else L.BF16
    lay = L.NCHW if args.layout == "NCHW" else L.NHWC
    b = 4 if args.dtype == "f32" else 2
    N = args.N
    g = torch.Generator(device=dev).manual_seed(0)
    descs, bufs, ws_max = [], [], 0
    for (C, HW) in layers:
        d = L.desc(N, C, HW, ldt, lay)
        ws_max = max(ws_max, L.workspace_bytes(d))
        shape = (N, C, HW) if args.layout == "NCHW" else (N, HW, C)
        x = torch.randn(shape, generator=g, device=dev).to(tdt)
        dz = torch.randn(shape, generator=g, device=dev).to(tdt)
        z = torch.empty_like(x) if out_of_place else x
        f32 = lambda v: torch.full((C,), v, dtype=torch.float32, device=dev)
        p = dict(gamma=torch.rand(C, generator=g, device=dev) + 0.5,
                 beta=torch.randn(C, generator=g, device=dev) * 0.1, rm=f32(0.0), rv=f32(1.0),
                 sm=f32(0.0), sv=f32(1.0), dg=f32(0.0), db=f32(0.0))
        descs.append(d)
        bufs.append(dict(x=x, dz=dz, z=z, **p))
    ws = torch.empty(max(ws_max, 16), dtype=torch.uint8, device=dev)
    E = sum(N * C * HW for C, HW in layers)

    def run_fwd(i, st):
        q, d = bufs[i], descs[i]
        L.call("iabn_forward", ctypes.byref(d), q["x"].data_ptr(), q["z"].data_ptr(),
               q["gamma"].data_ptr(), q["beta"].data_ptr(), q["rm"].data_ptr(),
               q["rv"].data_ptr(), q["sm"].data_ptr(), q["sv"].data_ptr(), 0.1, 1e-5, 0.01,
               args.flags, ws.data_ptr(), ws.numel(), st)

    def run_bwd(i, st):
        q, d = bufs[i], descs[i]
        L.call("iabn_backward", ctypes.byref(d), q["z"].data_ptr(), q["dz"].data_ptr(),
               q["dz"].data_ptr(), q["gamma"].data_ptr(), q["beta"].data_ptr(), None,
               q["sv"].data_ptr(), q["dg"].data_ptr(), q["db"].data_ptr(), 1e-5, 0.01,
               args.flags, ws.data_ptr(), ws.numel(), st)

    def sequence():
        st = torch.cuda.current_stream().cuda_stream
        for i in range(len(layers)):
            run_fwd(i, st)
        for i in reversed(range(len(layers))):
            run_bwd(i, st)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t_eager = timed(sequence, args.reps)
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        sequence()  # warm-up on the capture stream (kernel attributes, plans)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(graph):
        sequence()
    t_graph = timed(graph.replay, args.reps)

    # per-shape device time: for each distinct shape, the forwards of all its layers (in
    # network order, each on its own buffers) captured in one CUDA graph, the backwards in
    # another; replayed, device time per layer (launch gaps excluded as in the sequence)
    per = OrderedDict()
    for i, (C, HW) in enumerate(layers):
        per.setdefault(f"{C}x{HW}", dict(C=C, HW=HW, idx=[]))["idx"].append(i)
    for k, r in per.items():
        r["count"] = len(r["idx"])
        for name, fn in (("fwd_us", run_fwd), ("bwd_us", run_bwd)):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                for i in r["idx"]:
                    fn(i, s.cuda_stream)  # warm-up on the capture stream
            torch.cuda.synchronize()
            with torch.cuda.graph(gr, stream=s):
                for i in r["idx"]:
                    fn(i, s.cuda_stream)
            r[name] = timed(gr.replay, max(args.reps, 5)) * 1e3
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    shapes = []
    for k, r in per.items():
        e = N * r["C"] * r["HW"] * r["count"]
        t = (r["fwd_us"] + r["bwd_us"]) * 1e-6
        shapes.append(dict(shape=k, count=r["count"], fwd_us=round(r["fwd_us"] / r["count"], 2),
                           bwd_us=round(r["bwd_us"] / r["count"], 2),
                           share_pct=round(100 * (r["fwd_us"] + r["bwd_us"]) * 1e-3 / t_graph, 1),
                           pct_of_peak=round(100 * 5 * e * b / t / 1e9 / peak, 1)))
    res = dict(net=args.net, dtype=args.dtype, layout=args.layout, N=N, layers=len(layers),
               elements=E, algorithmic_bytes=5 * E * b, out_of_place=out_of_place,
               eager_ms=round(t_eager, 4), graph_ms=round(t_graph, 4),
               eager_pct_of_peak=round(100 * 5 * E * b / (t_eager * 1e-3) / 1e9 / peak, 1),
               graph_pct_of_peak=round(100 * 5 * E * b / (t_graph * 1e-3) / 1e9 / peak, 1),
               per_shape=shapes)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
