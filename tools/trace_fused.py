"""Phase timeline of the channel-resident kernels (experiments; run on a B200).

    IABN_FUSED_DEBUG=4 python tools/trace_fused.py [--config wrn38] [--pass fwd|bwd]

Runs one forward (and backward) of the workload, reads the per-CTA, per-channel
%globaltimer stamps the kernel recorded (see IABN_TRACE in kernels_fused.cuh)
and prints the distribution of each pipeline interval.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = ["issue0", "issueN", "got0", "gotN", "pushed", "gathered", "apply0", "applyN",
         "reduced", "summed", "slotfree", "published"]
F = len(NAMES)


def dump(L):
    n = L.lib.iabn_debug_trace(None, 0)
    buf = (ctypes.c_ulonglong * n)()
    L.lib.iabn_debug_trace(buf, n)
    per = L.lib.iabn_debug_trace_channels()
    return np.frombuffer(buf, dtype=np.uint64).reshape(-1, F).astype(np.int64), per


def report(tr, label, grid_ch):
    tr = tr.reshape(-1, grid_ch, F)  # [cta][t][8]
    valid = (tr > 0).all(axis=2)
    t0 = tr[tr > 0].min()
    print(f"== {label}: {tr.shape[0]} CTAs x {grid_ch} channels, span "
          f"{(tr[tr > 0].max() - t0) / 1e3:.1f} us")
    iv = {
        "load lat (issue0->got0)": tr[..., 2] - tr[..., 0],
        "slice arrival (got0->gotN)": tr[..., 3] - tr[..., 2],
        "reduce tail (gotN->pushed)": tr[..., 4] - tr[..., 3],
        "  last chunk (gotN->reduced)": tr[..., 8] - tr[..., 3],
        "  fold (reduced->summed)": tr[..., 9] - tr[..., 8],
        "  slot wait (summed->slotfree)": tr[..., 10] - tr[..., 9],
        "  push (slotfree->pushed)": tr[..., 4] - tr[..., 10],
        "exchange (pushed->gathered)": tr[..., 5] - tr[..., 4],
        "to apply (gathered->apply0)": tr[..., 6] - tr[..., 5],
        "  coefs (gathered->published)": tr[..., 11] - tr[..., 5],
        "  wake (published->apply0)": tr[..., 6] - tr[..., 11],
        "apply (apply0->applyN)": tr[..., 7] - tr[..., 6],
        "residence (issue0->applyN)": tr[..., 7] - tr[..., 0],
    }
    first = np.where(valid[:, 0], tr[:, 0, 0], 0)
    last = tr[..., 7].max(axis=1)
    ok = valid[:, 0]
    print(f"  CTA first issue after t0: p10 {np.percentile((first[ok] - t0) / 1e3, 10):.2f} p50 "
          f"{np.percentile((first[ok] - t0) / 1e3, 50):.2f} p90 {np.percentile((first[ok] - t0) / 1e3, 90):.2f}"
          f" max {(first[ok] - t0).max() / 1e3:.2f} us; CTA last store: p50 "
          f"{np.percentile((last[ok] - t0) / 1e3, 50):.2f} max {(last[ok] - t0).max() / 1e3:.2f} us")
    for k, v in iv.items():
        x = v[valid] / 1e3
        print(f"  {k:32s} p10 {np.percentile(x, 10):7.2f}  p50 {np.percentile(x, 50):7.2f}  "
              f"p90 {np.percentile(x, 90):7.2f} us")
    step = np.diff(tr[..., 7], axis=1)[valid[:, 1:] & valid[:, :-1]] / 1e3
    if step.size == 0:  # one channel per CTA
        return
    print(f"  {'step (applyN(t)->applyN(t+1))':32s} p10 {np.percentile(step, 10):7.2f}  p50 "
          f"{np.percentile(step, 50):7.2f}  p90 {np.percentile(step, 90):7.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wrn38")
    ap.add_argument("--shape", default=None, help="N,C,HW,dtype (overrides --config)")
    args = ap.parse_args()
    assert int(os.environ.get("IABN_FUSED_DEBUG", "0")) & 4, "set IABN_FUSED_DEBUG=4"
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    import synth_inputs as S
    L.lib.iabn_debug_trace.restype = ctypes.c_size_t
    L.lib.iabn_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    if args.shape:
        n_, c_, hw_, dt_ = args.shape.split(",")
        cfg = dict(N=int(n_), C=int(c_), HW=int(hw_), dtype=dt_)
    else:
        cfg = S.CONFIGS[args.config]
    N, C, HW = cfg["N"], cfg["C"], cfg["HW"]
    dev = torch.device("cuda", 0)
    x = S.make_x(N, C, HW, 1, dtype=cfg["dtype"], device=dev)
    dz = S.make_dz(N, C, HW, 1, dtype=cfg["dtype"], device=dev)
    p = S.make_params(C, 0, device=dev)
    L.lib.iabn_debug_trace_channels.restype = ctypes.c_uint32
    for _ in range(3):
        z, sm, sv = P.forward(x, p.gamma, p.beta, p.running_mean, p.running_var)
        torch.cuda.synchronize()
        trf = dump(L)
        P.backward(z, dz, p.gamma, p.beta, sv)
        torch.cuda.synchronize()
        trb = dump(L)
    d = L.desc(N, C, HW, L.BF16 if cfg["dtype"] == "bf16" else L.F32, L.NCHW)
    for (tr, per), label, pas in ((trf, "forward", 0), (trb, "backward", 1)):
        _, K = L.query_schedule(d, pas)
        report(tr, f"{label} K={K}", per)


if __name__ == "__main__":
    main()
