"""B200 analogue of the paper's timing / memory study (Fig. 4):
forward + backward through BN+Act+Conv blocks at the ResNeXt-101 stage shapes,
batch 32, averaged over 200 iterations, for three BN strategies:

  standard       torch BatchNorm2d + LeakyReLU (x, the BN output and z are kept)
  inplace_abn    this library's InPlace-ABN (z written over x; backward from z)
  checkpointing  torch BatchNorm2d + LeakyReLU under torch.utils.checkpoint
                 (only x kept; BN+Act recomputed in the backward)

Block (our reading; the paper does not give the exact module): conv_a -> BN+Act ->
conv_b, with conv_a a 1x1 conv producing the stage width W and conv_b the grouped
3x3 conv (32 groups) of a ResNeXt-101 32x4d bottleneck; stages W = 128, 256, 512,
1024 at 56^2, 28^2, 14^2, 7^2 (Conv1-Conv4).  The convolutions are cuDNN (library
code, identical in all three); only the BN+Act differs.  Reported: mean fwd+bwd
time (CUDA events; eager, and the same step replayed from a CUDA graph), its
increase over `standard`, and the peak memory of one
forward+backward above the resident parameters and input.

    python tools/fig4_blocks.py [--dtype f32|bf16] [--iters 200]
"""
import argparse
import json
import os
import sys

import torch
import torch.nn.functional as F
from torch.utils.checkpoint import checkpoint

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1712_02616_b200 import InPlaceABN  # noqa: E402

STAGES = [("Conv1", 128, 56), ("Conv2", 256, 28), ("Conv3", 512, 14), ("Conv4", 1024, 7)]


class Block(torch.nn.Module):
    def __init__(self, width, strategy, dtype, device):
        super().__init__()
        self.strategy = strategy
        self.conv_a = torch.nn.Conv2d(2 * width, width, 1, bias=False, device=device, dtype=dtype)
        self.conv_b = torch.nn.Conv2d(width, width, 3, padding=1, groups=32, bias=False,
                                      device=device, dtype=dtype)
        if strategy == "inplace_abn":
            self.bn = InPlaceABN(width, slope=0.01, device=device)
        else:
            self.bn = torch.nn.BatchNorm2d(width, device=device, dtype=torch.float32)

    def bn_act(self, x):
        if self.strategy == "inplace_abn":
            return self.bn(x)
        return F.leaky_relu(self.bn(x), 0.01)

    def forward(self, inp):
        x = self.conv_a(inp)
        if self.strategy == "checkpointing":
            z = checkpoint(self.bn_act, x, use_reentrant=False)
        else:
            z = self.bn_act(x)
        return self.conv_b(z)


def measure(width, hw, strategy, dtype, iters, device):
    torch.manual_seed(0)
    blk = Block(width, strategy, dtype, device)
    inp = torch.randn(32, 2 * width, hw, hw, device=device, dtype=dtype)
    gout = torch.randn(32, width, hw, hw, device=device, dtype=dtype)

    def step():
        out = blk(inp)
        out.backward(gout)

    for _ in range(10):
        step()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    step()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1) / iters
    # the same step captured in a CUDA graph: device time without the host-side launch
    # cost (at 14^2 and 7^2 the eager steps are bound by it in every variant)
    graph_ms, graph_err = None, None
    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(3):
                step()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph_ms = e0.elapsed_time(e1) / iters
    except Exception as e:  # reported, not hidden
        graph_err = f"{type(e).__name__}: {e}"[:200]
    return eager_ms, peak, graph_ms, graph_err


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    dtype = torch.float32 if args.dtype == "f32" else torch.bfloat16
    dev = torch.device("cuda", 0)
    torch.backends.cudnn.benchmark = True
    rows = []
    for name, width, hw in STAGES:
        res = {}
        for strategy in ("standard", "inplace_abn", "checkpointing"):
            ms, peak, gms, gerr = measure(width, hw, strategy, dtype, args.iters, dev)
            res[strategy] = dict(ms=round(ms, 4), peak_mb=round(peak / 2**20, 1),
                                 graph_ms=None if gms is None else round(gms, 4))
            if gerr:
                res[strategy]["graph_error"] = gerr
        std = res["standard"]
        for s in ("inplace_abn", "checkpointing"):
            res[s]["time_vs_standard_pct"] = round(100 * (res[s]["ms"] / std["ms"] - 1), 1)
            if res[s]["graph_ms"] is not None and std["graph_ms"] is not None:
                res[s]["graph_time_vs_standard_pct"] = round(
                    100 * (res[s]["graph_ms"] / std["graph_ms"] - 1), 1)
            res[s]["memory_vs_standard_pct"] = round(100 * (res[s]["peak_mb"] / std["peak_mb"] - 1), 1)
        rows.append(dict(block=name, width=width, hw=hw, batch=32, **res))
    print(json.dumps(dict(dtype=args.dtype, iters=args.iters, blocks=rows), indent=1))


if __name__ == "__main__":
    main()
