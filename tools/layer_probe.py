"""Run one BN+Act layer fwd+bwd a few times (for ncu launch lists of a single shape).

    python tools/layer_probe.py N C HW dtype layout [flags]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

N, C, HW = (int(v) for v in sys.argv[1:4])
dt = torch.float32 if sys.argv[4] == "f32" else torch.bfloat16
layout = sys.argv[5]
flags = int(sys.argv[6]) if len(sys.argv) > 6 else 0
dev = torch.device("cuda", 0)
shape = (N, C, HW) if layout == "NCHW" else (N, HW, C)
x = torch.randn(shape, device=dev).to(dt)
dz = torch.randn(shape, device=dev).to(dt)
g, b = torch.rand(C, device=dev) + 0.5, torch.randn(C, device=dev) * 0.1
for _ in range(3):
    z, sm, sv = P.forward(x, g, b, layout=layout, flags=flags)
    P.backward(z, dz, g, b, sv, layout=layout, flags=flags)
torch.cuda.synchronize()
print("ok")
