"""One NHWC layer's forward + backward (experiments: run under ncu for per-kernel times).

    python tools/nhwc_probe.py N HW C dtype [flags]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

N, HW, C = (int(v) for v in sys.argv[1:4])
dt = torch.bfloat16 if sys.argv[4] == "bf16" else torch.float32
fl = int(sys.argv[5]) if len(sys.argv) > 5 else 0
dev = torch.device("cuda", 0)
x = torch.randn(N, HW, C, device=dev).to(dt)
dz = torch.randn(N, HW, C, device=dev).to(dt)
g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
for _ in range(3):
    z, sm, sv = P.forward(x, g, b, layout="NHWC", flags=fl)
    P.backward(z, dz, g, b, sv, layout="NHWC", dx=torch.empty_like(dz), flags=fl)
torch.cuda.synchronize()
