"""One forward + backward of BN + `act` on one tensor, three times (for ncu launch lists).
    python tools/act_once.py sigmoid NHWC 32x256x3136 [f32|bf16]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402

act, layout, sh = sys.argv[1], sys.argv[2], sys.argv[3]
N, C, HW = (int(v) for v in sh.split("x"))
shape = (N, C, HW) if layout == "NCHW" else (N, HW, C)
dt = torch.bfloat16 if len(sys.argv) > 4 and sys.argv[4] == "bf16" else torch.float32
x = torch.randn(shape, device="cuda").to(dt)
dz = torch.randn(shape, device="cuda").to(dt)
g, b = torch.rand(C, device="cuda") + 0.5, torch.zeros(C, device="cuda")
for _ in range(3):
    z, sm, sv = P.forward(x, g, b, layout=layout, activation=act)
    P.backward(z, dz, g, b, sv, layout=layout, activation=act)
torch.cuda.synchronize()
