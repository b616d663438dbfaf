"""One fused-collective sync fwd + bwd over 2 virtual ranks (for profiler runs)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402
import synth_inputs as S  # noqa: E402

print({k: v[:80] for k, v in os.environ.items() if "INJECT" in k or k.startswith("NV_") or "NSIGHT" in k})
N, C, HW = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
G = int(sys.argv[4]) if len(sys.argv) > 4 else 2
x = S.make_x(N, C, HW, 5, dtype="bf16").cuda()
dz = S.make_dz(N, C, HW, 5, dtype="bf16").cuda()
p = S.make_params(C, 5)
g, b = p.gamma.cuda(), p.beta.cuda()
for _ in range(2):
    z, sm, sv = P.forward_sync_emulated(x.clone(), G, g, b)
    dx, dg, db = P.backward_sync_emulated(z, dz.clone(), G, g, b, sv)
torch.cuda.synchronize()
print("emu ok", float(dx.float().abs().sum()))
