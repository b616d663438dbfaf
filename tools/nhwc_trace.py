"""Phase timeline of the NHWC channel-group kernel (IABN_NHWC_TRACE=1): per CTA
%globaltimer stamps of start, PDL wait, loads issued, last box landed, reduce folded,
records exchanged, coefficients, applied, stores issued, exit -- median and max over CTAs,
in ns from the earliest start.

    IABN_NHWC_TRACE=1 python tools/nhwc_trace.py C HW dtype [pass] [N]
"""
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402

C, HW = int(sys.argv[1]), int(sys.argv[2])
dt = torch.bfloat16 if sys.argv[3] == "bf16" else torch.float32
pass_ = int(sys.argv[4]) if len(sys.argv) > 4 else 0
N = int(sys.argv[5]) if len(sys.argv) > 5 else 32
dev = torch.device("cuda", 0)
x = torch.randn(N, HW, C, device=dev).to(dt)
dz = torch.randn(N, HW, C, device=dev).to(dt)
g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
out = torch.empty_like(x)
for _ in range(3):
    z, sm, sv = P.forward(x, g, b, layout="NHWC", out=out)
    if pass_ == 1:
        P.backward(out, dz, g, b, sv, layout="NHWC", dx=x)
torch.cuda.synchronize()
fn = L.lib.iabn_debug_trace
fn.restype = ctypes.c_size_t
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_size_t]
n = fn(None, 0)
buf = (ctypes.c_ulonglong * n)()
fn(buf, n)
F = 10
rows = [list(buf[i * F:(i + 1) * F]) for i in range(n // F)]
rows = [r for r in rows if r[0]]
t0 = min(r[0] for r in rows)
names = ["start", "pdl_wait", "loads_issued", "last_box", "reduced", "exchanged", "coef",
         "applied", "stores_issued", "exit"]
print(f"{len(rows)} CTAs, C={C} HW={HW} N={N} {sys.argv[3]} pass={pass_}")
for k, nm in enumerate(names):
    v = [r[k] - t0 for r in rows if r[k]]
    if v:
        print(f"{nm:14s} median {statistics.median(v):8.0f} ns   max {max(v):8.0f} ns")
