"""Phase timeline of the register-resident small-layer kernel (IABN_SMALL_TRACE=1): per
CTA %globaltimer stamps (start, PDL wait, sums done, team partials, coefficients, stores
issued) -- median and max over CTAs in ns from the earliest start, for the last of
three calls (L2-cold inputs: a fresh tensor per call).

    IABN_SMALL_TRACE=1 python tools/small_trace.py C HW dtype [pass] [N]
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
g, b = torch.rand(C, device="cuda") + 0.5, torch.zeros(C, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    x = torch.randn(N, C, HW, device="cuda").to(dt)
    dz = torch.randn(N, C, HW, device="cuda").to(dt)
    z, sm, sv = P.forward(x, g, b, out=torch.empty_like(x)) if pass_ == 1 else (x, None, None)
    flush.zero_()
    if pass_ == 0:
        P.forward(x, g, b)
    else:
        P.backward(z, dz, g, b, sv)
torch.cuda.synchronize()
fn = L.lib.iabn_debug_trace
fn.restype = ctypes.c_size_t
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_size_t]
F = L.lib.iabn_debug_trace_channels()
n = fn(None, 0)
buf = (ctypes.c_ulonglong * n)()
fn(buf, n)
rows = [list(buf[i * F:(i + 1) * F]) for i in range(n // F)]
rows = [r for r in rows if r[0]]
t0 = min(r[0] for r in rows)
names = ["start", "pdl_wait", "sums_done", "team_partials", "coefficients", "stores_issued"]
print(f"{len(rows)} CTAs, C={C} HW={HW} N={N} {sys.argv[3]} pass={pass_}")
for k in range(F):
    v = [r[k] - t0 for r in rows if r[k]]
    if v:
        print(f"{names[k]:14s} median {statistics.median(v):8.0f} ns   max {max(v):8.0f} ns")
