"""Phase timeline of the NHWC bulk-ring reduction (IABN_NB_TRACE=1): per CTA %globaltimer
stamps (start, PDL wait, first chunk, last chunk, loop done, lanes summed, cluster met,
records written) -- median and max over CTAs in ns from the earliest start.

    IABN_NB_TRACE=1 python tools/nb_trace.py C HW dtype [pass] [N]
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
x = torch.randn(N, HW, C, device="cuda").to(dt)
dz = torch.randn(N, HW, C, device="cuda").to(dt)
g, b = torch.rand(C, device="cuda") + 0.5, torch.zeros(C, device="cuda")
for _ in range(3):
    if pass_ == 0:
        P.forward_reduce(x, layout="NHWC")
    else:
        P.backward_reduce(x, dz, g, b, layout="NHWC")
torch.cuda.synchronize()
fn = L.lib.iabn_debug_trace
fn.restype = ctypes.c_size_t
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_size_t]
F = L.lib.iabn_debug_trace_channels()
n = fn(None, 0)
buf = (ctypes.c_ulonglong * n)()
fn(buf, n)
rows = [list(buf[i * F:(i + 1) * F]) for i in range(n // F)]
t0 = min(r[0] for r in rows)
names = ["start", "pdl_wait", "first_chunk", "last_chunk", "loop_done", "lanes_summed",
         "cluster_met", "records"]
print(f"{len(rows)} CTAs, C={C} HW={HW} N={N} {sys.argv[3]} pass={pass_}")
for k in range(F):
    v = [r[k] - t0 for r in rows]
    print(f"{names[k]:14s} median {statistics.median(v):8.0f} ns   max {max(v):8.0f} ns")
