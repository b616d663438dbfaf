"""Host cost of one forward + backward call pair through the Python binding and
through the raw C ABI (ctypes, arguments prepared once), vs the device time of the
same work, for a small layer (ResNeXt-101 Conv4: 32 x 1024 x 7 x 7).

    python tools/call_overhead.py
"""
import ctypes
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402

N, C, HW = 32, 1024, 49
dev = torch.device("cuda", 0)
x = torch.randn(N, C, HW, device=dev)
dz = torch.randn(N, C, HW, device=dev)
g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
rm, rv = torch.zeros(C, device=dev), torch.ones(C, device=dev)
sm, sv, dg, db = (torch.empty(C, device=dev) for _ in range(4))
d = L.desc(N, C, HW, L.F32, L.NCHW)
ws = torch.zeros(L.workspace_bytes(d), dtype=torch.uint8, device=dev)
st = torch.cuda.current_stream().cuda_stream
fa = [ctypes.byref(d), x.data_ptr(), x.data_ptr(), g.data_ptr(), b.data_ptr(), rm.data_ptr(),
      rv.data_ptr(), sm.data_ptr(), sv.data_ptr(), 0.1, 1e-5, 0.01, 0, ws.data_ptr(), ws.numel(), st]
ba = [ctypes.byref(d), x.data_ptr(), dz.data_ptr(), dz.data_ptr(), g.data_ptr(), b.data_ptr(),
      None, sv.data_ptr(), dg.data_ptr(), db.data_ptr(), 1e-5, 0.01, 0, ws.data_ptr(),
      ws.numel(), st]


def python_api():
    z, _, v = P.forward(x, g, b, rm, rv)
    P.backward(z, dz, g, b, v)


def raw_abi():
    L.lib.iabn_forward(*fa)
    L.lib.iabn_backward(*ba)


res = {}
for name, fn in (("python_api", python_api), ("raw_c_abi", raw_abi)):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    n = 2000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(n):
        fn()
    t_host = (time.perf_counter() - t0) / n * 1e6
    e1.record()
    torch.cuda.synchronize()
    res[name] = dict(host_us_per_pair=round(t_host, 2),
                     wall_us_per_pair=round(e0.elapsed_time(e1) / n * 1e3, 2))
# device time alone: a CUDA graph of the pair
gph = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    python_api()
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(gph):
    python_api()
for _ in range(20):
    gph.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(500):
    gph.replay()
e1.record()
torch.cuda.synchronize()
res["graph_device_us_per_pair"] = round(e0.elapsed_time(e1) / 500 * 1e3, 2)
# Host cost per call without back-pressure: the loops above enqueue thousands of
# launches, so the launch queue fills and the host time tracks the device time.  Here
# short bursts (the queue never fills; the GPU is idle at the start of each burst),
# per entry point, with the kernels each call launches.
def raw_fwd():
    L.lib.iabn_forward(*fa)


def raw_bwd():
    L.lib.iabn_backward(*ba)


def py_fwd():
    P.forward(x, g, b, rm, rv)


def py_bwd():
    P.backward(x, dz, g, b, sv)


burst = {}
for name, fn in (("raw_forward", raw_fwd), ("raw_backward", raw_bwd), ("python_forward", py_fwd),
                 ("python_backward", py_bwd)):
    ts = []
    for _ in range(40):
        torch.cuda.synchronize()
        k0 = L.launch_count()
        t0 = time.perf_counter()
        for _ in range(8):
            fn()
        ts.append((time.perf_counter() - t0) / 8 * 1e6)
        k = (L.launch_count() - k0) / 8
    ts.sort()
    burst[name] = dict(host_us_per_call_median=round(ts[len(ts) // 2], 2),
                       host_us_per_call_min=round(ts[0], 2), kernels_per_call=k)
torch.cuda.synchronize()
res["burst_of_8_calls"] = burst
print(json.dumps(dict(shape=[N, C, HW], **res)))
