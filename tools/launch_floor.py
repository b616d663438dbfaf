"""Device-time floor of one forward / backward call per schedule on a tiny and a
small layer (CUDA-graph replay, so host cost is excluded).

    python tools/launch_floor.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402

dev = torch.device("cuda", 0)
res = {}
for (N, C, HW, dt) in ((2, 8, 256, torch.float32), (32, 512, 196, torch.float32),
                       (32, 512, 256, torch.bfloat16), (32, 128, 784, torch.bfloat16)):
    x = torch.randn(N, C, HW, device=dev).to(dt)
    dz = torch.randn(N, C, HW, device=dev).to(dt)
    g, b = torch.rand(C, device=dev) + 0.5, torch.zeros(C, device=dev)
    for name, fl in (("auto", 0), ("streaming", L.FORCE_STREAMING)):
        def fwd():
            return P.forward(x, g, b, flags=fl)

        z, sm, sv = fwd()
        def bwd():
            P.backward(z, dz, g, b, sv, flags=fl)
        out = {}
        for pname, fn in (("fwd", fwd), ("bwd", bwd)):
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                fn()
            torch.cuda.current_stream().wait_stream(s)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for _ in range(20):
                    fn()
            gr.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                gr.replay()
            e1.record()
            torch.cuda.synchronize()
            out[pname + "_us"] = round(e0.elapsed_time(e1) / 200 * 1e3, 2)
        res[f"{N}x{C}x{HW}_{str(dt)[6:]}_{name}"] = out
print(json.dumps(res, indent=1))
