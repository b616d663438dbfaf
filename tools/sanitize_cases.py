"""Small cases of every schedule, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck --error-exitcode 3 python tools/sanitize_cases.py [--no-sync]

One forward + backward per case through the C ABI (functional.py), each a different
kernel family: the channel-resident kernels (4-CTA/SM and 2-CTA/SM variants, aligned and
covering-range planes), the streaming kernels (NCHW ragged, NHWC), the grid-resident NHWC
schedule, eval mode, and the fused-collective sync over virtual ranks (one cooperative
launch; --no-sync skips it for the slow racecheck tool, whose instrumentation can stretch
the cross-cluster waits toward the 20 s trap).  Outputs are checked only for finiteness
here; parity is the job of tests/.
"""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1712_02616_b200 as P  # noqa: E402
from paper_1712_02616_b200 import _lib as L  # noqa: E402
import synth_inputs as S  # noqa: E402

CASES = [
    # name, N, C, HW, dtype, layout, flags
    ("cfg1 tiny f32", 2, 8, 16, "f32", "NCHW", 0),
    ("cfg2 r50s3 f32 (fused, 4 CTA/SM)", 64, 1024, 196, "f32", "NCHW", 0),
    ("bf16 56x56 (fused, 2 CTA/SM)", 8, 64, 3136, "bf16", "NCHW", 0),
    ("bf16 14x14 (covering-range)", 16, 96, 196, "bf16", "NCHW", 0),
    ("bf16 7x7 (covering-range)", 8, 40, 49, "bf16", "NCHW", 0),
    ("f32 ragged (streaming)", 3, 37, 77, "f32", "NCHW", L.FORCE_STREAMING),
    ("bf16 NHWC (streaming)", 8, 64, 784, "bf16", "NHWC", 0),
    ("bf16 NHWC (grid-resident)", 8, 64, 784, "bf16", "NHWC", L.FORCE_RESIDENT),
    ("f32 variant I (fused)", 4, 32, 1024, "f32", "NCHW", L.VARIANT_I),
]


def run_case(name, N, C, HW, dtype, layout, flags):
    x = S.make_x(N, C, HW, 1, layout=layout, dtype=dtype).cuda()
    dz = S.make_dz(N, C, HW, 1, layout=layout, dtype=dtype).cuda()
    p = S.make_params(C, 1)
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    z, sm, sv = P.forward(x, g, b, rm, rv, layout=layout, flags=flags)
    dx, dg, db = P.backward(z, dz, g, b, sv, layout=layout, flags=flags)
    ze, _, _ = P.forward(z.clone(), g, b, rm, rv, layout=layout, training=False)
    torch.cuda.synchronize()
    for t in (z, dx, dg, db, ze):
        assert torch.isfinite(t.float()).all(), name
    print(f"ok  {name}", flush=True)


def run_sync(G, N, C, HW, dtype):
    x = S.make_x(N * G, C, HW, 2, dtype=dtype).cuda()
    dz = S.make_dz(N * G, C, HW, 2, dtype=dtype).cuda()
    p = S.make_params(C, 2)
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    z, sm, sv = P.forward_sync_emulated(x, G, g, b, rm, rv)
    dx, dg, db = P.backward_sync_emulated(z, dz, G, g, b, sv)
    torch.cuda.synchronize()
    assert torch.isfinite(dx.float()).all()
    print(f"ok  sync emulated G={G} {N}x{C}x{HW} {dtype}", flush=True)


def main():
    torch.cuda.set_device(0)
    for c in CASES:
        run_case(*c)
    if "--no-sync" not in sys.argv:
        run_sync(2, 4, 24, 196, "bf16")
        run_sync(4, 2, 16, 1024, "f32")
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
