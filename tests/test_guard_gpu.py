"""Out-of-bounds and uninitialised-read checks of every kernel family, without a sanitizer.

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset), so
the bounds are checked by the tests themselves:

* guard bands -- every array the library touches (activations, per-channel vectors, the
  workspace) is a view into a larger buffer whose 4 KB before and after hold a byte
  pattern; after a forward + backward every guard byte must be unchanged (a stray store
  by any kernel, in any schedule, lands in a guard);
* poisoned scratch -- the same call with the workspace and the output buffers
  pre-filled with 0x00 and with 0xFF (NaN for both dtypes) must give bit-identical
  results: no kernel may read a workspace slot or an output element before writing it.

Cases: every schedule of tools/sanitize_cases.py (channel-resident 2- and 4-CTA/SM,
covering-range, streaming NCHW/NHWC, grid-resident NHWC, eval) plus the fused-collective
sync over virtual ranks.
"""
from __future__ import annotations

import ctypes

import pytest
import torch

import synth_inputs as S

pytestmark = pytest.mark.gpu

GUARD = 4096
PAT = 0xA5


class Guarded:
    """A CUDA byte buffer with a pattern-filled guard band on each side of the payload."""

    def __init__(self, nbytes: int, fill: int):
        self.n = nbytes
        self.buf = torch.full((GUARD + nbytes + GUARD,), PAT, dtype=torch.uint8, device="cuda")
        self.buf[GUARD:GUARD + nbytes] = fill

    def view(self, dtype, shape):
        return self.buf[GUARD:GUARD + self.n].view(dtype).view(shape)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr() + GUARD

    def intact(self) -> bool:
        g = torch.cat([self.buf[:GUARD], self.buf[GUARD + self.n:]])
        return bool((g == PAT).all().item())


CASES = [
    # name, N, C, HW, dtype, layout, flags, inplace
    ("tiny_f32", 2, 8, 16, "f32", "NCHW", 0, True),
    ("r50s3_f32_fused4", 64, 1024, 196, "f32", "NCHW", 0, True),
    ("bf16_56x56_fused2", 8, 64, 3136, "bf16", "NCHW", 0, False),
    ("bf16_14x14_cover", 16, 96, 196, "bf16", "NCHW", 0, True),
    ("bf16_7x7_cover", 8, 40, 49, "bf16", "NCHW", 0, False),
    ("f32_ragged_stream", 3, 37, 77, "f32", "NCHW", 1 << 8, True),
    ("bf16_nhwc_stream", 8, 64, 784, "bf16", "NHWC", 0, False),
    ("bf16_nhwc_resident", 8, 64, 784, "bf16", "NHWC", 1 << 11, True),
    ("f32_variant_I", 4, 32, 1024, "f32", "NCHW", 1 << 5, True),
]


def _run(N, C, HW, dtype, layout, flags, inplace, fill, emulated_ranks=0):
    from paper_1712_02616_b200 import _lib as L
    tdt = S.DTYPES[dtype]
    b = 4 if dtype == "f32" else 2
    shape = (N, C, HW) if layout == "NCHW" else (N, HW, C)
    E = N * C * HW
    x0 = S.make_x(N, C, HW, 3, layout=layout, dtype=dtype).cuda()
    dz0 = S.make_dz(N, C, HW, 3, layout=layout, dtype=dtype).cuda()
    p = S.make_params(C, 3)
    bufs = {}

    def arr(name, nbytes, dt, shp, init=None, f=fill):
        g = bufs[name] = Guarded(nbytes, f)
        v = g.view(dt, shp)
        if init is not None:
            v.copy_(init)
        return v

    x = arr("x", E * b, tdt, shape, x0)
    z = x if inplace else arr("z", E * b, tdt, shape)
    dz = arr("dz", E * b, tdt, shape, dz0)
    dx = dz if inplace else arr("dx", E * b, tdt, shape)
    g_ = arr("gamma", 4 * C, torch.float32, (C,), p.gamma)
    be = arr("beta", 4 * C, torch.float32, (C,), p.beta)
    rm = arr("rm", 4 * C, torch.float32, (C,), p.running_mean)
    rv = arr("rv", 4 * C, torch.float32, (C,), p.running_var)
    sm = arr("sm", 4 * C, torch.float32, (C,))
    sv = arr("sv", 4 * C, torch.float32, (C,))
    G = max(emulated_ranks, 1)
    dg = arr("dg", 4 * C * G, torch.float32, (G, C))
    db = arr("db", 4 * C * G, torch.float32, (G, C))
    dt_ = L.F32 if dtype == "f32" else L.BF16
    lay = L.NCHW if layout == "NCHW" else L.NHWC
    d = L.desc(N // G, C, HW, dt_, lay)
    dfull = L.desc(N, C, HW, dt_, lay)
    wsb = L.workspace_bytes(dfull)
    ws = arr("ws", wsb, torch.uint8, (wsb,))
    st = torch.cuda.current_stream().cuda_stream
    P_ = ctypes.c_void_p
    if emulated_ranks:
        L.call("iabn_forward_sync_emulated", ctypes.byref(d), G, P_(x.data_ptr()),
               P_(z.data_ptr()), P_(g_.data_ptr()), P_(be.data_ptr()), P_(rm.data_ptr()),
               P_(rv.data_ptr()), P_(sm.data_ptr()), P_(sv.data_ptr()), 0.1, 1e-5, 0.01, flags,
               P_(ws.data_ptr()), wsb, P_(st))
        L.call("iabn_backward_sync_emulated", ctypes.byref(d), G, P_(z.data_ptr()),
               P_(dz.data_ptr()), P_(dx.data_ptr()), P_(g_.data_ptr()), P_(be.data_ptr()), None,
               P_(sv.data_ptr()), P_(dg.data_ptr()), P_(db.data_ptr()), 1e-5, 0.01, flags,
               P_(ws.data_ptr()), wsb, P_(st))
    else:
        L.call("iabn_forward", ctypes.byref(d), P_(x.data_ptr()), P_(z.data_ptr()),
               P_(g_.data_ptr()), P_(be.data_ptr()), P_(rm.data_ptr()), P_(rv.data_ptr()),
               P_(sm.data_ptr()), P_(sv.data_ptr()), 0.1, 1e-5, 0.01, flags, P_(ws.data_ptr()),
               wsb, P_(st))
        L.call("iabn_backward", ctypes.byref(d), P_(z.data_ptr()), P_(dz.data_ptr()),
               P_(dx.data_ptr()), P_(g_.data_ptr()), P_(be.data_ptr()), P_(sm.data_ptr()),
               P_(sv.data_ptr()), P_(dg.data_ptr()), P_(db.data_ptr()), 1e-5, 0.01, flags,
               P_(ws.data_ptr()), wsb, P_(st))
        # eval-mode forward over the output (running statistics; streaming apply)
        ze = arr("ze", E * b, tdt, shape)
        L.call("iabn_forward", ctypes.byref(d), P_(z.data_ptr()), P_(ze.data_ptr()),
               P_(g_.data_ptr()), P_(be.data_ptr()), P_(rm.data_ptr()), P_(rv.data_ptr()),
               None, None, 0.1, 1e-5, 0.01, flags | L.EVAL, P_(ws.data_ptr()), wsb, P_(st))
    torch.cuda.synchronize()
    bad = [k for k, v in bufs.items() if not v.intact()]
    assert not bad, f"guard band overwritten: {bad}"
    out = {k: v.clone() for k, v in dict(z=z, dx=dx, sm=sm, sv=sv, rm=rm, rv=rv, dg=dg,
                                         db=db).items()}
    if not emulated_ranks:
        out["ze"] = bufs["ze"].view(tdt, shape).clone()
    return out


def _same(a, b):
    for k in a:
        assert torch.equal(a[k].view(torch.uint8), b[k].view(torch.uint8)), \
            f"{k} depends on the initial contents of the scratch / output buffers"


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_guards_and_poisoned_scratch(case):
    _, N, C, HW, dtype, layout, flags, inplace = case
    a = _run(N, C, HW, dtype, layout, flags, inplace, 0x00)
    b = _run(N, C, HW, dtype, layout, flags, inplace, 0xFF)
    _same(a, b)


@pytest.mark.parametrize("G,N,C,HW,dtype", [(2, 8, 24, 196, "bf16"), (4, 8, 16, 1024, "f32")],
                         ids=["G2_bf16_cover", "G4_f32"])
def test_guards_sync_emulated(G, N, C, HW, dtype):
    a = _run(N, C, HW, dtype, "NCHW", 0, True, 0x00, emulated_ranks=G)
    b = _run(N, C, HW, dtype, "NCHW", 0, True, 0xFF, emulated_ranks=G)
    _same(a, b)
