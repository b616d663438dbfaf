"""Parity of the register-resident schedule for small NCHW layers (csrc/kernels_small.cuh)
against the oracle: aligned and misaligned planes (bf16 14x14 = 392 B, 7x7 = 98 B; fp32
7x7 = 196 B), teams of 1-8 warps per channel, channels not a multiple of the channels
per CTA, both backward variants, in and out of place, stress inputs.  The schedule is
forced on (test hook ``iabn_debug_small``, not part of include/iabn.h) for shapes above
its size threshold too; the default choice is covered by the layer-shape tests."""
from __future__ import annotations

import ctypes

import pytest
import torch

from tests.harness import Case, compare, inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

VARIANT_I = 1 << 5


@pytest.fixture(params=[4, 8], ids=["R4", "R8"])
def small(request):
    from paper_1712_02616_b200 import _lib as L
    f, fr = L.lib.iabn_debug_small, L.lib.iabn_debug_small_r
    for h in (f, fr):
        h.argtypes = [ctypes.c_int]
        h.restype = None
    f(1)
    fr(request.param)
    yield
    f(0)
    fr(0)


CASES = [
    Case(32, 24, 196, dtype="bf16", seed=130),   # 392 B planes, tw = 4
    Case(32, 40, 49, dtype="bf16", seed=131),    # 98 B planes, tw = 1
    Case(32, 12, 49, dtype="f32", seed=132),     # 196 B planes
    Case(16, 20, 196, dtype="f32", seed=133),    # aligned 784 B planes, tw = 4
    Case(8, 9, 100, dtype="bf16", seed=134),     # ragged: 200 B planes, few samples
    Case(64, 6, 49, dtype="bf16", seed=135),     # tw = 2
    Case(2, 5, 8, dtype="f32", seed=136),        # tiny
    Case(32, 8, 49, dtype="bf16", stress="offset", seed=137),
    Case(32, 8, 196, dtype="f32", stress="constant", seed=138),
]


@pytest.mark.parametrize("variant", [0, VARIANT_I], ids=["II", "I"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c.dtype}_{c.N}x{c.C}x{c.HW}" +
                         (f"_{c.stress}" if c.stress else ""))
def test_small_layers(case, variant, small):
    from paper_1712_02616_b200 import _lib as L
    d = L.desc(case.N, case.C, case.HW, L.BF16 if case.dtype == "bf16" else L.F32, L.NCHW)
    assert L.query_schedule(d, 0)[0] == 5 and L.query_schedule(d, 1)[0] == 5
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    compare(case, run_gpu(case, x, dz, p, flags=variant), ref, p)
    compare(case, run_gpu(case, x, dz, p, flags=variant, inplace=False, dx_inplace=False), ref, p)


def test_small_layers_bitwise_in_place_and_repeat(small):
    case = Case(32, 64, 196, dtype="bf16", seed=139)
    x, dz, p = inputs(case)
    a = run_gpu(case, x, dz, p)
    b = run_gpu(case, x, dz, p, inplace=False, dx_inplace=False)
    c = run_gpu(case, x, dz, p)
    for k in a:
        assert torch.equal(a[k], b[k]) and torch.equal(a[k], c[k]), k
