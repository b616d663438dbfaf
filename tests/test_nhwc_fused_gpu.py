"""Parity of the NHWC channel-group-resident schedule (csrc/kernels_nhwc.cuh) against the
oracle: every group width g (16..256 bytes of a row), cluster size K = 1..8, persistent
clusters looping over several groups, partial last groups (C not a multiple of g),
ragged row splits, both dtypes, both backward variants, in and out of place.

The plan is forced through the library's test hook ``iabn_debug_nhwc_plan`` (not part of
include/iabn.h); the default planner's choice is covered by every NHWC case of the other
parity tests (tests/test_parity_gpu.py, tests/test_parity_networks_gpu.py).
"""
from __future__ import annotations

import ctypes

import pytest
import torch

from tests.harness import Case, compare, inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

VARIANT_I = 1 << 5


def _hook():
    from paper_1712_02616_b200 import _lib as L
    f = L.lib.iabn_debug_nhwc_plan
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
    f.restype = None
    return f


@pytest.fixture
def plan():
    f = _hook()
    yield f
    f(0, 0, 0)


def _schedule(case):
    from paper_1712_02616_b200 import _lib as L
    d = L.desc(case.N, case.C, case.HW, L.BF16 if case.dtype == "bf16" else L.F32, L.NHWC)
    return L.query_schedule(d, 0), L.query_schedule(d, 1)


CASES = [
    # (case, g, K, clusters)
    (Case(4, 64, 49, dtype="bf16", layout="NHWC", seed=90), 8, 1, 0),
    (Case(4, 64, 49, dtype="bf16", layout="NHWC", seed=90), 16, 2, 0),
    (Case(4, 64, 49, dtype="bf16", layout="NHWC", seed=90), 32, 4, 0),
    (Case(4, 64, 49, dtype="bf16", layout="NHWC", seed=90), 64, 8, 0),
    (Case(8, 256, 196, dtype="bf16", layout="NHWC", seed=91), 128, 8, 0),   # g*b = 256 B
    (Case(8, 96, 196, dtype="bf16", layout="NHWC", seed=92), 64, 4, 0),     # partial group
    (Case(8, 96, 196, dtype="bf16", layout="NHWC", seed=92), 8, 5, 3),      # persistent
    (Case(3, 40, 77, dtype="f32", layout="NHWC", seed=93), 4, 7, 0),        # ragged rows
    (Case(3, 40, 77, dtype="f32", layout="NHWC", seed=93), 8, 1, 2),        # persistent
    (Case(16, 128, 196, dtype="f32", layout="NHWC", seed=94), 32, 8, 0),
    (Case(16, 128, 196, dtype="f32", layout="NHWC", seed=94), 8, 3, 0),
    (Case(2, 1024, 9, dtype="f32", layout="NHWC", seed=95), 64, 1, 5),      # few rows, wide
    (Case(32, 128, 49, dtype="bf16", layout="NHWC", seed=96), 0, 0, 0),     # planner's choice
    (Case(5, 24, 7, dtype="f32", layout="NHWC", stress="offset", seed=97), 8, 2, 0),
    (Case(6, 16, 31, dtype="bf16", layout="NHWC", stress="constant", seed=98), 8, 3, 0),
]


@pytest.mark.parametrize("variant", [0, VARIANT_I], ids=["II", "I"])
@pytest.mark.parametrize("cfg", CASES,
                         ids=[f"{c.dtype}_{c.N}x{c.C}x{c.HW}_g{g}_K{k}_q{q}" + (f"_{c.stress}" if c.stress else "")
                              for c, g, k, q in CASES])
def test_nhwc_channel_groups(cfg, variant, plan):
    case, g, K, clusters = cfg
    plan(g, K, clusters)
    (s0, k0), (s1, k1) = _schedule(case)
    assert s0 == 4 and s1 == 4, "expected the channel-group NHWC schedule"
    if K:
        assert k0 == K and k1 == K
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    compare(case, run_gpu(case, x, dz, p, flags=variant), ref, p)
    compare(case, run_gpu(case, x, dz, p, flags=variant, inplace=False, dx_inplace=False), ref, p)


def test_nhwc_in_place_bitwise_equals_out_of_place(plan):
    case = Case(8, 64, 196, dtype="bf16", layout="NHWC", seed=99)
    plan(16, 4, 0)
    x, dz, p = inputs(case)
    a = run_gpu(case, x, dz, p)
    b = run_gpu(case, x, dz, p, inplace=False, dx_inplace=False)
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_nhwc_deterministic_across_plans_of_same_k(plan):
    """Repeated calls are bitwise identical (fixed fold order)."""
    case = Case(8, 128, 784, dtype="bf16", layout="NHWC", seed=100)
    x, dz, p = inputs(case)
    plan(32, 4, 0)
    a = run_gpu(case, x, dz, p)
    b = run_gpu(case, x, dz, p)
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_nhwc_falls_back_when_rows_not_16B(plan):
    """C*b not a multiple of 16: no 2-D TMA map; the streaming kernels run."""
    case = Case(3, 37, 10, layout="NHWC", seed=101)
    assert _schedule(case)[0][0] == 0
    x, dz, p = inputs(case)
    compare(case, run_gpu(case, x, dz, p), run_oracle(case, x, dz, p), p)
