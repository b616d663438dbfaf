"""NHWC streaming schedule with the bulk-ring reductions (kernels_nhwc_bulk.cuh: TMA
bulk copies of round-robin row chunks, 8-CTA cluster records over DSMEM) against the
oracle: every thread mapping (rt row lanes x cv vectors: cv = 1 .. 256), ragged row
chunks, both backward variants (II by default, I with IABN_VARIANT_I), both dtypes, and
the BN-dagger cancellation at |beta / gamma| = 20 in bf16."""
from __future__ import annotations

import ctypes

import pytest

from tests.harness import Case, compare, inputs, run_gpu, run_oracle, to64
from tests.util import chan_err, vec_err

pytestmark = pytest.mark.gpu

STREAM = 1 << 8
VARIANT_I = 1 << 5


def nb_records(case: Case) -> int:
    from paper_1712_02616_b200 import _lib as L
    f = L.lib.iabn_debug_nb_records
    f.argtypes = [ctypes.c_void_p]
    f.restype = ctypes.c_int
    d = L.desc(case.N, case.C, case.HW, L.BF16 if case.dtype == "bf16" else L.F32, L.NHWC)
    return f(ctypes.addressof(d))


CASES = [Case(4, 8, 3136, dtype="bf16", seed=110, layout="NHWC"),     # cv = 1, 256 row lanes
         Case(6, 96, 784, dtype="bf16", seed=111, layout="NHWC"),     # cv = 12, 21 lanes
         Case(4, 24, 3000, dtype="f32", seed=112, layout="NHWC"),     # cv = 6, ragged chunks
         Case(8, 128, 784, dtype="bf16", seed=113, layout="NHWC"),    # cv = 16
         Case(8, 1216, 49, dtype="bf16", seed=114, layout="NHWC"),    # cv = 152, one lane
         Case(4, 2048, 49, dtype="bf16", seed=115, layout="NHWC"),    # cv = 256
         Case(4, 1024, 60, dtype="f32", seed=116, layout="NHWC"),     # cv = 256, f32
         Case(3, 200, 333, dtype="f32", seed=117, layout="NHWC")]     # cv = 50, odd rows
IDS = ["cv1", "cv12", "cv6_ragged", "cv16", "cv152", "cv256_bf16", "cv256_f32", "cv50"]


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("flags", [STREAM, STREAM | VARIANT_I], ids=["II", "I"])
def test_nhwc_bulk_streaming_matches_oracle(case, flags):
    assert nb_records(case) > 0, "shape does not reach the bulk-ring reductions"
    x, dz, p = inputs(case)
    compare(case, run_gpu(case, x, dz, p, flags=flags), run_oracle(case, x, dz, p), p)


def test_nhwc_bulk_not_taken_for_wide_rows_and_tiny_tensors():
    assert nb_records(Case(4, 2080, 49, dtype="bf16", layout="NHWC")) == 0  # > 4 KB rows
    assert nb_records(Case(2, 8, 16, dtype="f32", layout="NHWC")) == 0      # < 8 stages
    assert nb_records(Case(32, 128, 3136, dtype="bf16", layout="NHWC")) == 32


@pytest.mark.parametrize("flags", [STREAM, STREAM | VARIANT_I], ids=["II", "I"])
def test_nhwc_bulk_large_beta_over_gamma_bf16(flags):
    """|beta / gamma| = 20, bf16 storage, NHWC streaming: the BN-dagger form
    (Q - beta S1)/g of the bulk-ring reduction against the oracle's Alg. 2 from the GPU's
    own rounded z (as tests/test_parity_gpu.py::test_large_beta_over_gamma_bf16)."""
    import oracle
    case = Case(8, 64, 784, dtype="bf16", seed=118, layout="NHWC")
    assert nb_records(case) > 0
    x, dz, p = inputs(case)
    p.beta = (20.0 * p.gamma.abs()).contiguous()
    got = run_gpu(case, x, dz, p, flags=flags)
    o = oracle.load()
    dx, dg, db = o.backward_inplace_I(to64(got["z"]), to64(dz), to64(got["var"]), to64(p.gamma),
                                      to64(p.beta), eps=case.eps, slope=case.slope,
                                      layout="NHWC")
    assert chan_err(to64(got["dx"]), dx, 2) < 2e-2
    assert vec_err(to64(got["dgamma"]), dg) < 1e-4 and vec_err(to64(got["dbeta"]), db) < 1e-4
