"""Test-of-tests on the GPU (fault injection): the parity harness must
FAIL when the library's output is wrong by a small amount.

``iabn_debug_fault`` (a debug export of libiabn.so, not part of include/iabn.h) makes every
later call perturb one of its outputs -- dgamma x 1.001, running_var x 1.001, or the first
element of z / dx (x 1.01 + 1e-2 in fp32: above the tolerance even where the R16
allowance of a channel with undecidable activation branches applies) -- after the real
kernels ran.  With the fault armed,
``tests.harness.compare`` against the oracle must raise; disarmed, the same case passes.
"""
from __future__ import annotations

import ctypes

import pytest

from tests.harness import Case, compare, inputs, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

FAULTS = {"dgamma": 1, "z": 2, "dx": 4, "running_var": 8}


def _lib():
    from paper_1712_02616_b200 import _lib as L
    f = L.lib.iabn_debug_fault
    f.argtypes = [ctypes.c_uint32]
    f.restype = None
    return f


@pytest.fixture
def fault():
    f = _lib()
    yield f
    f(0)


@pytest.mark.parametrize("case", [Case(8, 64, 1024, seed=80),                      # fused
                                  Case(3, 37, 77, seed=81),                        # streaming
                                  Case(8, 32, 196, dtype="bf16", seed=82),         # small layer
                                  Case(48, 32, 196, dtype="bf16", seed=84)],       # covering
                         ids=["f32_fused", "f32_streaming", "bf16_small", "bf16_cover"])
@pytest.mark.parametrize("what", sorted(FAULTS))
def test_harness_catches_injected_fault(case, what, fault):
    if case.dtype == "bf16" and what in ("dgamma", "running_var"):
        pytest.skip("a 1e-3 perturbation is below the bf16 tolerance (2e-2) by design")
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    fault(0)
    compare(case, run_gpu(case, x, dz, p), ref, p)  # clean: passes
    fault(FAULTS[what])
    got = run_gpu(case, x, dz, p)
    fault(0)
    with pytest.raises(AssertionError):
        compare(case, got, ref, p)


def test_harness_catches_fault_in_sync_emulated(fault):
    import torch

    import paper_1712_02616_b200 as P
    case = Case(8, 24, 196, dtype="f32", seed=83)
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)

    def run():
        g, b = p.gamma.cuda(), p.beta.cuda()
        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
        z, sm, sv = P.forward_sync_emulated(x.cuda(), 2, g, b, rm, rv)
        dx, dg, db = P.backward_sync_emulated(z, dz.cuda(), 2, g, b, sv)
        torch.cuda.synchronize()
        return dict(z=z.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(),
                    dx=dx.cpu(), dgamma=dg.sum(0).cpu(), dbeta=db.sum(0).cpu())

    fault(0)
    compare(case, run(), ref, p)
    fault(FAULTS["dgamma"])
    got = run()
    fault(0)
    with pytest.raises(AssertionError):
        compare(case, got, ref, p)
