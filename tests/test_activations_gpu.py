"""BN followed by sigmoid / tanh ("Many activation functions are actually
invertible ... sigmoid, hyperbolic tangent, Leaky ReLU"): the CUDA path
(IABN_ACT_SIGMOID / IABN_ACT_TANH: the channel-resident kernels for NCHW, the streaming
kernels of kernels_act.cuh otherwise) against the oracle's
forward_act / backward_inplace_act / backward_standard_act (fp64), element by element,
through the C ABI.  The activations are smooth, so no branch allowance (R16) applies:
per-channel normwise error <= 1e-4 (fp32 storage, BASELINE.json north_star)."""
from __future__ import annotations

import pytest
import torch

from tests.harness import Case, inputs, to64
from tests.util import chan_err, vec_err

pytestmark = pytest.mark.gpu

TOL = 1e-4
ACTS = ("sigmoid", "tanh")
CASES = [Case(3, 37, 77, seed=90),                    # ragged planes, odd C
         Case(8, 64, 1024, seed=91),                  # several tiles per channel
         Case(2, 8, 16, seed=92),                     # tiny
         Case(16, 32, 49, seed=93, layout="NHWC"),    # 7x7 NHWC
         Case(4, 130, 196, seed=94, layout="NHWC"),   # C not a multiple of 32
         Case(5, 3, 7, seed=95, layout="NHWC"),       # E not a multiple of 4
         Case(8, 24, 196, seed=96, gamma_mode="plain"),
         Case(8, 24, 196, seed=97, gamma_mode="fixed_one", layout="NHWC")]
IDS = ["ragged", "tiles", "tiny", "nhwc7", "nhwc130", "nhwc_tail", "plain", "fixed_one"]


def _oracle():
    import oracle
    return oracle.load()


def _run_gpu(case, x, dz, p, act, *, flags=0, inplace=True):
    import paper_1712_02616_b200 as P
    xd, dzd = x.cuda(), dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    out = None if inplace else torch.empty_like(xd)
    z, sm, sv = P.forward(xd, g, b, rm, rv, momentum=case.momentum, eps=case.eps, out=out,
                          gamma_mode=case.gamma_mode, layout=case.layout, flags=flags,
                          activation=act)
    if inplace:
        assert z.data_ptr() == xd.data_ptr()
    zc = z.clone()
    dx, dg, db = P.backward(z, dzd, g, b, sv, eps=case.eps, gamma_mode=case.gamma_mode,
                            layout=case.layout, flags=flags, activation=act,
                            dx=None if inplace else torch.empty_like(dzd))
    if inplace:
        assert dx.data_ptr() == dzd.data_ptr()
    torch.cuda.synchronize()
    return dict(z=zc.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(),
                dx=dx.cpu(), dgamma=dg.cpu(), dbeta=db.cpu())


def _ref(case, x, dz, p, act):
    o = _oracle()
    x64, dz64, g, b = to64(x), to64(dz), to64(p.gamma), to64(p.beta)
    z, mean, var = o.forward_act(x64, g, b, act=act, eps=case.eps, gamma_mode=case.gamma_mode,
                                 layout=case.layout)
    run = o.forward(x64, g, b, eps=case.eps, momentum=case.momentum,
                    running_mean=to64(p.running_mean), running_var=to64(p.running_var),
                    gamma_mode=case.gamma_mode, layout=case.layout)
    dx, dg, db = o.backward_standard_act(x64, dz64, g, b, act=act, eps=case.eps,
                                         gamma_mode=case.gamma_mode, layout=case.layout)
    return dict(z=z, mean=mean, var=var, rm=run.running_mean, rv=run.running_var, dx=dx,
                dgamma=dg, dbeta=db)


def _errs(case, got, ref):
    e = {k: chan_err(to64(got[k]), ref[k], case.ax) for k in ("z", "dx")}
    e.update({k: vec_err(to64(got[k]), ref[k])
              for k in ("mean", "var", "rm", "rv", "dgamma", "dbeta")})
    return e


@pytest.mark.parametrize("case", CASES, ids=IDS)
@pytest.mark.parametrize("act", ACTS)
def test_act_parity(case, act):
    """z, batch / running statistics and the gradients from z alone (Alg. 2 inverting
    z through f^-1) equal the oracle's stored-x chain rule."""
    x, dz, p = inputs(case)
    errs = _errs(case, _run_gpu(case, x, dz, p, act), _ref(case, x, dz, p, act))
    assert all(v <= TOL for v in errs.values()), errs


@pytest.mark.parametrize("flags", [0, 1 << 8], ids=["auto", "streaming"])
@pytest.mark.parametrize("act", ACTS)
def test_act_out_of_place_and_variants(act, flags):
    """Out-of-place equals in-place bit for bit, on the channel-resident and the streaming
    schedule; IABN_VARIANT_I (per-element dy x^) and the default II (sum dy y, then
    (Q - beta S1)/g) agree with each other and with the oracle."""
    from paper_1712_02616_b200 import _lib as L
    case = Case(4, 20, 100, seed=98)
    x, dz, p = inputs(case)
    a = _run_gpu(case, x, dz, p, act, flags=flags)
    b = _run_gpu(case, x, dz, p, act, flags=flags, inplace=False)
    c = _run_gpu(case, x, dz, p, act, flags=flags | L.VARIANT_I)
    ref = _ref(case, x, dz, p, act)
    for k in a:
        assert torch.equal(a[k], b[k]), k
    for got in (a, c):
        errs = _errs(case, got, ref)
        assert all(v <= TOL for v in errs.values()), errs


@pytest.mark.parametrize("act", ACTS)
def test_act_schedules_agree(act):
    """Every NCHW schedule with the activation as a template parameter -- register-resident
    small layers (default here), channel-resident (IABN_FORCE_FUSED; covering-range variant
    for the misaligned fp32 plane of 7x11), streaming -- against the oracle, both
    variants."""
    from paper_1712_02616_b200 import _lib as L
    flag = L.ACT_SIGMOID if act == "sigmoid" else L.ACT_TANH
    for case in (Case(8, 48, 196, seed=101), Case(6, 24, 77, seed=102),
                 Case(32, 40, 49, seed=103)):
        d = L.desc(case.N, case.C, case.HW, L.F32, L.NCHW)
        for pass_ in (0, 1):
            assert L.query_schedule(d, pass_, flag)[0] == 5
            assert L.query_schedule(d, pass_, flag | L.FORCE_FUSED)[0] == 1
            assert L.query_schedule(d, pass_, flag | L.FORCE_STREAMING)[0] == 0
        x, dz, p = inputs(case)
        ref = _ref(case, x, dz, p, act)
        for fl in (0, L.FORCE_FUSED, L.FORCE_STREAMING, L.VARIANT_I, L.FORCE_FUSED | L.VARIANT_I):
            errs = _errs(case, _run_gpu(case, x, dz, p, act, flags=fl), ref)
            assert all(v <= TOL for v in errs.values()), (fl, errs)


@pytest.mark.parametrize("layout", ["NCHW", "NHWC"])
@pytest.mark.parametrize("act", ACTS)
def test_act_eval(act, layout):
    """Eval mode: z = f(g (x - running_mean)/sqrt(running_var + eps) + beta)
    with the running statistics read-only; reference: the same formula in fp64 torch."""
    import paper_1712_02616_b200 as P
    case = Case(4, 17, 33, seed=99, layout=layout)
    x, _, p = inputs(case)
    rm = torch.randn(case.C) * 0.5
    rv = torch.rand(case.C) + 0.5
    z, sm, sv = P.forward(x.cuda(), p.gamma.cuda(), p.beta.cuda(), rm.cuda(), rv.cuda(),
                          training=False, layout=layout, activation=act)
    assert sm is None and sv is None
    sh = [1, 1, 1]
    sh[case.ax] = case.C
    g64 = (p.gamma.double().abs() + case.eps).view(sh)
    y = (x.double() - rm.double().view(sh)) / torch.sqrt(rv.double().view(sh) + case.eps) * g64 \
        + p.beta.double().view(sh)
    ref = torch.sigmoid(y) if act == "sigmoid" else torch.tanh(y)
    assert chan_err(to64(z), ref.numpy(), case.ax) <= TOL


@pytest.mark.parametrize("act", ACTS)
def test_act_saturated_channel_stays_finite(act):
    """A channel driven far into saturation (y ~ +-40: z rounds to the asymptote in fp32)
    has no finite f^-1(z); the clamp (R17) keeps every output finite, and the
    unsaturated channels still match the oracle."""
    case = Case(4, 6, 64, seed=100)
    x, dz, p = inputs(case)
    p.gamma[2] = 40.0
    got = _run_gpu(case, x, dz, p, act)
    for k, v in got.items():
        assert torch.isfinite(v).all(), k
    ref = _ref(case, x, dz, p, act)
    keep = [c for c in range(case.C) if c != 2]
    for k in ("z", "dx"):
        assert chan_err(to64(got[k])[:, keep], ref[k][:, keep], 1) <= TOL, k
    assert vec_err(to64(got["dbeta"])[keep], ref["dbeta"][keep]) <= TOL


@pytest.mark.parametrize("act", ACTS)
def test_act_module_matches_torch_autograd(act):
    """InPlaceABN(activation=...) through autograd (z over x, dx over dz) against
    torch BatchNorm + sigmoid / tanh in fp64 on the CPU."""
    import paper_1712_02616_b200 as P
    torch.manual_seed(5)
    m = P.InPlaceABN(12, activation=act, device="cuda")
    with torch.no_grad():
        m.weight.copy_(torch.rand(12) + 0.5)
        m.bias.copy_(torch.randn(12) * 0.3)
    x = torch.randn(6, 12, 9, 9) * 2 + 1
    g = torch.randn_like(x)
    xd = x.cuda().requires_grad_(False)
    inp = xd.clone().requires_grad_(True)
    z = m(inp * 1.0)
    z.backward(g.cuda())
    xr = x.double().requires_grad_(True)
    w = m.weight.detach().cpu().double().requires_grad_(True)
    bb = m.bias.detach().cpu().double().requires_grad_(True)
    yr = torch.nn.functional.batch_norm(xr, None, None, w.abs() + 1e-5, bb, training=True)
    zr = torch.sigmoid(yr) if act == "sigmoid" else torch.tanh(yr)
    zr.backward(g.double())
    assert chan_err(to64(z), zr.detach().numpy(), 1) <= TOL
    assert chan_err(to64(inp.grad), xr.grad.numpy(), 1) <= TOL
    assert vec_err(to64(m.weight.grad), w.grad.numpy()) <= TOL
    assert vec_err(to64(m.bias.grad), bb.grad.numpy()) <= TOL


def test_act_rejections_and_schedule():
    """bf16 storage, both activation flags, and the split-phase / synchronized entries
    return errors; the schedule query reports streaming."""
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    x = torch.randn(2, 8, 16, device="cuda")
    g, b = torch.ones(8, device="cuda"), torch.zeros(8, device="cuda")
    with pytest.raises(L.IabnError):
        P.forward(x.bfloat16(), g, b, activation="sigmoid")
    with pytest.raises(L.IabnError):
        P.forward(x.clone(), g, b, flags=L.ACT_SIGMOID | L.ACT_TANH)
    with pytest.raises(L.IabnError):
        P.forward_sync_emulated(x.clone(), 2, g, b, flags=L.ACT_TANH)
    st = P.forward_reduce(x)
    with pytest.raises(L.IabnError):
        P.forward_apply(x.clone(), st, g, b, flags=L.ACT_SIGMOID)
    d = L.desc(32, 64, 3136, L.F32, L.NHWC)  # NHWC: streaming
    for pass_ in (0, 1):
        assert tuple(L.query_schedule(d, pass_, L.ACT_TANH)) == (0, 0)
        assert tuple(L.query_schedule(d, pass_, L.ACT_TANH | (1 << 8))) == (0, 0)


@pytest.mark.parametrize("act", ACTS)
def test_act_nhwc_channel_groups(act):
    """NHWC layers whose channel groups fit on chip take the channel-group kernels with the
    activation as a template parameter (schedule 4); against the oracle with both
    variants, and the streaming schedule (bulk-ring reduction with f: both variants)."""
    from paper_1712_02616_b200 import _lib as L
    flag = L.ACT_SIGMOID if act == "sigmoid" else L.ACT_TANH
    for case in (Case(16, 64, 196, seed=104, layout="NHWC"),
                 Case(8, 96, 784, seed=105, layout="NHWC")):
        d = L.desc(case.N, case.C, case.HW, L.F32, L.NHWC)
        assert L.query_schedule(d, 0, flag)[0] == 4 and L.query_schedule(d, 1, flag)[0] == 4
        x, dz, p = inputs(case)
        ref = _ref(case, x, dz, p, act)
        for fl in (0, L.VARIANT_I, L.FORCE_STREAMING, L.FORCE_STREAMING | L.VARIANT_I):
            errs = _errs(case, _run_gpu(case, x, dz, p, act, flags=fl), ref)
            assert all(v <= TOL for v in errs.values()), (fl, errs)
