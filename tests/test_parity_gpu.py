"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs, element by element (tests/harness.py for the metric,
tolerances and the activation-branch reading R16)."""
import numpy as np
import pytest
import torch

import synth_inputs as S
from tests.harness import Case, compare, inputs, run_gpu, run_oracle, to64
from tests.util import chan_err, vec_err

pytestmark = pytest.mark.gpu

FUSED, STREAM = 1 << 9, 1 << 8


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_02616_b200  # noqa: F401  (fails loudly if libiabn.so is missing)


def _check(case, flags=0, **kw):
    x, dz, p = inputs(case)
    got = run_gpu(case, x, dz, p, flags=flags, **kw)
    ref = run_oracle(case, x, dz, p)
    return compare(case, got, ref, p)


# ------------------------------------------------------------------ cfg1 (BASELINE.json configs[0])
@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("flags", [0, STREAM], ids=["auto", "streaming"])
def test_cfg1_tiny(seed, flags):
    _check(Case(2, 8, 16, seed=seed), flags)


def test_cfg1_tiny_is_on_chip_by_default():
    """cfg1 takes a one-launch on-chip schedule (register-resident small layers, or the
    channel-resident kernels)."""
    from paper_1712_02616_b200 import _lib as L
    d = L.desc(2, 8, 16, L.F32, L.NCHW)
    assert L.query_schedule(d, 0)[0] in (1, 5)
    assert L.query_schedule(d, 1)[0] in (1, 5)


# ------------------------------------------------------------------ ragged / edge shapes
EDGE = [
    Case(3, 5, 7),                              # HW*4 not 16-aligned -> scalar streaming
    Case(5, 37, 49, dtype="bf16"),              # 7x7 bf16
    Case(4, 20, 196, dtype="bf16"),             # 14x14 bf16 (392 B planes, 8-aligned)
    Case(4, 20, 196),                           # 14x14 fp32 (fused)
    # m = 2, the minimum for training.  dx = g rstd (dy1-dy2) eps/(2(var+eps)): with
    # eps << var it is a cancellation fp32 cannot resolve, so eps is taken large here.
    Case(1, 3, 2, eps=0.5),
    Case(2, 1, 4096),                           # one channel
    Case(7, 64, 12, layout="NHWC"),             # NHWC, aligned channels
    Case(3, 37, 10, layout="NHWC"),             # NHWC, C*4 not 16-aligned
    Case(2, 136, 9, dtype="bf16", layout="NHWC"),
    Case(9, 300, 64, dtype="bf16"),             # several CTAs per channel, ragged split
    Case(33, 3, 1000),                          # many planes, few channels
]


@pytest.mark.parametrize("case", EDGE, ids=lambda c: f"{c.N}x{c.C}x{c.HW}-{c.dtype}-{c.layout}")
@pytest.mark.parametrize("flags", [0, STREAM], ids=["auto", "streaming"])
def test_edge_shapes(case, flags):
    _check(case, flags)


@pytest.mark.parametrize("gamma_mode", ["plain", "fixed_one"])
def test_gamma_modes(gamma_mode):
    _check(Case(4, 24, 64, gamma_mode=gamma_mode, seed=3))
    _check(Case(4, 24, 64, gamma_mode=gamma_mode, seed=3), STREAM)


@pytest.mark.parametrize("slope", [0.01, 0.1, 1.0])
def test_slopes(slope):
    _check(Case(4, 16, 100, slope=slope, seed=4))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_stress_offset(dtype):
    """|mean|/std = 1e3: cancellation in the variance (R8)."""
    _check(Case(8, 16, 256, dtype=dtype, stress="offset", seed=5))
    _check(Case(8, 16, 256, dtype=dtype, stress="offset", seed=5), STREAM)


def test_stress_constant_channel():
    _check(Case(8, 16, 256, stress="constant", seed=6))
    _check(Case(8, 16, 256, stress="constant", seed=6), STREAM)


def test_momentum_extremes():
    _check(Case(4, 8, 32, momentum=0.0))
    _check(Case(4, 8, 32, momentum=1.0))


def test_out_of_place_bitwise_equal_to_in_place():
    case = Case(6, 40, 196, seed=7)
    x, dz, p = inputs(case)
    for flags in (0, STREAM):
        a = run_gpu(case, x, dz, p, flags=flags)
        b = run_gpu(case, x, dz, p, flags=flags, inplace=False, dx_inplace=False)
        for k in a:
            assert torch.equal(a[k], b[k]), (flags, k)


def test_deterministic():
    case = Case(16, 64, 784, dtype="bf16", seed=8)
    x, dz, p = inputs(case)
    for flags in (0, STREAM):
        a = run_gpu(case, x, dz, p, flags=flags)
        b = run_gpu(case, x, dz, p, flags=flags)
        for k in a:
            assert torch.equal(a[k], b[k]), (flags, k)


def test_fused_and_streaming_agree():
    case = Case(8, 32, 784, seed=9)
    x, dz, p = inputs(case)
    a = run_gpu(case, x, dz, p, flags=FUSED)
    b = run_gpu(case, x, dz, p, flags=STREAM)
    for k in ("z", "dx"):
        assert chan_err(to64(a[k]), to64(b[k]), 1) < 1e-5
    for k in ("mean", "var", "dgamma", "dbeta"):
        assert vec_err(to64(a[k]), to64(b[k])) < 1e-5


@pytest.mark.parametrize("case", [
    Case(4, 12, 50, seed=10),                              # NCHW rows apply, ragged planes
    Case(3, 20, 3, seed=11),                               # NCHW HW < V: per-element channel
    Case(2, 32, 4, seed=12),                               # NCHW aligned small planes
    Case(4, 64, 49, dtype="bf16", seed=13),                # bf16 straddling vectors
    Case(4, 64, 50, layout="NHWC", seed=14),               # NHWC fixed channel groups
    Case(3, 7, 11, layout="NHWC", seed=15),                # NHWC unaligned rows
    Case(4, 16, 64, gamma_mode="plain", seed=16),          # gamma used as given
    Case(4, 16, 64, gamma_mode="fixed_one", layout="NHWC", seed=17)],
    ids=["rows", "hw3", "hw4", "bf16", "nhwc", "nhwc_odd", "plain", "fixed_one"])
def test_eval_mode(case):
    """Eval forward in one launch (the apply derives the coefficients from
    the running statistics, every apply variant) against the oracle's eval forward."""
    import oracle
    import paper_1712_02616_b200 as P
    x, _, p = inputs(case)
    rm = torch.randn(case.C) * 0.1
    rv = torch.rand(case.C) + 0.5
    z, sm, sv = P.forward(x.cuda(), p.gamma.cuda(), p.beta.cuda(), rm.cuda(), rv.cuda(),
                          training=False, layout=case.layout, gamma_mode=case.gamma_mode)
    assert sm is None and sv is None
    ref = oracle.load().forward_eval(to64(x), to64(p.gamma), to64(p.beta), to64(rm), to64(rv),
                                     layout=case.layout, gamma_mode=case.gamma_mode)
    assert chan_err(to64(z), ref, case.ax) < (1e-5 if case.dtype == "f32" else 1e-2)


# ------------------------------------------------------------------ cfg2 (BASELINE.json configs[1]) full size
@pytest.mark.parametrize("flags", [0, STREAM], ids=["fused", "streaming"])
def test_cfg2_r50_stage3_full(flags):
    errs = _check(Case(64, 1024, 196, seed=0), flags)
    assert errs["z"] < 1e-5


def test_cfg2_nhwc_full():
    _check(Case(64, 1024, 196, layout="NHWC", seed=1))


# ------------------------------------------------------------------ sync variant on one GPU (split phase)
@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_sync_split_phase_equals_concatenated_batch(G, dtype):
    """InPlace-ABN^sync: shards' statistics and gradient sums are
    summed (torch.add here standing in for the NCCL all-reduce), and the result
    must equal the oracle on the concatenated batch.  Shards have unequal N."""
    import paper_1712_02616_b200 as P
    case = Case(11, 24, 100, dtype=dtype, seed=11)
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    bounds = np.linspace(0, case.N, G + 1).astype(int)
    bounds[1] = max(bounds[1] - 1, 1)  # unequal shards
    xs = [x[bounds[i]:bounds[i + 1]].cuda().contiguous() for i in range(G)]
    dzs = [dz[bounds[i]:bounds[i + 1]].cuda().contiguous() for i in range(G)]
    g, b = p.gamma.cuda(), p.beta.cuda()
    stats = [P.forward_reduce(xi) for xi in xs]
    tot = torch.stack(stats).sum(0)
    zs, svs = [], []
    for xi in xs:
        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
        zi, smi, svi = P.forward_apply(xi, tot, g, b, rm, rv)
        zs.append(zi)
        svs.append(svi)
    sums = [P.backward_reduce(zi, dzi, g, b) for zi, dzi in zip(zs, dzs)]
    gsum = torch.stack(sums).sum(0)
    dxs, dgs, dbs = [], [], []
    for zi, dzi, si in zip(zs, dzs, sums):
        dxi, dgi, dbi = P.backward_apply(zi, dzi, gsum, si, g, b, svs[0])
        dxs.append(dxi)
        dgs.append(dgi)
        dbs.append(dbi)
    torch.cuda.synchronize()
    got = dict(z=torch.cat([t.cpu() for t in zs]), dx=torch.cat([t.cpu() for t in dxs]),
               mean=smi.cpu(), var=svs[0].cpu(), rm=rm.cpu(), rv=rv.cpu(),
               dgamma=sum(t.cpu() for t in dgs), dbeta=sum(t.cpu() for t in dbs))
    compare(case, got, ref, p)
    # every shard saw the same (global) statistics
    for svi in svs[1:]:
        assert torch.equal(svi, svs[0])
    # global-param-grads flag returns the all-shard sums directly
    _, dgg, dbg = P.backward_apply(zs[0], dzs[0].clone(), gsum, sums[0], g, b, svs[0],
                                   dx=torch.empty_like(zs[0]), global_param_grads=True)
    assert vec_err(to64(dgg), ref["dgamma"]) < 1e-4 * (50 if dtype == "bf16" else 1)
    assert vec_err(to64(dbg), ref["dbeta"]) < 1e-4 * (50 if dtype == "bf16" else 1)


# ------------------------------------------------------------------ autograd wrapper
def test_autograd_module_matches_oracle():
    import paper_1712_02616_b200 as P
    import oracle
    case = Case(4, 16, 64, seed=12)
    x, dz, p = inputs(case)
    m = P.InPlaceABN(16, device="cuda")
    with torch.no_grad():
        m.weight.copy_(p.gamma)
        m.bias.copy_(p.beta)
    xin = x.view(4, 16, 8, 8).cuda().requires_grad_(True)
    h = xin * 1.0  # leaf can't be modified in place
    z = m(h)
    z.backward(dz.view(4, 16, 8, 8).cuda())
    o = oracle.load()
    f = o.forward(to64(x), to64(p.gamma), to64(p.beta))
    dx, dg, db = o.backward_standard(to64(x), to64(dz), to64(p.gamma), to64(p.beta))
    assert chan_err(to64(z.detach().view(4, 16, 64)), f.z, 1) < 1e-4
    assert chan_err(to64(xin.grad.view(4, 16, 64)), dx, 1) < 1e-4
    assert vec_err(to64(m.weight.grad), dg) < 1e-4 and vec_err(to64(m.bias.grad), db) < 1e-4


@pytest.mark.parametrize("share", [True, False], ids=["grad_inplace", "fresh_dx"])
def test_autograd_gradient_sharing(share):
    """dL/dx may overwrite dL/dz -- with grad_inplace the gradient reaching
    the layer's input is the very buffer the layer received; the values match either way."""
    import paper_1712_02616_b200 as P
    case = Case(4, 16, 64, seed=14)
    x, dz, p = inputs(case)
    seen = {}
    outs = []
    for _ in range(2):
        m = P.InPlaceABN(16, device="cuda", grad_inplace=share)
        with torch.no_grad():
            m.weight.copy_(p.gamma)
            m.bias.copy_(p.beta)
        xin = x.view(4, 16, 8, 8).cuda().requires_grad_(True)
        h = xin * 1.0
        h.register_hook(lambda g: seen.__setitem__("dx", g.data_ptr()))
        z = m(h)
        z.register_hook(lambda g: seen.__setitem__("dz", g.data_ptr()))
        (z * dz.view(4, 16, 8, 8).cuda()).sum().backward()
        outs.append(xin.grad.clone())
    assert (seen["dx"] == seen["dz"]) == share
    assert torch.equal(outs[0], outs[1])


def test_channels_last_module():
    import paper_1712_02616_b200 as P
    import oracle
    case = Case(2, 32, 36, seed=13)
    x, dz, p = inputs(case)
    m = P.InPlaceABN(32, device="cuda")
    with torch.no_grad():
        m.weight.copy_(p.gamma)
        m.bias.copy_(p.beta)
    xin = x.view(2, 32, 6, 6).cuda().to(memory_format=torch.channels_last)
    z = m(xin.clone())
    ref = oracle.load().forward(to64(x), to64(p.gamma), to64(p.beta))
    assert chan_err(to64(z.contiguous().view(2, 32, 36)), ref.z, 1) < 1e-4


# ------------------------------------------------------------------ native code is what runs
def test_kernels_launch_through_the_library():
    from paper_1712_02616_b200 import _lib as L
    before = L.launch_count()
    _check(Case(2, 8, 16))
    assert L.launch_count() - before >= 2
    import os
    maps = open(f"/proc/{os.getpid()}/maps").read()
    assert "libiabn.so" in maps


# ------------------------------------------------------------------ backward variants (Alg. 2 I / II)
VARIANT_I = 1 << 5


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("flags", [0, VARIANT_I], ids=["II", "I"])
def test_backward_variants(dtype, flags):
    _check(Case(8, 32, 784, dtype=dtype, seed=14), flags)


@pytest.mark.parametrize("flags", [0, VARIANT_I, STREAM], ids=["II", "I", "streaming"])
def test_large_beta_over_gamma(flags):
    """|beta / gamma| = 20: the cancellation of the BN-dagger sum (Q - beta S1)/g
     stays within the fp32 tolerance."""
    case = Case(8, 16, 784, seed=15)
    x, dz, p = inputs(case)
    p.beta = (20.0 * p.gamma.abs()).contiguous()
    got = run_gpu(case, x, dz, p, flags=flags)
    ref = run_oracle(case, x, dz, p)
    compare(case, got, ref, p)


@pytest.mark.parametrize("flags", [0, VARIANT_I, STREAM], ids=["II", "I", "streaming"])
def test_large_beta_over_gamma_bf16(flags):
    """|beta / gamma| = 20 with bf16 storage.  The stored z is rounded to bf16, so x^
    recovered from it carries 2^-9 |y| / gamma~ ~ 4 % of error here (reading R9) whatever
    the reduction; to isolate the BN-dagger cancellation (Q - beta S1)/gamma~ of the
    default kernels, the expected gradients are the oracle's Alg. 2 from the GPU's own
    rounded z (in double).  dgamma/dbeta are fp32 outputs: 1e-4."""
    import oracle
    from tests.util import vec_err
    case = Case(8, 16, 784, dtype="bf16", seed=16)
    x, dz, p = inputs(case)
    p.beta = (20.0 * p.gamma.abs()).contiguous()
    got = run_gpu(case, x, dz, p, flags=flags)
    o = oracle.load()
    dx, dg, db = o.backward_inplace_I(to64(got["z"]), to64(dz), to64(got["var"]), to64(p.gamma),
                                      to64(p.beta), eps=case.eps, slope=case.slope)
    assert chan_err(to64(got["dx"]), dx, 1) < 2e-2
    assert vec_err(to64(got["dgamma"]), dg) < 1e-4 and vec_err(to64(got["dbeta"]), db) < 1e-4


# ------------------------------------------------------------------ streaming kernels at large planes
@pytest.mark.parametrize("case", [
    Case(3, 5, 64 * 64, dtype="bf16", seed=16),  # bf16, HW >= kThreads * 8: row-cursor apply
    Case(2, 7, 1100, dtype="f32", seed=17),      # f32, HW >= kThreads * 4, ragged plane / thread
    Case(5, 3, 2056, dtype="bf16", seed=18),     # plane not a multiple of the thread step
], ids=["bf16_4096", "f32_1100", "bf16_2056"])
@pytest.mark.parametrize("flags", [0, STREAM], ids=["auto", "streaming"])
def test_large_planes(case, flags):
    _check(case, flags)


# ------------------------------------------------------------------ test-time folding
@pytest.mark.parametrize("gamma_mode", ["abs_eps", "plain", "fixed_one"])
@pytest.mark.parametrize("with_bias", [True, False], ids=["bias", "nobias"])
def test_fold_conv(gamma_mode, with_bias, orc):
    import numpy as np
    import paper_1712_02616_b200 as P
    g = torch.Generator().manual_seed(19)
    cout, shape = 37, (37, 19, 3, 3)
    w = torch.randn(shape, generator=g)
    b = torch.randn(cout, generator=g) if with_bias else None
    gamma = torch.rand(cout, generator=g) + 0.5
    gamma[::3] *= -1
    beta, rm = torch.randn(cout, generator=g), torch.randn(cout, generator=g)
    rv = torch.rand(cout, generator=g) * 3 + 0.1
    dev = torch.device("cuda", 0)
    cu = lambda t: None if t is None else t.to(dev)
    w2, b2 = P.fold_conv(cu(w), cu(b), cu(rm), cu(rv), cu(gamma), cu(beta), gamma_mode=gamma_mode)
    rw, rb = orc.fold_conv(w.numpy(), None if b is None else b.numpy(), rm.numpy(), rv.numpy(),
                           gamma.numpy(), beta.numpy(), eps=1e-5, gamma_mode=gamma_mode)
    w2, b2 = w2.cpu().double().numpy(), b2.cpu().double().numpy()
    assert np.abs(w2 - rw).max() / np.abs(rw).max() < 1e-6
    assert np.abs(b2 - rb).max() / np.abs(rb).max() < 1e-6
    # in place gives the same bits
    wi, bi = cu(w.clone()), cu(b.clone()) if b is not None else None
    wo, bo = P.fold_conv(wi, bi, cu(rm), cu(rv), cu(gamma), cu(beta), gamma_mode=gamma_mode,
                         inplace=True)
    assert wo.data_ptr() == wi.data_ptr()
    assert torch.equal(wo.cpu(), torch.from_numpy(w2).float())
    assert torch.equal(bo.cpu(), torch.from_numpy(b2).float())


# ------------------------------------------------------------------ streaming at any plane alignment
MISALIGNED = [
    Case(8, 40, 196, dtype="bf16", seed=26),   # 392-byte planes: covering vectors, straddles
    Case(4, 24, 49, dtype="bf16", seed=27),    # 98-byte planes
    Case(3, 5, 7, dtype="bf16", seed=28),      # plane shorter than a vector: generic apply
    Case(5, 6, 9, dtype="f32", seed=29),       # 36-byte planes
    Case(2, 33, 1001, dtype="bf16", seed=30),  # long odd planes
    Case(4, 37, 30, dtype="bf16", layout="NHWC", seed=31),  # NHWC, rows not 16-byte multiples
    Case(4, 40, 30, dtype="bf16", layout="NHWC", seed=32),  # NHWC aligned, C/V = 5 vectors
]


@pytest.mark.parametrize("case", MISALIGNED, ids=lambda c: f"{c.layout}_{c.dtype}_{c.N}x{c.C}x{c.HW}")
def test_streaming_any_alignment(case):
    _check(case, STREAM)


# ------------------------------------------------------------------ fused, planes not 16-byte aligned
MIS_CASES = [
    Case(8, 40, 196, dtype="bf16", seed=33),    # 392-byte planes (head 0 or 8 bytes)
    Case(6, 24, 49, dtype="bf16", seed=34),     # 98-byte planes (7 x 7)
    Case(4, 16, 9, dtype="f32", seed=35),       # 36-byte planes
    Case(16, 8, 1001, dtype="bf16", seed=36),   # long odd planes, K > 1 planes per CTA
    Case(32, 64, 49, dtype="f32", seed=37),     # 196-byte planes, many planes per slice
    Case(4, 1500, 49, dtype="bf16", seed=38),   # more channels than clusters: slots reused
]


@pytest.mark.parametrize("case", MIS_CASES, ids=lambda c: f"{c.dtype}_{c.N}x{c.C}x{c.HW}")
def test_fused_misaligned_planes(case):
    from paper_1712_02616_b200 import _lib as L
    d = L.desc(case.N, case.C, case.HW, L.BF16 if case.dtype == "bf16" else L.F32, L.NCHW)
    assert L.query_schedule(d, 0, FUSED)[0] == 1 and L.query_schedule(d, 1, FUSED)[0] == 1
    _check(case, FUSED)


# ------------------------------------------------------------------ CUDA graphs
@pytest.mark.parametrize("case", [Case(8, 32, 784, dtype="bf16", seed=40),
                                  Case(4, 40, 196, dtype="bf16", seed=41),
                                  Case(3, 24, 49, dtype="f32", layout="NHWC", seed=42)],
                         ids=["fused", "streaming_misaligned", "nhwc"])
def test_cuda_graph_capture(case):
    """The calls only enqueue device work (no host synchronisation): a forward + backward
    captured in a CUDA graph and replayed gives the eager results bit for bit."""
    import paper_1712_02616_b200 as P
    x, dz, p = inputs(case)
    eager = run_gpu(case, x, dz, p)
    xs, dzs = x.cuda(), dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    kw = dict(eps=case.eps, slope=case.slope, gamma_mode=case.gamma_mode, layout=case.layout)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm-up: workspaces, kernel attributes, plans
        z, _, sv = P.forward(xs.clone(), g, b, rm.clone(), rv.clone(), momentum=case.momentum, **kw)
        P.backward(z, dzs.clone(), g, b, sv, **kw)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        z, sm, sv = P.forward(xs, g, b, rm, rv, momentum=case.momentum, **kw)
        dx, dg, db = P.backward(z, dzs, g, b, sv, save_mean=sm, **kw)
    xs.copy_(x.cuda())
    dzs.copy_(dz.cuda())
    rm.copy_(p.running_mean.cuda())
    rv.copy_(p.running_var.cuda())
    graph.replay()
    torch.cuda.synchronize()
    got = dict(z=z.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(), dx=dx.cpu(),
               dgamma=dg.cpu(), dbeta=db.cpu())
    for k in got:
        assert torch.equal(got[k], eager[k]), k


def test_two_streams_concurrently():
    """Calls on different streams use different workspaces: two layers run
    concurrently give the results each gives alone."""
    import paper_1712_02616_b200 as P
    cases = [Case(4, 24, 196, dtype="bf16", seed=43), Case(4, 24, 196, dtype="bf16", seed=44)]
    alone = [run_gpu(c, *inputs(c)) for c in cases]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    torch.cuda.synchronize()
    for c, s in zip(cases, streams):
        x, dz, p = inputs(c)
        with torch.cuda.stream(s):
            xd, dzd = x.cuda(), dz.cuda()
            g, b = p.gamma.cuda(), p.beta.cuda()
            rm, rv = p.running_mean.cuda(), p.running_var.cuda()
            z, sm, sv = P.forward(xd, g, b, rm, rv, momentum=c.momentum, eps=c.eps, slope=c.slope)
            dx, dg, db = P.backward(z, dzd, g, b, sv, eps=c.eps, slope=c.slope)
            outs.append(dict(z=z, dx=dx, dgamma=dg, dbeta=db, mean=sm, var=sv))
    torch.cuda.synchronize()
    for o, a in zip(outs, alone):
        for k in o:
            assert torch.equal(o[k].cpu(), a[k]), k


# ------------------------------------------------------------------ grid-resident NHWC schedule
GRES_CASES = [
    Case(8, 64, 49, dtype="bf16", layout="NHWC", seed=45),    # cv = 8
    Case(8, 96, 49, dtype="bf16", layout="NHWC", seed=46),    # cv = 12: 252 active threads
    Case(4, 40, 196, dtype="f32", layout="NHWC", seed=47),    # cv = 10
    Case(32, 128, 196, dtype="bf16", layout="NHWC", seed=48), # DenseNet bottleneck, 14 x 14
    Case(3, 1024, 5, dtype="f32", layout="NHWC", seed=49),    # few rows, wide rows (cv = 256)
    Case(5, 24, 7, dtype="f32", layout="NHWC", stress="offset", seed=50),  # |mean|/std = 1e3
]


RESIDENT = 1 << 11


@pytest.mark.parametrize("case", GRES_CASES, ids=lambda c: f"{c.dtype}_{c.N}x{c.C}x{c.HW}")
def test_grid_resident_nhwc(case):
    from paper_1712_02616_b200 import _lib as L
    d = L.desc(case.N, case.C, case.HW, L.BF16 if case.dtype == "bf16" else L.F32, L.NHWC)
    assert L.query_schedule(d, 0)[0] == 4  # default: channel groups; grid-resident is opt-in
    assert L.query_schedule(d, 0, RESIDENT)[0] == 3 and L.query_schedule(d, 1, RESIDENT)[0] == 3
    _check(case, RESIDENT)


def test_grid_resident_matches_streaming_bitwise_stats():
    """Same per-channel statistics up to the combine order; outputs agree to fp32 rounding."""
    case = Case(16, 64, 196, dtype="f32", layout="NHWC", seed=51)
    x, dz, p = inputs(case)
    a = run_gpu(case, x, dz, p, flags=RESIDENT)
    b = run_gpu(case, x, dz, p, flags=STREAM)
    for k in ("z", "dx"):
        assert (a[k] - b[k]).abs().max().item() <= 1e-5 * b[k].abs().max().item(), k


# ------------------------------------------------------------------ sync variant through NCCL
@pytest.mark.parametrize("case", [Case(4, 24, 196, dtype="f32", seed=52),
                                  Case(4, 40, 64, dtype="bf16", layout="NHWC", seed=53)],
                         ids=["nchw_f32", "nhwc_bf16"])
def test_sync_entry_points_single_rank(case):
    """iabn_forward_sync / iabn_backward_sync with a real NCCL communicator of ONE rank:
    communicator setup and teardown, and the one-rank shortcut (nranks == 1 takes the
    non-synchronized path, no all-reduce) match the oracle.  The all-reduce path itself
    (nranks >= 2) is tests/test_sync_shim_gpu.py (and tests/test_sync_multigpu.py on a
    multi-GPU box)."""
    import paper_1712_02616_b200 as P
    comm = P.Comm.create(1, 0, P.Comm.unique_id())
    try:
        x, dz, p = inputs(case)
        xd, dzd = x.cuda(), dz.cuda()
        g, b = p.gamma.cuda(), p.beta.cuda()
        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
        z, sm, sv = P.forward(xd, g, b, rm, rv, momentum=case.momentum, eps=case.eps,
                              slope=case.slope, layout=case.layout, comm=comm)
        dx, dg, db = P.backward(z, dzd, g, b, sv, eps=case.eps, slope=case.slope,
                                layout=case.layout, comm=comm)
        torch.cuda.synchronize()
        got = dict(z=z.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(),
                   dx=dx.cpu(), dgamma=dg.cpu(), dbeta=db.cpu())
        compare(case, got, run_oracle(case, x, dz, p), p)
    finally:
        comm.close()


def test_binding_desc_cache_keeps_validation():
    """The binding caches descriptors per (shape, dtype, layout): a cached shape must
    still reject a non-contiguous tensor, and two shapes must not share a descriptor."""
    import paper_1712_02616_b200 as P
    dev = torch.device("cuda", 0)
    C = 16
    g, b = torch.ones(C, device=dev), torch.zeros(C, device=dev)
    x = torch.randn(4, C, 8, 8, device=dev)
    z1, m1, v1 = P.forward(x.clone(), g, b)
    xt = torch.randn(4, 8, 8, C, device=dev).permute(0, 3, 1, 2)  # same shape, strided
    assert xt.shape == x.shape and not xt.is_contiguous()
    with pytest.raises(ValueError):
        P.forward(xt, g, b)
    y = torch.randn(2, C, 8, 8, device=dev)
    z2, m2, v2 = P.forward(y.clone(), g, b)
    torch.cuda.synchronize()
    ref = y.double().transpose(0, 1).reshape(C, -1)
    assert torch.allclose(m2.double().cpu(), ref.mean(1).cpu(), atol=1e-5)
    assert torch.allclose(m1.double().cpu(), x.double().transpose(0, 1).reshape(C, -1).mean(1).cpu(),
                          atol=1e-5)
