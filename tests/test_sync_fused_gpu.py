"""GPU parity of the fused-collective synchronized variant (InPlace-ABN^sync,
PAPER.md:315, :356) in its one-GPU emulation: the G ranks' shards of one tensor in
one cooperative launch of the channel-resident kernels, the ranks' per-channel
records exchanged through the same peer-record protocol the multi-GPU path uses
(include/iabn.h, "fused-collective sync").  Expected values: the oracle on the
concatenated batch (R7), including each shard's own dgamma/dbeta
contribution (oracle.param_grads_sharded)."""
import pytest
import torch

from tests.harness import Case, compare, inputs, run_oracle, to64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_02616_b200  # noqa: F401  (fails loudly if libiabn.so is missing)


def _run(case, G, x, dz, p, *, global_param_grads=False, stream=None):
    import paper_1712_02616_b200 as P
    xd, dzd = x.cuda(), dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    kw = dict(eps=case.eps, slope=case.slope, gamma_mode=case.gamma_mode)
    z, sm, sv = P.forward_sync_emulated(xd, G, g, b, rm, rv, momentum=case.momentum, **kw)
    dx, dg, db = P.backward_sync_emulated(z, dzd, G, g, b, sv, dx=torch.empty_like(dzd),
                                          global_param_grads=global_param_grads, **kw)
    torch.cuda.synchronize()
    return dict(z=z, dzd=dzd, mean=sm, var=sv, rm=rm, rv=rv, dx=dx, dg=dg, db=db, g=g, b=b)


CASES = [
    Case(8, 24, 100, dtype="f32", seed=21),     # planes 400 B
    Case(8, 40, 196, dtype="bf16", seed=22),    # planes 392 B: covering-range kernels
    Case(16, 64, 784, dtype="bf16", seed=23),   # several channels per cluster
    Case(8, 300, 49, dtype="f32", seed=24),     # 7x7 fp32, more channels than clusters
]


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c.N}x{c.C}x{c.HW}-{c.dtype}")
def test_sync_fused_equals_concatenated_batch(case, G):
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    out = _run(case, G, x, dz, p)
    got = dict(z=out["z"].cpu(), dx=out["dx"].cpu(), mean=out["mean"].cpu(),
               var=out["var"].cpu(), rm=out["rm"].cpu(), rv=out["rv"].cpu(),
               dgamma=out["dg"].sum(0).cpu(), dbeta=out["db"].sum(0).cpu())
    compare(case, got, ref, p)
    assert out["dg"].shape == (G, case.C)


@pytest.mark.parametrize("G", [2, 4])
@pytest.mark.parametrize("case", CASES[:2], ids=lambda c: f"{c.N}x{c.C}x{c.HW}-{c.dtype}")
def test_sync_fused_local_param_grads(case, G):
    """Row r of dgamma/dbeta is shard r's own contribution (R7), against the oracle's
    per-shard gradients on the concatenated batch (oracle.param_grads_sharded); with
    global_param_grads every row holds the all-shard sums."""
    import oracle
    from tests.harness import ambiguous, shard_param_errs, TOL
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    amb = ambiguous(case, ref, p)
    out = _run(case, G, x, dz, p)
    n = case.N // G
    dgl, dbl = oracle.load().param_grads_sharded(to64(x), to64(dz), to64(p.gamma), to64(p.beta),
                                                 [n] * G, eps=case.eps, slope=case.slope,
                                                 gamma_mode=case.gamma_mode)
    for r in range(G):
        e = shard_param_errs(case, ref, amb, slice(r * n, (r + 1) * n), out["dg"][r].cpu(),
                             out["db"][r].cpu(), dgl[r], dbl[r])
        assert max(e.values()) <= TOL[case.dtype], (r, e)
    glob = _run(case, G, x, dz, p, global_param_grads=True)
    for r in range(G):
        assert torch.equal(glob["dg"][r], glob["dg"][0])
        assert torch.equal(glob["db"][r], glob["db"][0])
    e = shard_param_errs(case, ref, amb, slice(0, case.N), glob["dg"][0].cpu(),
                         glob["db"][0].cpu(), dgl.sum(0), dbl.sum(0))
    assert max(e.values()) <= TOL[case.dtype], e


def test_sync_fused_repeated_calls_and_graph_replay():
    """The record buffers are reused call after call (two parity halves, a device-side
    call counter): consecutive calls and CUDA-graph replays see only their own records."""
    import paper_1712_02616_b200 as P
    case = Case(8, 64, 256, dtype="bf16", seed=31)
    G = 4
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    kw = dict(eps=case.eps, slope=case.slope)
    results = []
    with torch.cuda.stream(side):
        for seed in (31, 32, 33):
            c = Case(case.N, case.C, case.HW, dtype=case.dtype, seed=seed)
            x, dz, p = inputs(c)
            out = _run(c, G, x, dz, p)
            ref = run_oracle(c, x, dz, p)
            compare(c, dict(z=out["z"].cpu(), dx=out["dx"].cpu(), mean=out["mean"].cpu(),
                            var=out["var"].cpu(), rm=out["rm"].cpu(), rv=out["rv"].cpu(),
                            dgamma=out["dg"].sum(0).cpu(), dbeta=out["db"].sum(0).cpu()), ref, p)
            results.append((c, x, dz, p))
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    # capture one forward + backward on the warmed-up stream, replay with new inputs
    c, x, dz, p = results[0]
    xs, dzs = x.cuda(), dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    dxs = torch.empty_like(dzs)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        z, sm, sv = P.forward_sync_emulated(xs, G, g, b, rm, rv, **kw)
        dx, dg, db = P.backward_sync_emulated(z, dzs, G, g, b, sv, dx=dxs, **kw)
    for c, x, dz, p in results[1:] + results[:1]:
        xs.copy_(x.cuda())
        dzs.copy_(dz.cuda())
        g.copy_(p.gamma.cuda())
        b.copy_(p.beta.cuda())
        rm.copy_(p.running_mean.cuda())
        rv.copy_(p.running_var.cuda())
        graph.replay()
        torch.cuda.synchronize()
        ref = run_oracle(c, x, dz, p)
        compare(c, dict(z=z.cpu(), dx=dx.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(),
                        rv=rv.cpu(), dgamma=dg.sum(0).cpu(), dbeta=db.sum(0).cpu()), ref, p)


def test_sync_fused_matches_single_rank_fused():
    """G = 1 is the plain channel-resident kernel: bitwise equal to iabn_forward /
    iabn_backward on the same tensor."""
    import paper_1712_02616_b200 as P
    from tests.harness import run_gpu
    case = Case(8, 48, 196, dtype="f32", seed=35)
    x, dz, p = inputs(case)
    eager = run_gpu(case, x, dz, p, dx_inplace=False, flags=1 << 9)  # channel-resident
    out = _run(case, 1, x, dz, p)
    assert torch.equal(out["z"].cpu(), eager["z"])
    assert torch.equal(out["dx"].cpu(), eager["dx"])
    assert torch.equal(out["dg"][0].cpu(), eager["dgamma"])
    assert torch.equal(out["db"][0].cpu(), eager["dbeta"])


def test_sync_fused_rejects_bad_arguments():
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200._lib import IabnError
    x = torch.randn(6, 8, 16, device="cuda")
    g, b = torch.ones(8, device="cuda"), torch.zeros(8, device="cuda")
    with pytest.raises(ValueError):
        P.forward_sync_emulated(x, 4, g, b)  # 6 samples do not split into 4 shards
    with pytest.raises(IabnError):
        P.forward_sync_emulated(x.repeat(2, 1, 1)[:9 * 1], 9, g, b)  # more than 8 ranks


@pytest.mark.slow
def test_sync_fused_full_size_sampled_channels():
    """bench.py's workload (WideResNet-38 16x4096x112x112 bf16) as 8 virtual ranks of 2
    crops (the launch configuration of its `sync_emulated` figure): sampled whole channels
    against the oracle on the full batch, every channel's dbeta against sum(dy) from z."""
    import numpy as np
    import paper_1712_02616_b200 as P
    import synth_inputs as S
    cfg = S.CONFIGS["wrn38"]
    N, C, HW, G = cfg["N"], cfg["C"], cfg["HW"], 8
    x = S.make_x(N, C, HW, 0, dtype="bf16")
    dz = S.make_dz(N, C, HW, 0, dtype="bf16")
    p = S.make_params(C, 0)
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    z, sm, sv = P.forward_sync_emulated(x.cuda(), G, g, b, rm, rv)
    dzd = dz.cuda()
    dx, dg, db = P.backward_sync_emulated(z, dzd, G, g, b, sv, dx=torch.empty_like(dzd))
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    ch = torch.tensor(sorted({0, C - 1, *rng.choice(C, 10, replace=False).tolist()}))
    sub = Case(N, len(ch), HW, dtype="bf16")
    ps = S.Params(p.gamma[ch], p.beta[ch], p.running_mean[ch], p.running_var[ch])
    chd = ch.cuda()
    got = dict(z=z[:, chd, :].cpu(), dx=dx[:, chd, :].cpu(), mean=sm[chd].cpu(),
               var=sv[chd].cpu(), rm=rm[chd].cpu(), rv=rv[chd].cpu(),
               dgamma=dg[:, chd].sum(0).cpu(), dbeta=db[:, chd].sum(0).cpu())
    compare(sub, got, run_oracle(sub, x[:, ch, :].contiguous(), dz[:, ch, :].contiguous(), ps), ps)
    zf = z.double()
    dy = torch.where(zf >= 0, dzd.double(), dzd.double() * 0.01)
    ref = dy.sum(dim=(0, 2))
    assert ((db.double().sum(0) - ref).abs().max() / ref.abs().max()).item() < 1e-3
    # each virtual rank's row is its own shard's sum
    n = N // G
    for r in (0, G - 1):
        refr = dy[r * n:(r + 1) * n].sum(dim=(0, 2))
        assert ((db[r].double() - refr).abs().max() / refr.abs().max()).item() < 1e-3


@pytest.mark.parametrize("gamma_mode,flags", [("plain", 0), ("fixed_one", 0), ("abs_eps", 1 << 5),
                                              ("abs_eps", 1 << 2)],
                         ids=["gamma_plain", "gamma_fixed_one", "variant_I", "running_var_biased"])
def test_sync_fused_modes(gamma_mode, flags):
    """The record exchange under every reparametrisation / variant / running-stat flag."""
    import paper_1712_02616_b200 as P
    case = Case(8, 40, 196, dtype="bf16", seed=41, gamma_mode=gamma_mode)
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    G = 4
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    kw = dict(eps=case.eps, slope=case.slope, gamma_mode=gamma_mode)
    z, sm, sv = P.forward_sync_emulated(x.cuda(), G, g, b, rm, rv, momentum=case.momentum,
                                        running_var_biased=bool(flags & (1 << 2)), **kw)
    dzd = dz.cuda()
    dx, dg, db = P.backward_sync_emulated(z, dzd, G, g, b, sv, dx=torch.empty_like(dzd),
                                          flags=flags & (1 << 5), **kw)
    torch.cuda.synchronize()
    got = dict(z=z.cpu(), dx=dx.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(),
               dgamma=dg.sum(0).cpu(), dbeta=db.sum(0).cpu())
    if flags & (1 << 2):  # biased running variance (SPEC.md:272 reading; oracle pinned to it)
        import oracle
        ref["rv"] = oracle.load().forward(
            to64(x), to64(p.gamma), to64(p.beta), eps=case.eps, slope=case.slope,
            momentum=case.momentum, running_mean=to64(p.running_mean),
            running_var=to64(p.running_var), gamma_mode=gamma_mode,
            running_var_biased=True).running_var
    compare(case, got, ref, p)
    # each virtual rank's dgamma / dbeta row: its own shard's contribution (R7), from the
    # oracle's per-shard gradients on the concatenated batch
    import oracle
    from tests.harness import ambiguous, shard_param_errs
    dgl, dbl = oracle.load().param_grads_sharded(to64(x), to64(dz), to64(p.gamma), to64(p.beta),
                                                 [case.N // G] * G, eps=case.eps,
                                                 slope=case.slope, gamma_mode=gamma_mode)
    amb = ambiguous(case, ref, p)
    n = case.N // G
    for r in range(G):
        e = shard_param_errs(case, ref, amb, slice(r * n, (r + 1) * n), dg[r].cpu(),
                             db[r].cpu(), dgl[r], dbl[r])
        assert max(e.values()) <= 2e-2, (r, e)
