"""Parity at BASELINE.json's full single-GPU size, in the launch configuration
bench.py times (default schedule): WideResNet-38 crops 16x4096x112x112 bf16
NCHW (configs[3] at G=1).  Channels are independent problems, so the oracle
checks a sample of whole channels (first, last and random ones) exactly, and
the remaining channels are checked through properties that hold at any size."""
import numpy as np
import pytest
import torch

import synth_inputs as S
from tests.harness import TOL, Case, compare, to64

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def full_run():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    cfg = S.CONFIGS["wrn38"]
    N, C, HW = cfg["N"], cfg["C"], cfg["HW"]
    case = Case(N, C, HW, dtype="bf16", seed=0)
    x = S.make_x(N, C, HW, 0, dtype="bf16")
    dz = S.make_dz(N, C, HW, 0, dtype="bf16")
    p = S.make_params(C, 0)
    d = L.desc(N, C, HW, L.BF16, L.NCHW)
    sched = (L.query_schedule(d, 0), L.query_schedule(d, 1))
    xd, dzd = x.cuda(), dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    z, sm, sv = P.forward(xd, g, b, rm, rv)
    dx, dg, db = P.backward(z, dzd, g, b, sv)
    torch.cuda.synchronize()
    rng = np.random.default_rng(123)
    chans = sorted({0, C - 1, *rng.choice(C, 14, replace=False).tolist()})
    return dict(case=case, x=x, dz=dz, p=p, z=z, dx=dx, sm=sm, sv=sv, rm=rm, rv=rv, dg=dg,
                db=db, chans=chans, sched=sched)


def test_schedule_is_channel_resident(full_run):
    (s0, k0), (s1, k1) = full_run["sched"]
    assert s0 == 1 and s1 == 1 and k0 >= 1 and k1 >= 1


def test_sampled_channels_match_oracle(full_run):
    r = full_run
    ch = torch.tensor(r["chans"])
    case = r["case"]
    sub = Case(case.N, len(ch), case.HW, dtype="bf16")
    ps = S.Params(r["p"].gamma[ch], r["p"].beta[ch], r["p"].running_mean[ch],
                  r["p"].running_var[ch])
    xs = r["x"][:, ch, :].contiguous()
    dzs = r["dz"][:, ch, :].contiguous()
    chd = ch.cuda()
    got = dict(z=r["z"][:, chd, :].cpu(), dx=r["dx"][:, chd, :].cpu(), mean=r["sm"][chd].cpu(),
               var=r["sv"][chd].cpu(), rm=r["rm"][chd].cpu(), rv=r["rv"][chd].cpu(),
               dgamma=r["dg"][chd].cpu(), dbeta=r["db"][chd].cpu())
    from tests.harness import run_oracle
    ref = run_oracle(sub, xs, dzs, ps)
    errs = compare(sub, got, ref, ps)
    print("full-size sampled parity:", errs)


def test_all_channels_properties(full_run):
    """For every channel: finite outputs; the batch variance saved equals the
    variance of x (torch fp64 reduction of the stored input); dbeta equals
    sum(dy) recomputed from z and dz with torch (sign of z gives f')."""
    r = full_run
    z, dx = r["z"], r["dx"]
    assert torch.isfinite(z.float()).all() and torch.isfinite(dx.float()).all()
    xd = r["x"].cuda().double()
    var = xd.var(dim=(0, 2), unbiased=False)
    rel = ((r["sv"].double() - var).abs() / var.clamp_min(1e-30)).max().item()
    assert rel < 1e-4, rel
    zf, dzf = z.double(), r["dz"].cuda().double()
    dy = torch.where(zf >= 0, dzf, dzf * 0.01)
    dbeta = dy.sum(dim=(0, 2))
    err = ((r["db"].double() - dbeta).abs().max() / dbeta.abs().max()).item()
    assert err < TOL["bf16"], err
