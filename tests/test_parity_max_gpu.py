"""Maximum sizes: a tensor of more than 2^31 elements (4.3 GB bf16 per tensor), so the
streaming schedule's elementwise passes run in several launches of < 2^31 elements
and the 32-bit per-channel counts (m = N*HW = 2.1 M) are exercised far from their
small-test values.  Sampled whole channels against the oracle, as in
test_parity_full_gpu.py."""
import numpy as np
import pytest
import torch

import synth_inputs as S
from tests.harness import Case, compare, run_oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_more_than_2_pow_31_elements():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    N, C, HW = 16, 1024, 131200
    assert N * C * HW > 2**31
    dev = torch.device("cuda", 0)
    x = S.make_x(N, C, HW, 7, dtype="bf16", device=dev)
    dz = S.make_dz(N, C, HW, 7, dtype="bf16", device=dev)
    pc = S.make_params(C, 7)  # CPU draw, so the oracle sees the same parameters
    p = S.Params(pc.gamma.to(dev), pc.beta.to(dev), pc.running_mean.to(dev),
                 pc.running_var.to(dev))
    rng = np.random.default_rng(7)
    chans = sorted({0, C - 1, *rng.choice(C, 6, replace=False).tolist()})
    ch = torch.tensor(chans, device=dev)
    xs, dzs = x[:, ch, :].cpu(), dz[:, ch, :].cpu()  # inputs of the sampled channels
    d = L.desc(N, C, HW, L.BF16, L.NCHW)
    assert L.query_schedule(d, 0)[0] == 0  # 4.2 MB channels: streaming
    z, sm, sv = P.forward(x, p.gamma, p.beta, p.running_mean, p.running_var)
    dx, dg, db = P.backward(z, dz, p.gamma, p.beta, sv)
    torch.cuda.synchronize()
    got = dict(z=z[:, ch, :].cpu(), dx=dx[:, ch, :].cpu(), mean=sm[ch].cpu(), var=sv[ch].cpu(),
               rm=p.running_mean[ch].cpu(), rv=p.running_var[ch].cpu(), dgamma=dg[ch].cpu(),
               dbeta=db[ch].cpu())
    sub = Case(N, len(chans), HW, dtype="bf16")
    ps = S.Params(pc.gamma[chans], pc.beta[chans], pc.running_mean[chans],
                  pc.running_var[chans])
    ref = run_oracle(sub, xs, dzs, ps)
    print("2^31+ parity:", compare(sub, got, ref, ps))
    # every channel: finite outputs (the last launch chunk included)
    assert torch.isfinite(z[-1].float()).all() and torch.isfinite(dx[-1].float()).all()
