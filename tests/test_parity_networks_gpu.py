"""Parity over every distinct BN+Act layer shape of BASELINE.json configs[2] and [4]:
ResNeXt-101 32x4d (cfg3, PAPER.md:245 / Fig. 4's batch 32 per GPU, :414) and
DenseNet-264 (cfg5), N = 32, fp32 and bf16, NCHW and NHWC, on the
schedule each shape takes by default (channel-resident, covering-range or streaming).
DenseNet's BN reads the shared concatenated feature buffer, so its z and dx are out of
place; ResNeXt's are in place.

Channels are independent problems: the oracle checks three whole channels per shape
(first, last, one seeded-random) element by element; every channel is checked through a
property that holds at any size (dbeta = sum of dy recomputed from z and dz).  Inputs are
generated on the device (seeded Philox) and the sampled channels copied to the host.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth_inputs as S
from tests.harness import TOL, Case, compare, run_oracle

pytestmark = pytest.mark.gpu

N = 32


def _shapes(layers):
    seen, out = set(), []
    for s in layers:
        if s not in seen:
            seen.add(s)
            out.append(s)
    return out


RX = _shapes(S.rx101_layers())
DN = _shapes(S.densenet264_layers())
CASES = [("rx101", c, hw, dt, lay) for c, hw in RX for dt in ("f32", "bf16")
         for lay in ("NCHW", "NHWC")] + \
        [("densenet264", c, hw, dt, lay) for c, hw in DN for dt in ("f32", "bf16")
         for lay in ("NCHW", "NHWC")]


@pytest.mark.parametrize("net,C,HW,dtype,layout", CASES,
                         ids=[f"{n}_{c}x{hw}_{d}_{l}" for n, c, hw, d, l in CASES])
def test_network_layer_shape(net, C, HW, dtype, layout):
    import paper_1712_02616_b200 as P
    seed = (C * 7919 + HW) % 100_003
    dev = torch.device("cuda", 0)
    x = S.make_x(N, C, HW, seed, layout=layout, dtype=dtype, device=dev)
    dz = S.make_dz(N, C, HW, seed, layout=layout, dtype=dtype, device=dev)
    p = S.make_params(C, seed)
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    out_of_place = net == "densenet264"
    xin = x.clone() if not out_of_place else x
    zbuf = torch.empty_like(x) if out_of_place else None
    z, sm, sv = P.forward(xin, g, b, rm, rv, out=zbuf, layout=layout)
    dxbuf = torch.empty_like(dz) if out_of_place else None
    dzin = dz.clone() if not out_of_place else dz
    dx, dg, db = P.backward(z, dzin, g, b, sv, dx=dxbuf, layout=layout)
    torch.cuda.synchronize()
    if out_of_place:
        assert z.data_ptr() != x.data_ptr() and dx.data_ptr() != dz.data_ptr()

    rng = np.random.default_rng(seed)
    ch = sorted({0, C - 1, int(rng.integers(C))})
    cax = 1 if layout == "NCHW" else 2
    idx = torch.tensor(ch, device=dev)
    sub = Case(N, len(ch), HW, dtype=dtype, layout=layout, seed=seed)
    ps = S.Params(p.gamma[ch], p.beta[ch], p.running_mean[ch], p.running_var[ch])
    sel = lambda t: t.index_select(cax, idx).contiguous().cpu()  # noqa: E731
    ref = run_oracle(sub, sel(x), sel(dz), ps)
    got = dict(z=sel(z), dx=sel(dx), mean=sm[idx].cpu(), var=sv[idx].cpu(), rm=rm[idx].cpu(),
               rv=rv[idx].cpu(), dgamma=dg[idx].cpu(), dbeta=db[idx].cpu())
    compare(sub, got, ref, ps)

    # every channel: dbeta = sum dy, dy from the sign of z
    zf, dzf = z.double(), dz.double()
    dy = torch.where(zf >= 0, dzf, dzf * 0.01)
    red = (0, 2) if layout == "NCHW" else (0, 1)
    dbeta = dy.sum(dim=red)
    err = ((db.double() - dbeta).abs().max() / dbeta.abs().max()).item()
    assert err < TOL[dtype], err
