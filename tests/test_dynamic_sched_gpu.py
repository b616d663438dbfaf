"""Dynamic channel scheduling of the channel-resident kernels (kernels_fused.cuh: clusters
draw channels from a ticket counter instead of the static q, q + Q, ... order).  The
per-channel arithmetic does not depend on which cluster processes a channel, so results
must be bitwise reproducible across calls, streams and CUDA-graph replays (the counters are
re-armed by each launch's last cluster), and match the oracle."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import synth_inputs as S
from tests.harness import Case, compare, run_oracle

pytestmark = pytest.mark.gpu


def _dyn_flag() -> int:
    from paper_1712_02616_b200 import _lib as L
    f = L.lib.iabn_debug_last_dynamic
    f.restype = __import__("ctypes").c_int
    return f()


def _run(x, dz, p, stream=None):
    import paper_1712_02616_b200 as P
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    z, sm, sv = P.forward(x.clone(), g, b, rm, rv, stream=stream)
    dx, dg, db = P.backward(z, dz.clone(), g, b, sv, stream=stream)
    return dict(z=z, dx=dx, mean=sm, var=sv, rm=rm, rv=rv, dgamma=dg, dbeta=db)


SHAPE = (8, 96, 112 * 112)  # bf16: 200 KB per channel -> large slices, dynamic order


def test_dynamic_parity_and_bitwise_repeat():
    N, C, HW = SHAPE
    case = Case(N, C, HW, dtype="bf16", seed=110)
    x = S.make_x(N, C, HW, 110, dtype="bf16")
    dz = S.make_dz(N, C, HW, 110, dtype="bf16")
    p = S.make_params(C, 110)
    xd, dzd = x.cuda(), dz.cuda()
    a = _run(xd, dzd, p)
    torch.cuda.synchronize()
    assert _dyn_flag() == 1, "expected the dynamic channel order on this shape"
    for _ in range(2):
        b = _run(xd, dzd, p)
        torch.cuda.synchronize()
        for k in a:
            assert torch.equal(a[k], b[k]), k
    rng = np.random.default_rng(5)
    ch = torch.tensor(sorted({0, C - 1, *rng.choice(C, 6, replace=False).tolist()}))
    sub = Case(N, len(ch), HW, dtype="bf16")
    ps = S.Params(p.gamma[ch], p.beta[ch], p.running_mean[ch], p.running_var[ch])
    chd = ch.cuda()
    got = dict(z=a["z"][:, chd].cpu(), dx=a["dx"][:, chd].cpu(), mean=a["mean"][chd].cpu(),
               var=a["var"][chd].cpu(), rm=a["rm"][chd].cpu(), rv=a["rv"][chd].cpu(),
               dgamma=a["dgamma"][chd].cpu(), dbeta=a["dbeta"][chd].cpu())
    compare(sub, got, run_oracle(sub, x[:, ch].contiguous(), dz[:, ch].contiguous(), ps), ps)


def test_dynamic_graph_replay_and_two_streams():
    N, C, HW = SHAPE
    x = S.make_x(N, C, HW, 111, dtype="bf16").cuda()
    dz = S.make_dz(N, C, HW, 111, dtype="bf16").cuda()
    p = S.make_params(C, 111)
    ref = _run(x, dz, p)
    torch.cuda.synchronize()
    import paper_1712_02616_b200 as P
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g, b = p.gamma.cuda(), p.beta.cuda()
    xs, dzs = x.clone(), dz.clone()
    with torch.cuda.stream(side):
        # first call on this stream outside the capture: its counters exist before capture
        P.forward(x.clone(), g, b, p.running_mean.cuda(), p.running_var.cuda())
        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            z, sm, sv = P.forward(xs, g, b, rm, rv)
            dx, dg, db = P.backward(z, dzs, g, b, sv)
    for _ in range(3):
        xs.copy_(x)
        dzs.copy_(dz)
        rm.copy_(p.running_mean.cuda())
        rv.copy_(p.running_var.cuda())
        graph.replay()
        torch.cuda.synchronize()
        for k, v in dict(z=z, dx=dx, mean=sm, var=sv, dgamma=dg, dbeta=db).items():
            assert torch.equal(v, ref[k]), k
    # two streams at once, each with its own counters
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        o1 = _run(x, dz, p, stream=s1)
    with torch.cuda.stream(s2):
        o2 = _run(x, dz, p, stream=s2)
    torch.cuda.synchronize()
    for k in ref:
        assert torch.equal(o1[k], ref[k]) and torch.equal(o2[k], ref[k]), k


@pytest.mark.slow
def test_dynamic_order_forced_on_small_slices_and_sync_emulation():
    """The dynamic order on every channel-resident launch (IABN_FUSED_DYN=2, IABN_SYNC_DYN=2:
    also small slices and the fused-collective sync over virtual ranks -- opt-in there --
    where each rank draws its own increasing channel sequence): the sync-emulation and plain
    parity suites rerun in a subprocess (the variables are read once per process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, IABN_FUSED_DYN="2", IABN_SYNC_DYN="2")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "tests/test_sync_fused_gpu.py", "tests/test_parity_gpu.py",
                        "-k", "not full_size"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
