"""Pins for the CPU oracle: checks against what the paper and mathematics fix,
never against the oracle's own formulas retyped.  Each pin is a function of an
``oracle.Oracle`` that raises AssertionError on failure, so the same list runs
against the real oracle (tests/test_oracle_pins.py, all must pass) and against
deliberately broken builds (tests/test_oracle_mutants.py, each must trip at
least one pin).

What pins what:
  golden_*           SPEC.md worked examples (hand values of PAPER.md Eq.(1), f, f^-1)
  whitening          closed form: mean_c(x^) = 0, var_c(x^) = var/(var+eps)  (Eq.(1))
  torch_f64_*        library routine: torch float64 batch_norm + leaky_relu + autograd
  finite_diff        brute force: central differences of L = sum w*z, stats recomputed
  three_way          algebra: stored-x chain rule == Alg.2 I (from z) == Alg.2 II (BN-dagger)
  const_dz           closed form: a = 1, dz = const -> dx = 0, dbeta = m*const, dgamma = 0
  dx_moments         closed forms: sum_c dx = 0, sum_c dx*x^ = g*rstd*dg*eps/(var+eps)
  scaling            metamorphic: x -> 2^k x, eps -> 4^k eps leaves z, scales dx by 2^-k
  sync_concat        merged shard stats == stats of the concatenated batch
  golden_fold        SPEC.md folding examples (identity BN, beta shift)
  fold_conv          library routine: torch float64 conv2d(w', b') == batch_norm(eval)(conv2d(w, b))
"""
from __future__ import annotations

import json
import os

import numpy as np
import torch
import torch.nn.functional as F

from tests.util import chan_err, rel_err, vec_err

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                      "spec_worked_examples.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _rand_problem(N=3, C=5, HW=7, seed=0, layout="NCHW", gamma_neg=True):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(N, C, HW)) * rng.uniform(0.5, 3, size=(1, C, 1)) \
        + rng.uniform(-2, 2, size=(1, C, 1))
    gamma = rng.uniform(0.5, 1.5, size=C)
    if gamma_neg:
        gamma[::2] *= -1
    beta = rng.uniform(-0.5, 0.5, size=C)
    dz = rng.normal(size=(N, C, HW))
    if layout == "NHWC":
        x = np.ascontiguousarray(x.transpose(0, 2, 1))
        dz = np.ascontiguousarray(dz.transpose(0, 2, 1))
    return x, dz, gamma, beta


# ---------------------------------------------------------------- golden
def pin_golden_bn(o):
    g = _golden()["bn_1234"]
    x = np.array(g["x"]).reshape(4, 1, 1)
    r = o.forward(x, [g["gamma"]], [g["beta"]], eps=1e-5, slope=1.0, gamma_mode="plain")
    assert abs(r.mean[0] - g["mean"]) < 1e-12 and abs(r.var[0] - g["var"]) < 1e-12
    assert np.max(np.abs(r.z.ravel() - np.array(g["y"]))) < g["tol"]
    r1 = o.forward(x, [1.0], [0.0], eps=1e-5, slope=1.0, gamma_mode="plain")
    assert np.max(np.abs(r1.z.ravel() - np.array(g["xhat"]))) < g["tol"]
    # with the paper's slope a = 0.01 only the negative entry changes
    ra = o.forward(x, [g["gamma"]], [g["beta"]], eps=1e-5, slope=0.01, gamma_mode="plain")
    want = np.array(g["y"]) * np.where(np.array(g["y"]) < 0, 0.01, 1.0)
    assert np.max(np.abs(ra.z.ravel() - want)) < g["tol"]


def pin_golden_leaky(o):
    gd = _golden()
    f = gd["leaky_forward"]
    y = np.array(f["y"]).reshape(1, 3, 1)  # eval mode with r_mu=0, r_var=1, eps=0 -> z = f(x)
    z = o.forward_eval(y, np.ones(3), np.zeros(3), np.zeros(3), np.ones(3), eps=0.0,
                       slope=f["slope"], gamma_mode="fixed_one")
    assert np.max(np.abs(z.ravel() - np.array(f["z"]))) < 1e-15
    b = gd["leaky_backward_from_output"]
    z = np.array(b["z"]).reshape(1, 2, 1)
    dz = np.array(b["dz"]).reshape(1, 2, 1)
    # m = 1 per channel: dbeta = dy (Alg. 2 l.2); BN-dagger with gamma~=1, beta=0 gives
    # dgamma = dy*y, so y = dgamma/dbeta = f^-1(z)
    _, dg, db = o.backward_inplace_II(z, dz, np.ones(2), np.ones(2), np.zeros(2), eps=1e-5,
                                      slope=b["slope"], gamma_mode="fixed_one")
    assert np.max(np.abs(db - np.array(b["dy"]))) < 1e-15
    assert np.max(np.abs(dg / db - np.array([-3.0, 2.0]))) < 1e-12


def pin_golden_running(o):
    g = _golden()["running_update"]
    x = np.full((2, 1, 1), g["batch_mean"])
    r = o.forward(x, [1.0], [0.0], momentum=g["momentum"], running_mean=[g["running_mean"]],
                  running_var=[1.0])
    assert abs(r.running_mean[0] - g["expected"]) < 1e-12


def pin_golden_running_biased(o):
    """IABN_RUNNING_VAR_BIASED follows SPEC.md's reading (:224, :272): the running
    variance is updated with the biased batch variance."""
    g = _golden()["running_update_var_biased"]
    x = np.array(g["x"]).reshape(-1, 1, 1)
    r = o.forward(x, [1.0], [0.0], momentum=g["momentum"], running_mean=[g["running_mean"]],
                  running_var=[g["running_var"]], running_var_biased=True)
    assert abs(r.running_mean[0] - g["expected_running_mean"]) < 1e-12
    assert abs(r.running_var[0] - g["expected_running_var"]) < 1e-12


def pin_golden_sync(o):
    g = _golden()["sync_merge"]
    shards = [np.array(s).reshape(-1, 1, 1) for s in g["shards"]]
    st = [o.channel_stats(s) for s in shards]
    cnt, mean, var = o.merge_stats([s.shape[0] for s in shards], [m for m, _ in st],
                                   [v for _, v in st])
    assert cnt == g["count"] and abs(mean[0] - g["mean"]) < 1e-15 and abs(var[0] - g["var"]) < 1e-15


# ---------------------------------------------------------------- closed forms
def pin_whitening(o):
    for layout in ("NCHW", "NHWC"):
        x, _, _, _ = _rand_problem(4, 6, 9, seed=1, layout=layout)
        C = 6
        eps = 1e-3
        r = o.forward(x, np.ones(C), np.zeros(C), eps=eps, slope=1.0, gamma_mode="fixed_one",
                      layout=layout)
        xh = r.z if layout == "NCHW" else r.z.transpose(0, 2, 1)
        xs = x if layout == "NCHW" else x.transpose(0, 2, 1)
        m_ = xh.mean(axis=(0, 2))
        v_ = ((xh - m_[None, :, None]) ** 2).mean(axis=(0, 2))
        true_var = xs.var(axis=(0, 2))
        assert np.max(np.abs(m_)) < 1e-12
        assert np.max(np.abs(v_ - true_var / (true_var + eps))) < 1e-12


def pin_const_dz(o):
    x, _, gamma, beta = _rand_problem(3, 4, 5, seed=2)
    dz = np.full_like(x, 0.75)
    dx, dg, db = o.backward_standard(x, dz, gamma, beta, slope=1.0)
    assert np.max(np.abs(dx)) < 1e-12
    assert np.max(np.abs(db - 15 * 0.75)) < 1e-12
    assert np.max(np.abs(dg)) < 1e-12


def pin_dx_moments(o):
    eps = 1e-2  # large eps so that the second moment identity is far from 0
    for layout in ("NCHW", "NHWC"):
        x, dz, gamma, beta = _rand_problem(4, 5, 6, seed=3, layout=layout)
        dx, dg, _ = o.backward_standard(x, dz, gamma, beta, eps=eps, layout=layout)
        xs = x if layout == "NCHW" else x.transpose(0, 2, 1)
        dxs = dx if layout == "NCHW" else dx.transpose(0, 2, 1)
        mu = xs.mean(axis=(0, 2), keepdims=True)
        var = xs.var(axis=(0, 2), keepdims=True)
        xhat = (xs - mu) / np.sqrt(var + eps)
        scale = np.abs(dxs).max()
        assert np.max(np.abs(dxs.sum(axis=(0, 2)))) < 1e-12 * scale * xs[:, 0].size
        g = np.abs(gamma) + eps
        dgt = dg * np.where(gamma < 0, -1.0, 1.0)  # gradient w.r.t. gamma~
        v = var.ravel()
        lhs = (dxs * xhat).sum(axis=(0, 2))
        rhs = g / np.sqrt(v + eps) * dgt * eps / (v + eps)
        assert np.max(np.abs(lhs - rhs)) < 1e-10 * max(1.0, np.abs(rhs).max())


# ---------------------------------------------------------------- library routine
def _torch_ref(x, dz, gamma, beta, eps, slope, momentum, layout):
    """PyTorch float64: F.batch_norm(training=True) + F.leaky_relu + autograd,
    with weight = |gamma| + eps (the reparametrised scale, R4)."""
    xt = torch.tensor(x if layout == "NCHW" else x.transpose(0, 2, 1), dtype=torch.float64,
                      requires_grad=True)
    dzt = torch.tensor(dz if layout == "NCHW" else dz.transpose(0, 2, 1), dtype=torch.float64)
    gt = torch.tensor(gamma, dtype=torch.float64, requires_grad=True)
    bt = torch.tensor(beta, dtype=torch.float64, requires_grad=True)
    C = len(gamma)
    rm = torch.zeros(C, dtype=torch.float64)
    rv = torch.ones(C, dtype=torch.float64)
    w = gt.abs() + eps
    y = F.batch_norm(xt, rm, rv, weight=w, bias=bt, training=True, momentum=momentum, eps=eps)
    z = F.leaky_relu(y, negative_slope=slope)
    z.backward(dzt)
    back = (lambda t: t) if layout == "NCHW" else (lambda t: t.permute(0, 2, 1))
    return (back(z.detach()).numpy(), back(xt.grad).numpy(), gt.grad.numpy(), bt.grad.numpy(),
            rm.numpy(), rv.numpy())


def pin_torch_f64(o):
    for layout in ("NCHW", "NHWC"):
        for seed in (4, 5):
            x, dz, gamma, beta = _rand_problem(4, 6, 10, seed=seed, layout=layout)
            ax = 1 if layout == "NCHW" else 2
            zt, dxt, dgt, dbt, rmt, rvt = _torch_ref(x, dz, gamma, beta, 1e-5, 0.01, 0.1, layout)
            r = o.forward(x, gamma, beta, eps=1e-5, slope=0.01, momentum=0.1,
                          running_mean=np.zeros(6), running_var=np.ones(6), layout=layout)
            dx, dg, db = o.backward_standard(x, dz, gamma, beta, eps=1e-5, slope=0.01,
                                             layout=layout)
            assert chan_err(r.z, zt, ax) < 1e-12
            assert chan_err(dx, dxt, ax) < 1e-12
            assert vec_err(dg, dgt) < 1e-12 and vec_err(db, dbt) < 1e-12
            assert vec_err(r.running_mean, rmt) < 1e-12 and vec_err(r.running_var, rvt) < 1e-12


def pin_torch_eval(o):
    x, _, gamma, beta = _rand_problem(3, 4, 6, seed=6)
    rm = np.array([0.1, -0.2, 0.3, 0.0])
    rv = np.array([1.5, 0.5, 2.0, 1.0])
    z = o.forward_eval(x, gamma, beta, rm, rv, eps=1e-5, slope=0.01)
    y = F.batch_norm(torch.tensor(x), torch.tensor(rm), torch.tensor(rv),
                     weight=torch.tensor(np.abs(gamma) + 1e-5), bias=torch.tensor(beta),
                     training=False, eps=1e-5)
    zt = F.leaky_relu(y, 0.01).numpy()
    assert chan_err(z, zt, 1) < 1e-13


# ---------------------------------------------------------------- brute force
def _loss(o, x, w, gamma, beta, gamma_mode, slope, eps):
    r = o.forward(x, gamma, beta, eps=eps, slope=slope, gamma_mode=gamma_mode)
    return float((w * r.z).sum())


def pin_finite_diff(o):
    """Central differences of L = sum w*z on the tiny config (N=2, C=8, 4x4),
    perturbing x BEFORE statistics, for dx, dgamma, dbeta."""
    N, C, HW, eps, slope, h = 2, 8, 16, 1e-5, 0.01, 1e-6
    for gamma_mode in ("abs_eps", "plain"):
        seed = 7
        while True:
            x, w, gamma, beta = _rand_problem(N, C, HW, seed=seed)
            y = o.forward(x, gamma, beta, eps=eps, slope=1.0, gamma_mode=gamma_mode).z
            if np.min(np.abs(y)) > 1e-4:  # keep away from the kink (R15)
                break
            seed += 100
        dx, dg, db = o.backward_standard(x, w, gamma, beta, eps=eps, slope=slope,
                                         gamma_mode=gamma_mode)
        fd = np.empty_like(x)
        for i in range(x.size):
            xp, xm = x.copy(), x.copy()
            xp.flat[i] += h
            xm.flat[i] -= h
            fd.flat[i] = (_loss(o, xp, w, gamma, beta, gamma_mode, slope, eps)
                          - _loss(o, xm, w, gamma, beta, gamma_mode, slope, eps)) / (2 * h)
        fdg, fdb = np.empty(C), np.empty(C)
        for c in range(C):
            for arr, out in ((gamma, fdg), (beta, fdb)):
                p, m = arr.copy(), arr.copy()
                p[c] += h
                m[c] -= h
                if arr is gamma:
                    lp = _loss(o, x, w, p, beta, gamma_mode, slope, eps)
                    lm = _loss(o, x, w, m, beta, gamma_mode, slope, eps)
                else:
                    lp = _loss(o, x, w, gamma, p, gamma_mode, slope, eps)
                    lm = _loss(o, x, w, gamma, m, gamma_mode, slope, eps)
                out[c] = (lp - lm) / (2 * h)
        assert rel_err(dx, fd) < 1e-6, rel_err(dx, fd)
        assert rel_err(dg, fdg) < 1e-6, rel_err(dg, fdg)
        assert rel_err(db, fdb) < 1e-6, rel_err(db, fdb)


# ---------------------------------------------------------------- algebra
def pin_three_way(o):
    """Standard-from-x == InPlace-ABN I from z == InPlace-ABN II from y, to 1e-10
    in double (Appendix :452-460)."""
    for layout in ("NCHW", "NHWC"):
        for gamma_mode in ("abs_eps", "plain", "fixed_one"):
            x, dz, gamma, beta = _rand_problem(3, 6, 11, seed=8, layout=layout)
            ax = 1 if layout == "NCHW" else 2
            r = o.forward(x, gamma, beta, eps=1e-5, slope=0.01, gamma_mode=gamma_mode,
                          layout=layout)
            ref = o.backward_standard(x, dz, gamma, beta, eps=1e-5, slope=0.01,
                                      gamma_mode=gamma_mode, layout=layout)
            for fn in (o.backward_inplace_I, o.backward_inplace_II):
                got = fn(r.z, dz, r.var, gamma, beta, eps=1e-5, slope=0.01,
                         gamma_mode=gamma_mode, layout=layout)
                assert chan_err(got[0], ref[0], ax) < 1e-10
                assert vec_err(got[1], ref[1]) < 1e-10 and vec_err(got[2], ref[2]) < 1e-10


def pin_fixed_one(o):
    """gamma fixed to 1: z does not depend on gamma, and the
    returned dgamma is dL/dgamma~ at gamma~ = 1, i.e. the plain-mode gradient at
    gamma = 1 (itself pinned by finite differences)."""
    x, dz, gamma, beta = _rand_problem(2, 4, 8, seed=9)
    r1 = o.forward(x, gamma, beta, gamma_mode="fixed_one")
    r2 = o.forward(x, 3 * gamma, beta, gamma_mode="fixed_one")
    rp = o.forward(x, np.ones(4), beta, gamma_mode="plain")
    assert np.array_equal(r1.z, r2.z) and np.max(np.abs(r1.z - rp.z)) < 1e-15
    _, dg1, db1 = o.backward_standard(x, dz, gamma, beta, gamma_mode="fixed_one")
    _, dgp, dbp = o.backward_standard(x, dz, np.ones(4), beta, gamma_mode="plain")
    assert vec_err(dg1, dgp) < 1e-14 and vec_err(db1, dbp) < 1e-14


# ---------------------------------------------------------------- metamorphic
def pin_scaling(o):
    x, dz, gamma, beta = _rand_problem(3, 5, 8, seed=10)
    k, eps = 3, 1e-4
    r = o.forward(x, gamma, beta, eps=eps, gamma_mode="plain")
    rs = o.forward(x * 2.0 ** k, gamma, beta, eps=eps * 4.0 ** k, gamma_mode="plain")
    assert chan_err(rs.z, r.z, 1) < 1e-13
    dx = o.backward_standard(x, dz, gamma, beta, eps=eps, gamma_mode="plain")[0]
    dxs = o.backward_standard(x * 2.0 ** k, dz, gamma, beta, eps=eps * 4.0 ** k,
                              gamma_mode="plain")[0]
    assert chan_err(dxs * 2.0 ** k, dx, 1) < 1e-12


def pin_sync_concat(o):
    """sync_stats(split(t, k)) == stats(t)."""
    x, _, _, _ = _rand_problem(8, 5, 6, seed=11)
    mean, var = o.channel_stats(x)
    for k in (2, 4):
        shards = np.split(x, k, axis=0)
        st = [o.channel_stats(s) for s in shards]
        cnt, mm, vv = o.merge_stats([s.shape[0] * s.shape[2] for s in shards],
                                    [a for a, _ in st], [b for _, b in st])
        assert cnt == x.shape[0] * x.shape[2]
        assert np.max(np.abs(mm - mean)) < 1e-12 and np.max(np.abs(vv - var)) < 1e-12


def pin_sharded_param_grads(o):
    """Per-shard dgamma/dbeta of the synchronized layer (R7): their sum
    over shards is the whole batch's gradient (the brute-force/torch-pinned
    backward_standard); one shard is the whole batch; a batch made of two copies of x
    gives each copy x's own gradient (the statistics of [x; x] are those of x)."""
    for layout in ("NCHW", "NHWC"):
        for mode in ("abs_eps", "plain"):
            x, dz, gamma, beta = _rand_problem(7, 5, 6, seed=21, layout=layout)
            _, dg, db = o.backward_standard(x, dz, gamma, beta, gamma_mode=mode, layout=layout)
            sdg, sdb = o.param_grads_sharded(x, dz, gamma, beta, [2, 3, 2], gamma_mode=mode,
                                             layout=layout)
            assert vec_err(sdg.sum(0), dg) < 1e-12 and vec_err(sdb.sum(0), db) < 1e-12
            one_g, one_b = o.param_grads_sharded(x, dz, gamma, beta, [7], gamma_mode=mode,
                                                 layout=layout)
            assert vec_err(one_g[0], dg) < 1e-13 and vec_err(one_b[0], db) < 1e-13
            x2, dz2 = np.concatenate([x, x]), np.concatenate([dz, dz])
            hg, hb = o.param_grads_sharded(x2, dz2, gamma, beta, [7, 7], gamma_mode=mode,
                                           layout=layout)
            for k in range(2):
                assert vec_err(hg[k], dg) < 1e-12 and vec_err(hb[k], db) < 1e-12


def pin_act_torch_f64(o):
    """Other invertible activations: BN + sigmoid / tanh from stored x against
    PyTorch float64 (F.batch_norm, torch.sigmoid / torch.tanh, autograd), both layouts."""
    for act, fn in (("sigmoid", torch.sigmoid), ("tanh", torch.tanh)):
        for layout in ("NCHW", "NHWC"):
            x, dz, gamma, beta = _rand_problem(4, 5, 9, seed=31, layout=layout)
            z, mean, var = o.forward_act(x, gamma, beta, act=act, layout=layout)
            dx, dg, db = o.backward_standard_act(x, dz, gamma, beta, act=act, layout=layout)
            xt = torch.tensor(x if layout == "NCHW" else np.transpose(x, (0, 2, 1)),
                              requires_grad=True)
            gt = torch.tensor(gamma, requires_grad=True)
            bt = torch.tensor(beta, requires_grad=True)
            geff = gt.abs() + 1e-5
            zt = fn(F.batch_norm(xt, None, None, weight=geff, bias=bt, training=True, eps=1e-5))
            dzt = torch.tensor(dz if layout == "NCHW" else np.transpose(dz, (0, 2, 1)))
            zt.backward(dzt)
            tr = (lambda a: a) if layout == "NCHW" else (lambda a: np.transpose(a, (0, 2, 1)))
            assert chan_err(z, tr(zt.detach().numpy()), 1 if layout == "NCHW" else 2) < 1e-12
            assert chan_err(dx, tr(xt.grad.numpy()), 1 if layout == "NCHW" else 2) < 1e-10
            assert vec_err(dg, gt.grad.numpy()) < 1e-10 and vec_err(db, bt.grad.numpy()) < 1e-10


def pin_act_inplace_equals_stored_x(o):
    """Alg. 2 from z (f^-1, f' from z) equals the stored-x chain rule for sigmoid / tanh
    (the invariant of BASELINE.json: 'gradient via inversion of z equals gradient via
    stored x'); with act = leaky it reduces to oracle_backward_inplace_I."""
    for act in ("sigmoid", "tanh", "leaky"):
        x, dz, gamma, beta = _rand_problem(5, 4, 8, seed=32)
        z, mean, var = o.forward_act(x, gamma, beta, act=act)
        a = o.backward_standard_act(x, dz, gamma, beta, act=act)
        b = o.backward_inplace_act(z, dz, var, gamma, beta, act=act)
        for u, v in zip(a, b):
            assert rel_err(v, u) < 1e-9, act
    x, dz, gamma, beta = _rand_problem(5, 4, 8, seed=33)
    f = o.forward(x, gamma, beta)
    ref = o.backward_inplace_I(f.z, dz, f.var, gamma, beta)
    got = o.backward_inplace_act(f.z, dz, f.var, gamma, beta, act="leaky")
    for u, v in zip(ref, got):
        assert rel_err(v, u) < 1e-14


def pin_permute_batch(o):
    x, dz, gamma, beta = _rand_problem(5, 4, 6, seed=12)
    perm = np.array([3, 0, 4, 1, 2])
    r = o.forward(x, gamma, beta)
    rp = o.forward(x[perm], gamma, beta)
    assert chan_err(rp.z, r.z[perm], 1) < 1e-13
    assert vec_err(rp.var, r.var) < 1e-13
    dx = o.backward_standard(x, dz, gamma, beta)[0]
    dxp = o.backward_standard(x[perm], dz[perm], gamma, beta)[0]
    assert chan_err(dxp, dx[perm], 1) < 1e-12


# ---------------------------------------------------------------- test-time folding
def pin_golden_fold(o):
    g = _golden()
    for key in ("fold_identity", "fold_beta_shift"):
        e = g[key]
        eps = 1e-5
        w_out, b_out = o.fold_conv(np.array(e["w"]), np.array(e["bias"]),
                                   np.array([e["running_mean"]]),
                                   np.array([e["running_var_plus_eps"] - eps]),
                                   np.array([e["gamma"]]), np.array([e["beta"]]), eps=eps,
                                   gamma_mode="plain")
        assert np.abs(w_out - np.array(e["w_out"])).max() < 1e-12, key
        assert np.abs(b_out - np.array(e["bias_out"])).max() < 1e-12, key


def pin_fold_conv(o):
    rng = np.random.default_rng(11)
    for kh, with_bias in ((3, True), (1, False)):
        x = rng.normal(size=(2, 3, 6, 5))
        w = rng.normal(size=(4, 3, kh, kh))
        b = rng.normal(size=4) if with_bias else None
        gamma = rng.uniform(0.5, 1.5, 4) * np.array([1, -1, 1, 1])
        beta, rm = rng.normal(size=4), rng.normal(size=4)
        rv = rng.uniform(0.2, 3.0, 4)
        w2, b2 = o.fold_conv(w, b, rm, rv, gamma, beta, eps=1e-5)
        v = F.conv2d(torch.tensor(x), torch.tensor(w), None if b is None else torch.tensor(b))
        two_stage = F.batch_norm(v, torch.tensor(rm), torch.tensor(rv),
                                 weight=torch.tensor(np.abs(gamma) + 1e-5),
                                 bias=torch.tensor(beta), training=False, eps=1e-5)
        folded = F.conv2d(torch.tensor(x), torch.tensor(w2), torch.tensor(b2))
        assert (folded - two_stage).abs().max().item() < 1e-12 * max(1.0, two_stage.abs().max().item())


PINS = [pin_golden_bn, pin_golden_leaky, pin_golden_running, pin_golden_running_biased,
        pin_golden_sync, pin_sharded_param_grads, pin_whitening,
        pin_const_dz, pin_dx_moments, pin_torch_f64, pin_torch_eval, pin_finite_diff,
        pin_three_way, pin_fixed_one, pin_scaling, pin_sync_concat, pin_permute_batch,
        pin_golden_fold, pin_fold_conv, pin_act_torch_f64, pin_act_inplace_equals_stored_x]
