"""Parity harness: run the CUDA path (through the C ABI) and the oracle on the
same seeded inputs, and compare.  Test infrastructure.

Tolerances (BASELINE.json north_star): max relative error 1e-4 for fp32
storage and 2e-2 for bf16 storage, per-channel normwise (reading R10).

Activation branch (reading R16): the GPU decides f / f' from the sign of its
fp32 y; the oracle from its fp64 y.  Where |y_oracle| < delta_c the two may
legitimately differ (both are correct within fp32), so those elements are
excluded from the elementwise dx comparison and their largest possible effect
(1 - a) |dz_i| (1 + |x^_i|) is added to the dgamma / dbeta tolerance.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

import synth_inputs as S
from tests.util import chan_err

TOL = {"f32": 1e-4, "bf16": 2e-2}


@dataclass
class Case:
    N: int
    C: int
    HW: int
    dtype: str = "f32"
    layout: str = "NCHW"
    seed: int = 0
    eps: float = 1e-5
    slope: float = 0.01
    momentum: float = 0.1
    gamma_mode: str = "abs_eps"
    stress: str | None = None

    @property
    def ax(self) -> int:  # channel axis of the 3-D storage view
        return 1 if self.layout == "NCHW" else 2


def inputs(case: Case):
    x = S.make_x(case.N, case.C, case.HW, case.seed, layout=case.layout, dtype=case.dtype,
                 stress=case.stress)
    dz = S.make_dz(case.N, case.C, case.HW, case.seed, layout=case.layout, dtype=case.dtype)
    p = S.make_params(case.C, case.seed)
    return x, dz, p


def to64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def run_gpu(case: Case, x, dz, p, *, flags=0, inplace=True, dx_inplace=True):
    import paper_1712_02616_b200 as P
    xd = x.cuda()
    dzd = dz.cuda()
    g, b = p.gamma.cuda(), p.beta.cuda()
    rm, rv = p.running_mean.cuda(), p.running_var.cuda()
    out = None if inplace else torch.empty_like(xd)
    z, sm, sv = P.forward(xd, g, b, rm, rv, momentum=case.momentum, eps=case.eps,
                          slope=case.slope, out=out, gamma_mode=case.gamma_mode,
                          layout=case.layout, flags=flags)
    if inplace:
        assert z.data_ptr() == xd.data_ptr()
    dxo = None if dx_inplace else torch.empty_like(dzd)
    dx, dg, db = P.backward(z, dzd, g, b, sv, save_mean=sm, eps=case.eps, slope=case.slope,
                            dx=dxo, gamma_mode=case.gamma_mode, layout=case.layout, flags=flags)
    torch.cuda.synchronize()
    return dict(z=z.cpu(), mean=sm.cpu(), var=sv.cpu(), rm=rm.cpu(), rv=rv.cpu(), dx=dx.cpu(),
                dgamma=dg.cpu(), dbeta=db.cpu())


def run_oracle(case: Case, x, dz, p):
    import oracle
    o = oracle.load()
    x64, dz64 = to64(x), to64(dz)
    g, b = to64(p.gamma), to64(p.beta)
    f = o.forward(x64, g, b, eps=case.eps, slope=case.slope, momentum=case.momentum,
                  running_mean=to64(p.running_mean), running_var=to64(p.running_var),
                  gamma_mode=case.gamma_mode, layout=case.layout)
    y = o.forward(x64, g, b, eps=case.eps, slope=1.0, gamma_mode=case.gamma_mode,
                  layout=case.layout).z
    dx, dg, db = o.backward_standard(x64, dz64, g, b, eps=case.eps, slope=case.slope,
                                     gamma_mode=case.gamma_mode, layout=case.layout)
    return dict(z=f.z, mean=f.mean, var=f.var, rm=f.running_mean, rv=f.running_var, dx=dx,
                dgamma=dg, dbeta=db, y=y, dz=dz64, x=x64)


def ambiguous(case: Case, ref, p) -> np.ndarray:
    """Elements whose activation branch fp32 cannot decide (R16)."""
    gamma = to64(p.gamma)
    g = {"abs_eps": np.abs(gamma) + case.eps, "plain": np.abs(gamma),
         "fixed_one": np.ones_like(gamma)}[case.gamma_mode]
    delta = 1e-5 * (np.abs(to64(p.beta)) + g)
    shape = [1, 1, 1]
    shape[case.ax] = case.C
    return np.abs(ref["y"]) < delta.reshape(shape)


def dx_err(case: Case, got_dx, ref, p, amb) -> float:
    """Per-channel normwise dx error (R10) with the R16 allowance.  An element whose
    activation branch fp32 cannot decide is excluded, and -- because its branch enters the
    channel sums -- every other dx_j of its channel may move by
      gamma~ rstd (1 - a) |dz_i| (1 + |x^_i| |x^_j|) / m
    (dx_j = gamma~ rstd (dy_j - x^_j S2/m - S1/m) with dS1 = (1 - a) dz_i, dS2 = dS1 x^_i),
    which is subtracted from the channel's absolute error before normalising."""
    gamma = to64(p.gamma)
    g = {"abs_eps": np.abs(gamma) + case.eps, "plain": np.abs(gamma),
         "fixed_one": np.ones_like(gamma)}[case.gamma_mode]
    shape = [1, 1, 1]
    shape[case.ax] = case.C
    axes = tuple(i for i in range(3) if i != case.ax)
    m = ref["dz"].size / case.C
    rstd = 1.0 / np.sqrt(ref["var"] + case.eps)
    xh = (ref["y"] - to64(p.beta).reshape(shape)) / g.reshape(shape)
    xh_max = np.abs(xh).max(axis=axes)
    allow = (g * rstd * (1 - case.slope) / m) * \
        (np.abs(ref["dz"]) * (1.0 + np.abs(xh) * xh_max.reshape(shape)) * amb).sum(axis=axes)
    d = np.where(amb, 0.0, np.abs(got_dx - ref["dx"]))
    d = np.maximum(d.max(axis=axes) - allow, 0.0)
    r = np.maximum(np.abs(ref["dx"]).max(axis=axes), 1e-30)
    return float(np.max(d / r))


def compare(case: Case, got, ref, p, *, tol=None):
    """Return dict of errors; raise AssertionError with all of them if any fails."""
    tol = TOL[case.dtype] if tol is None else tol
    amb = ambiguous(case, ref, p)
    errs = {}
    errs["z"] = chan_err(to64(got["z"]), ref["z"], case.ax)
    errs["dx"] = dx_err(case, to64(got["dx"]), ref, p, amb)
    for k in ("mean", "var", "rm", "rv"):
        r = ref[k]
        errs[k] = float(np.max(np.abs(to64(got[k]) - r)) / max(np.max(np.abs(r)), 1e-30))
    # dgamma/dbeta: allowance for ambiguous elements
    axes = tuple(i for i in range(3) if i != case.ax)
    xh = ref["y"]  # |x^| <= (|y| + |beta|)/g; bound loosely with |y| + 1
    allow = ((1 - case.slope) * np.abs(ref["dz"]) * (2.0 + np.abs(xh)) * amb).sum(axis=axes)
    for k in ("dgamma", "dbeta"):
        r = ref[k]
        scale = max(np.max(np.abs(r)), 1e-30)
        d = np.abs(to64(got[k]) - r) - allow
        errs[k] = float(max(np.max(d), 0.0) / scale)
    errs["n_ambiguous"] = int(amb.sum())
    bad = {k: v for k, v in errs.items() if k != "n_ambiguous" and not (v <= tol)}
    assert not bad, f"parity failed ({case}): {errs}"
    return errs


def shard_param_errs(case: Case, ref, amb, sl: slice, got_dg, got_db, exp_dg, exp_db) -> dict:
    """Normwise errors of one shard's dgamma / dbeta (samples ``sl`` of the concatenated
    batch) with the R16 allowance of that shard's ambiguous activation branches."""
    a = amb[sl]
    allow = (1 - case.slope) * np.abs(ref["dz"][sl]) * (2.0 + np.abs(ref["y"][sl])) * a
    allow = allow.sum(axis=tuple(i for i in range(3) if i != case.ax))
    out = {}
    for k, got, exp in (("dgamma", got_dg, exp_dg), ("dbeta", got_db, exp_db)):
        d = np.maximum(np.abs(np.asarray(got, dtype=np.float64) - exp) - allow, 0.0)
        out[k] = float(d.max() / max(np.abs(exp).max(), 1e-30))
    return out
