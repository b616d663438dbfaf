"""InPlace-ABN^sync through the library's reduce -> ncclAllReduce -> apply path with
nranks >= 2 (PAPER.md:315 "virtual increase of batch size", :356 "gradient-synchronized").

The ranks are threads of one subprocess on one GPU, each with its own stream, shard and
``iabn_comm``; NCCL is the test NCCL of tests/nccl_shim (loaded through IABN_NCCL_LIB),
whose all-reduce sums the ranks' fp64 buffers in rank order on the device.  Expected
values come from the oracle on the concatenated batch: z and dx element-wise, the
statistics and running statistics on every rank, and each rank's local dgamma / dbeta
(reading R7) from ``oracle.param_grads_sharded``.  The worker also asserts that a second
call reproduces the first bit for bit; this test asserts that the all-reduce really ran
(2 calls per rank per step) -- a one-rank communicator would skip it.
"""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from tests.harness import TOL, Case, ambiguous, dx_err, inputs, run_oracle, shard_param_errs, to64
from tests.util import chan_err, vec_err

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

CASES = [
    # (shards, C, HW, dtype, layout, gamma_mode, global_param_grads[, sync_fused requested])
    ((3, 5), 24, 196, "f32", "NCHW", "abs_eps", False),
    # fused-collective kernels requested, but the ranks cannot all run them with one plan
    # (unequal shards; NHWC has no channel-resident plan): the collective agreement
    # (one all-gather per shape and pass) sends every rank down the all-reduce path
    ((3, 5), 24, 196, "f32", "NCHW", "abs_eps", False, True),
    ((2, 2), 40, 64, "bf16", "NHWC", "abs_eps", False, True),
    ((2, 2), 64, 3136, "bf16", "NCHW", "abs_eps", False),
    ((1, 2, 3, 2), 40, 784, "bf16", "NCHW", "abs_eps", False),
    ((4, 2), 64, 49, "bf16", "NHWC", "abs_eps", False),
    ((2, 1, 3), 37, 77, "f32", "NCHW", "plain", True),
    ((16, 16, 16, 16), 1024, 196, "f32", "NCHW", "abs_eps", False),  # cfg2 over 4 ranks
    ((1, 1), 16, 1, "f32", "NHWC", "abs_eps", False),                 # global m = 2
]


def _id(c):
    return f"G{len(c[0])}_{'-'.join(map(str, c[0]))}x{c[1]}x{c[2]}_{c[3]}_{c[4]}" + \
        ("_global" if c[6] else "") + ("_fused_requested" if c[7:] and c[7] else "")


@pytest.mark.parametrize("cfg", CASES, ids=[_id(c) for c in CASES])
def test_sync_nccl_path_multi_rank(cfg, tmp_path):
    shards, C, HW, dtype, layout, gmode, glob = cfg[:7]
    fused_req = len(cfg) > 7 and cfg[7]
    seed = 60 + CASES.index(cfg)
    out = tmp_path / "r.npz"
    cmd = [sys.executable, os.path.join(ROOT, "tests", "sync_shim_worker.py"), str(out),
           "--shards", ",".join(map(str, shards)), "--C", str(C), "--HW", str(HW),
           "--dtype", dtype, "--layout", layout, "--seed", str(seed), "--gamma-mode", gmode]
    if glob:
        cmd.append("--global-param-grads")
    if fused_req:
        cmd.append("--sync-fused")
    env = dict(os.environ)
    env.pop("IABN_SYNC_FUSED", None)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    got = np.load(out)
    G = len(shards)
    assert int(got["allreduce_calls"]) == 2 * 2 * G  # (fwd + bwd) x 2 calls x G ranks
    # the schedule agreement: one all-gather per pass and rank, cached for the second call
    assert int(got["allgather_calls"]) == (2 * G if fused_req else 0)
    # iabn_comm_phase_ms: every phase of both passes was timed on the device
    assert got["phases"].shape == (G, 6) and (got["phases"] > 0).all(), got["phases"]

    case = Case(sum(shards), C, HW, dtype=dtype, layout=layout, seed=seed, gamma_mode=gmode)
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    tol = TOL[dtype]
    amb = ambiguous(case, ref, p)
    errs = {"z": chan_err(got["z"], ref["z"], case.ax),
            "dx": dx_err(case, got["dx"].astype(np.float64), ref, p, amb)}
    if sum(shards) * HW <= 4:
        # m_G <= 4: dx = gamma~ rstd (dy - x^ S2/m - S1/m) cancels to O(eps / sigma^2) of its
        # terms (for m = 2 exactly (d1 - d2)/2 * eps/(sigma^2 + eps)), so fp32 can only be
        # judged against the size of the terms that cancel, gamma~ rstd |dz|
        gt = np.abs(to64(p.gamma)) + case.eps if gmode == "abs_eps" else np.abs(to64(p.gamma))
        shape = [1, 1, 1]
        shape[case.ax] = C
        term = (gt / np.sqrt(ref["var"] + case.eps)).reshape(shape) * np.abs(ref["dz"])
        axes = tuple(i for i in range(3) if i != case.ax)
        errs["dx"] = float(np.max(np.abs(got["dx"] - ref["dx"]).max(axis=axes)
                                  / term.max(axis=axes)))
    for r_ in range(G):  # every rank sees the global statistics
        for k in ("mean", "var", "rm", "rv"):
            errs[f"{k}[{r_}]"] = vec_err(got[k][r_], ref[k])
    for k in ("mean", "var"):
        assert all(np.array_equal(got[k][0], got[k][r_]) for r_ in range(G)), \
            f"{k} differs between ranks"
    o = __import__("oracle").load()
    dg_loc, db_loc = o.param_grads_sharded(to64(x), to64(dz), to64(p.gamma), to64(p.beta),
                                           list(shards), eps=case.eps, slope=case.slope,
                                           gamma_mode=gmode, layout=layout)
    n_off = np.concatenate([[0], np.cumsum(shards)])
    for r_ in range(G):
        if glob:  # IABN_SYNC_GLOBAL_PARAM_GRADS: every rank returns the whole batch's sums
            e = shard_param_errs(case, ref, amb, slice(0, n_off[-1]), got["dgamma"][r_],
                                 got["dbeta"][r_], dg_loc.sum(0), db_loc.sum(0))
        else:
            e = shard_param_errs(case, ref, amb, slice(n_off[r_], n_off[r_ + 1]),
                                 got["dgamma"][r_], got["dbeta"][r_], dg_loc[r_], db_loc[r_])
        errs.update({f"{k}[{r_}]": v for k, v in e.items()})
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"sync parity failed: {errs}"
