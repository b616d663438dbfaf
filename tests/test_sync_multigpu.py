"""InPlace-ABN^sync over real GPUs: one process per GPU, real NCCL.

Skipped below 2 visible GPUs (every lease of this build has one; the 8-GPU box runs it).
Each rank holds its shard of one seeded global batch (unequal shards in the NCCL case) and
calls the library through the Python binding with an ``iabn_comm`` built from the
torch.distributed group:

* the default reduce -> ncclAllReduce -> apply path;
* the fused-collective path (IABN_SYNC_FUSED: channel-resident kernels exchanging
  per-channel records with every peer over CUDA IPC mappings / NVLink inside the kernel),
  equal shards -- and, with unequal shards, the library's collective fallback to the
  NCCL path (the ranks agree on the schedule before any kernel waits on a peer).

Rank 0 gathers z, dx, statistics and per-rank dgamma/dbeta and compares them with the
oracle on the concatenated batch (the same checks as tests/test_sync_shim_gpu.py).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shards, C, HW, dtype, fused, seed, outdir):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    import synth_inputs as S

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    comm = P.Comm.from_process_group()
    try:
        N = sum(shards)
        off = sum(shards[:rank])
        x = S.make_x(N, C, HW, seed, dtype=dtype)[off:off + shards[rank]].cuda()
        dz = S.make_dz(N, C, HW, seed, dtype=dtype)[off:off + shards[rank]].cuda()
        p = S.make_params(C, seed)
        g, b = p.gamma.cuda(), p.beta.cuda()
        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
        fl = L.SYNC_FUSED if fused else 0
        z, sm, sv = P.forward(x, g, b, rm, rv, comm=comm, flags=fl)
        dx, dg, db = P.backward(z, dz, g, b, sv, comm=comm, flags=fl)
        torch.cuda.synchronize()
        np.savez(os.path.join(outdir, f"r{rank}.npz"),
                 **{k: v.float().cpu().numpy() for k, v in dict(
                     z=z, dx=dx, mean=sm, var=sv, rm=rm, rv=rv, dgamma=dg, dbeta=db).items()})
        dist.barrier()
    finally:
        comm.close()
        dist.destroy_process_group()


def _run(shards, C, HW, dtype, fused, seed, tmp_path):
    import torch.multiprocessing as mp
    world = len(shards)
    mp.spawn(_worker, args=(world, _free_port(), shards, C, HW, dtype, fused, seed,
                            str(tmp_path)), nprocs=world, join=True)
    return [dict(np.load(tmp_path / f"r{r}.npz")) for r in range(world)]


def _check(res, shards, C, HW, dtype, seed):
    from tests.harness import TOL, Case, ambiguous, dx_err, inputs, run_oracle, shard_param_errs, to64
    from tests.util import chan_err, vec_err
    import oracle
    case = Case(sum(shards), C, HW, dtype=dtype, seed=seed)
    x, dz, p = inputs(case)
    ref = run_oracle(case, x, dz, p)
    amb = ambiguous(case, ref, p)
    errs = {"z": chan_err(np.concatenate([r["z"] for r in res]), ref["z"], 1),
            "dx": dx_err(case, np.concatenate([r["dx"] for r in res]).astype(np.float64), ref, p,
                         amb)}
    dgl, dbl = oracle.load().param_grads_sharded(to64(x), to64(dz), to64(p.gamma),
                                                 to64(p.beta), list(shards))
    n_off = np.concatenate([[0], np.cumsum(shards)])
    for i, r in enumerate(res):
        for k in ("mean", "var", "rm", "rv"):
            errs[f"{k}[{i}]"] = vec_err(r[k], ref[k])
        e = shard_param_errs(case, ref, amb, slice(n_off[i], n_off[i + 1]), r["dgamma"],
                             r["dbeta"], dgl[i], dbl[i])
        errs.update({f"{k}[{i}]": v for k, v in e.items()})
    bad = {k: v for k, v in errs.items() if not v <= TOL[dtype]}
    assert not bad, errs


NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
need2 = pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs (one process per GPU)")


@need2
@pytest.mark.parametrize("fused", [False, True], ids=["nccl", "fused"])
def test_sync_real_gpus_equal_shards(fused, tmp_path):
    G = min(NGPU, 8)
    shards = [2] * G
    res = _run(shards, 64, 3136, "bf16", fused, 70, tmp_path)
    _check(res, shards, 64, 3136, "bf16", 70)


@need2
@pytest.mark.parametrize("fused", [False, True], ids=["nccl", "fused_requested"])
def test_sync_real_gpus_unequal_shards(fused, tmp_path):
    G = min(NGPU, 4)
    shards = [1 + r for r in range(G)]
    res = _run(shards, 40, 784, "f32", fused, 71, tmp_path)
    _check(res, shards, 40, 784, "f32", 71)
