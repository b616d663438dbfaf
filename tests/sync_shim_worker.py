"""Worker of tests/test_sync_shim_gpu.py (test infrastructure, run as a subprocess).

G ranks as G threads on one GPU, each on its own stream with its own shard of one
seeded global batch (split along N, shards may differ in size), call
``iabn_forward_sync`` / ``iabn_backward_sync`` through the Python binding with an
``iabn_comm`` of G ranks.  NCCL is the test NCCL of tests/nccl_shim (IABN_NCCL_LIB, set
before the package loads), so the library's reduce -> ncclAllReduce -> apply path runs
with nranks = G on one GPU.  Results go to an .npz for the parent test, which compares
them with the oracle on the concatenated batch.

    python tests/sync_shim_worker.py OUT.npz --shards 3,5 --C 24 --HW 196 --dtype f32 \
        --layout NCHW --seed 60 [--global-param-grads] [--gamma-mode abs_eps]
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from tests import nccl_shim  # noqa: E402

os.environ["IABN_NCCL_LIB"] = nccl_shim.build()

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1712_02616_b200 as P  # noqa: E402
import synth_inputs as S  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--shards", required=True)
    ap.add_argument("--C", type=int, required=True)
    ap.add_argument("--HW", type=int, required=True)
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--layout", default="NCHW")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--gamma-mode", default="abs_eps")
    ap.add_argument("--global-param-grads", action="store_true")
    ap.add_argument("--eps", type=float, default=1e-5)
    ap.add_argument("--slope", type=float, default=0.01)
    ap.add_argument("--momentum", type=float, default=0.1)
    ap.add_argument("--sync-fused", action="store_true",
                    help="request the fused-collective kernels (IABN_SYNC_FUSED); the ranks "
                         "must then agree to fall back (unequal shards, no fused plan)")
    a = ap.parse_args()

    shards = [int(s) for s in a.shards.split(",")]
    G, Ntot = len(shards), sum(shards)
    offs = np.concatenate([[0], np.cumsum(shards)]).astype(int)
    x = S.make_x(Ntot, a.C, a.HW, a.seed, layout=a.layout, dtype=a.dtype)
    dz = S.make_dz(Ntot, a.C, a.HW, a.seed, layout=a.layout, dtype=a.dtype)
    p = S.make_params(a.C, a.seed)
    torch.cuda.set_device(0)
    uid = P.Comm.unique_id()
    shim = ctypes.CDLL(os.environ["IABN_NCCL_LIB"])
    shim.shim_allreduce_calls.restype = ctypes.c_uint64
    shim.shim_allgather_calls.restype = ctypes.c_uint64
    calls0 = shim.shim_allreduce_calls()
    gathers0 = shim.shim_allgather_calls()
    flags = P._lib.SYNC_FUSED if a.sync_fused else 0
    res: list[dict | None] = [None] * G
    errs: list[BaseException] = []

    def rank(r: int):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                comm = P.Comm.create(G, r, uid)
                try:
                    out = []
                    for it in range(2):  # the second call must reproduce the first bit for bit
                        comm.set_timing(it == 1)  # phase events on the second call
                        xr = x[offs[r]:offs[r + 1]].cuda()
                        dzr = dz[offs[r]:offs[r + 1]].cuda()
                        g, b = p.gamma.cuda(), p.beta.cuda()
                        rm, rv = p.running_mean.cuda(), p.running_var.cuda()
                        z, sm, sv = P.forward(xr, g, b, rm, rv, momentum=a.momentum, eps=a.eps,
                                              slope=a.slope, gamma_mode=a.gamma_mode,
                                              layout=a.layout, comm=comm, flags=flags)
                        dx, dg, db = P.backward(z, dzr, g, b, sv, eps=a.eps, slope=a.slope,
                                                gamma_mode=a.gamma_mode, layout=a.layout,
                                                comm=comm, flags=flags,
                                                global_param_grads=a.global_param_grads)
                        st.synchronize()
                        out.append({k: v.float().cpu().numpy() for k, v in dict(
                            z=z, dx=dx, mean=sm, var=sv, rm=rm, rv=rv, dgamma=dg,
                            dbeta=db).items()})
                    for k in out[0]:
                        assert np.array_equal(out[0][k], out[1][k]), f"rank {r}: {k} not repeatable"
                    res[r] = out[1]
                    ph = comm.phase_ms()
                    res[r]["phases"] = np.array([ph[p_][k] for p_ in ("forward", "backward")
                                                 for k in ("reduce", "allreduce", "apply")])
                finally:
                    comm.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    calls = shim.shim_allreduce_calls() - calls0
    gathers = shim.shim_allgather_calls() - gathers0
    cat = lambda k: np.concatenate([res[r][k] for r in range(G)], axis=0)  # noqa: E731
    np.savez(a.out, z=cat("z"), dx=cat("dx"),
             mean=np.stack([res[r]["mean"] for r in range(G)]),
             var=np.stack([res[r]["var"] for r in range(G)]),
             rm=np.stack([res[r]["rm"] for r in range(G)]),
             rv=np.stack([res[r]["rv"] for r in range(G)]),
             dgamma=np.stack([res[r]["dgamma"] for r in range(G)]),
             dbeta=np.stack([res[r]["dbeta"] for r in range(G)]),
             phases=np.stack([res[r]["phases"] for r in range(G)]),
             allreduce_calls=np.array(calls), allgather_calls=np.array(gathers))
    print(f"sync shim worker: G={G} shards={shards} all-reduce calls={calls} "
          f"all-gather calls={gathers}")


if __name__ == "__main__":
    main()
