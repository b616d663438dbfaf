"""Multi-process (world size 2, gloo, CPU) coverage of the N > 1 host logic:
process-group rendezvous on 127.0.0.1, broadcast of the communicator id,
strong-scaling shards, the sync semantics of the split-phase buffers (raw fp64
moments and gradient sums are summed over ranks; R7)
checked against the oracle on the concatenated batch, and the max-over-ranks
timing reduction of bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface failures to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    return out


# ---------------------------------------------------------------- worker bodies (module level: picklable)
def _id_broadcast(rank, world):
    from paper_1712_02616_b200.functional import broadcast_unique_id
    uid = broadcast_unique_id(None, lambda: bytes(range(128)))
    return uid == bytes(range(128))


def _sync_stats(rank, world):
    """Forward: each rank's raw moments (count, sum, sumsq) of its shard, summed
    over ranks with the collective, give the statistics of the whole batch."""
    import oracle
    import synth_inputs as S
    from bench import shard_sizes
    N, C, HW = 7, 5, 12
    x = S.make_x(N, C, HW, 3).double().numpy()
    sizes = shard_sizes(N, world)
    lo = sum(sizes[:rank])
    xs = x[lo:lo + sizes[rank]]
    raw = np.stack([np.full(C, xs.shape[0] * HW, dtype=np.float64), xs.sum(axis=(0, 2)),
                    (xs * xs).sum(axis=(0, 2))], axis=1)  # [C][3], the iabn_forward_reduce layout
    t = torch.from_numpy(raw.copy())
    dist.all_reduce(t)
    g = t.numpy()
    mean = g[:, 1] / g[:, 0]
    var = g[:, 2] / g[:, 0] - mean ** 2
    ref_mean, ref_var = oracle.load().channel_stats(x)
    return (float(np.max(np.abs(mean - ref_mean))), float(np.max(np.abs(var - ref_var) / ref_var)),
            float(g[0, 0]))


def _sync_grads(rank, world):
    """Backward: per-rank (S1, S2) with the GLOBAL statistics, summed over ranks,
    equal the oracle's dbeta and dgamma~ on the whole batch; the count slot of
    the [2C+1] buffer sums to the global m."""
    import oracle
    import synth_inputs as S
    from bench import shard_sizes
    N, C, HW = 6, 4, 10
    x = S.make_x(N, C, HW, 4).double().numpy()
    dz = S.make_dz(N, C, HW, 4).double().numpy()
    p = S.make_params(C, 4)
    g, b = p.gamma.double().numpy(), p.beta.double().numpy()
    o = oracle.load()
    f = o.forward(x, g, b)  # global statistics (what the forward all-reduce produced)
    gt = np.abs(g) + 1e-5
    sizes = shard_sizes(N, world)
    lo = sum(sizes[:rank])
    zs, dzs = f.z[lo:lo + sizes[rank]], dz[lo:lo + sizes[rank]]
    dy = np.where(zs >= 0, dzs, 0.01 * dzs)
    y = np.where(zs >= 0, zs, zs / 0.01)
    xh = (y - b[None, :, None]) / gt[None, :, None]
    sums = np.zeros(2 * C + 1)
    sums[0:2 * C:2] = dy.sum(axis=(0, 2))
    sums[1:2 * C:2] = (dy * xh).sum(axis=(0, 2))
    sums[2 * C] = zs.shape[0] * HW
    t = torch.from_numpy(sums)
    dist.all_reduce(t)
    _, dg, db = o.backward_standard(x, dz, g, b)
    s = t.numpy()
    e1 = np.max(np.abs(s[0:2 * C:2] - db)) / np.max(np.abs(db))
    e2 = np.max(np.abs(s[1:2 * C:2] * np.where(g < 0, -1, 1) - dg)) / np.max(np.abs(dg))
    return float(e1), float(e2), float(s[2 * C])


def _max_timing(rank, world):
    from bench import max_over_ranks
    return max_over_ranks([1.0 + rank, 5.0 - rank], "cpu", dist, world)


def _dist_plumb(rank, world):
    """bench.py's N > 1 plumbing (DistPlumb): barrier and element-wise max over ranks."""
    from bench import DistPlumb
    pl = DistPlumb(rank, world, "cpu")
    pl.barrier()
    m = pl.allmax([float(rank), 10.0 - rank, -1.0 * rank])
    pl.barrier()
    return m


# ---------------------------------------------------------------- tests
def test_bench_dist_plumb():
    out = _run(_dist_plumb)
    assert out[0] == out[1] == [1.0, 10.0, 0.0]


def test_bench_preflight_env():
    from bench import preflight_env
    env = preflight_env({"MASTER_PORT": "29500", "RANK": "1", "TORCHELASTIC_USE_AGENT_STORE": "True",
                         "TORCHELASTIC_RUN_ID": "x", "WORLD_SIZE": "2"})
    assert env == {"MASTER_PORT": "29517", "RANK": "1", "WORLD_SIZE": "2"}

def test_unique_id_broadcast():
    out = _run(_id_broadcast)
    assert out == {0: True, 1: True}


def test_sync_forward_statistics_equal_concatenated_batch():
    out = _run(_sync_stats)
    for rank, (emean, evar, count) in out.items():
        assert emean < 1e-12 and evar < 1e-12 and count == 7 * 12


def test_sync_backward_sums_equal_concatenated_batch():
    out = _run(_sync_grads)
    for rank, (e1, e2, count) in out.items():
        assert e1 < 1e-12 and e2 < 1e-10 and count == 6 * 10


def test_max_over_ranks():
    out = _run(_max_timing)
    assert out[0] == [2.0, 5.0] and out[1] == [2.0, 5.0]


@pytest.mark.parametrize("N,G", [(16, 1), (16, 2), (16, 4), (16, 8), (7, 3)])
def test_strong_scaling_shards(N, G):
    from bench import shard_sizes
    s = shard_sizes(N, G)
    assert sum(s) == N and max(s) - min(s) <= 1 and len(s) == G
