#!/usr/bin/env python
"""Benchmark of the InPlace-ABN hot path on B200 (BASELINE.json metric:
"InPlace-ABN fwd+bwd achieved HBM GB/s (% of peak) at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config wrn38|r50s3|tiny]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

A step = one forward (Alg. 1: statistics, normalise/affine/leaky-ReLU, z written
over x) + one backward (Alg. 2 I: from z and dz only, dx written over dz) of one
BN+Act layer on a synthetic batch resident in HBM.  Default workload
(BASELINE.json configs[3], the one quoted "at 1/2/4/8 B200"): WideResNet-38
segmentation crops, global batch 16 x 4096 x 112 x 112, bf16, NCHW; strong
scaling -- rank r holds its share of the 16 crops and, for N > 1, the batch
statistics and gradient sums are all-reduced over NVLink with NCCL inside the
library (InPlace-ABN^sync).

value = algorithmic HBM bytes of all ranks per step / max-over-ranks step time,
where the algorithmic bytes are the method's minimum, 5*E*b per layer (forward
reads x and writes z; backward reads z and dz and writes dx; DESIGN.md
"Roofline").  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "InPlace-ABN fwd+bwd achieved HBM GB/s (% of peak) at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024

WORKLOADS = {
    "wrn38": dict(N=16, C=4096, HW=112 * 112, dtype="bf16", layout="NCHW",
                  desc="WideResNet-38 segmentation crops 16x4096x112x112 bf16 NCHW "
                       "(BASELINE.json configs[3]); sync InPlace-ABN, strong scaling"),
    "r50s3": dict(N=64, C=1024, HW=14 * 14, dtype="f32", layout="NCHW",
                  desc="ResNet-50 stage-3 activation 64x1024x14x14 fp32 NCHW "
                       "(BASELINE.json configs[1])"),
    "tiny": dict(N=2, C=8, HW=16, dtype="f32", layout="NCHW",
                 desc="tiny 2x8x4x4 fp32 (BASELINE.json configs[0])"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(WORKLOADS), default="wrn38")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--schedule", choices=["auto", "streaming", "fused"], default="auto",
                    help="schedule override (IABN_FORCE_*), for experiments")
    ap.add_argument("--sync", choices=["nccl", "fused"], default="nccl",
                    help="N > 1: reduce / ncclAllReduce / apply kernels (default), or the "
                         "fused-collective kernels (IABN_SYNC_FUSED: record exchange over "
                         "NVLink inside the channel-resident kernels)")
    ap.add_argument("--sync-emulated", type=int, default=8,
                    help="N = 1: also time the fused-collective sync over this many virtual "
                         "ranks on the same workload (one-GPU emulation; 0 = off)")
    return ap.parse_args()


def shard_sizes(N: int, world: int) -> list[int]:
    """Strong scaling: rank r holds samples [N r / G, N (r+1) / G) of the global batch."""
    return [N * (r + 1) // world - N * r // world for r in range(world)]


def max_over_ranks(values, device, dist, world: int) -> list[float]:
    """Element-wise max of per-rank timings (the slowest rank defines the step)."""
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def load_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


SCHEDULES = ["streaming", "fused", "one-launch", "grid-resident"]  # iabn_query_schedule codes


def load_traffic(config: str):
    """dram read+write bytes per launch of the dominant kernel from the committed
    ncu --set full capture summary (profiles/), if one exists for this workload."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(config)
    except Exception:
        return None


# ---------------------------------------------------------------- clocks (NVML, during the timed region)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}
    BAD = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}

    def __init__(self, device_index: int):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            try:
                import torch
                pr = torch.cuda.get_device_properties(device_index)
                bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = get_reasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(self.samples)}

    def bad(self) -> bool:
        s = self.summary()
        if not self.ok or not self.samples:
            return False
        stuck = s["sm_mhz"] is not None and self.max_mhz and s["sm_mhz"] < 0.5 * self.max_mhz \
            and not (set(s["reasons"]) - {"gpu_idle"})
        return bool(self.BAD & set(s["reasons"])) or bool(stuck)


# ---------------------------------------------------------------- CPU oracle baseline
def oracle_sample(wl: dict, channels: int, seed: int = 0):
    import synth_inputs as S
    x = S.make_x(wl["N"], channels, wl["HW"], seed, dtype=wl["dtype"])
    dz = S.make_dz(wl["N"], channels, wl["HW"], seed, dtype=wl["dtype"])
    p = S.make_params(channels, seed)
    import numpy as np
    f64 = lambda t: t.to(__import__("torch").float64).numpy()  # noqa: E731
    return (np.ascontiguousarray(f64(x)), np.ascontiguousarray(f64(dz)), f64(p.gamma),
            f64(p.beta), f64(p.running_mean), f64(p.running_var))


def oracle_step(o, sample):
    x, dz, g, b, rm, rv = sample
    o.forward(x, g, b, running_mean=rm, running_var=rv)
    o.backward_standard(x, dz, g, b)


def cpu_cores() -> int:
    n = os.environ.get("OMP_NUM_THREADS")
    if n and n.isdigit():
        return int(n)
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(wl: dict, seconds: float) -> dict:
    """The oracle as it stands, on a bounded sample of the same workload."""
    import oracle
    o = oracle.load()
    b = 2 if wl["dtype"] == "bf16" else 4
    # calibrate on one channel, then size the sample to ~seconds/3 per step
    one = oracle_sample(wl, 1)
    oracle_step(o, one)
    t0 = time.perf_counter()
    oracle_step(o, one)
    t1 = max(time.perf_counter() - t0, 1e-4)
    ch = int(max(1, min(wl["C"], (seconds / 3.0) / t1)))
    sample = oracle_sample(wl, ch)
    times = []
    start = time.perf_counter()
    while len(times) < 3 or (time.perf_counter() - start < seconds and len(times) < 20):
        t0 = time.perf_counter()
        oracle_step(o, sample)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - start > 3 * seconds:
            break
    E = wl["N"] * ch * wl["HW"]
    t = statistics.median(times)
    return {"value": round(5 * E * b / t / 1e9, 4), "unit": "GB/s", "cores": cpu_cores(),
            "kind": "oracle",
            "sample": f"{ch} of {wl['C']} channels ({wl['N']}x{ch}x{wl['HW']}, {E} elements, "
                      f"bf16 values widened to fp64), oracle forward + stored-x backward, "
                      f"median of {len(times)} runs, {t:.3f} s each",
            "elements_per_s": round(E / t, 1)}


def run_reference(args, wl):
    """--impl reference: the CPU oracle timed on host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    o = oracle.load()
    b = 2 if wl["dtype"] == "bf16" else 4
    one = oracle_sample(wl, 1)
    oracle_step(o, one)  # first call pays library/OpenMP start-up
    t0 = time.perf_counter()
    oracle_step(o, one)
    t1 = max(time.perf_counter() - t0, 1e-4)
    budget = 120.0 / max(args.steps + args.warmup, 1)  # whole run within ~2 minutes
    ch = int(max(1, min(wl["C"], budget / t1)))
    sample = oracle_sample(wl, ch)
    for _ in range(args.warmup):
        oracle_step(o, sample)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_step(o, sample)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    E = wl["N"] * ch * wl["HW"]
    value = 5 * E * b / dt / 1e9
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config + ": " + wl["desc"], "sample_channels": ch,
                       "N": wl["N"], "HW": wl["HW"]},
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cpu_cores(),
                             "kind": "oracle",
                             "sample": f"{ch} of {wl['C']} channels per step "
                                       f"({wl['N']}x{ch}x{wl['HW']})"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def main():
    args = parse()
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    import synth_inputs as S

    N_local = shard_sizes(wl["N"], world)[rank]
    C, HW = wl["C"], wl["HW"]
    b = 2 if wl["dtype"] == "bf16" else 4
    E = N_local * C * HW
    E_all = wl["N"] * C * HW
    comm = P.Comm.from_process_group() if world > 1 else None

    # inputs resident in HBM (same recipe as the parity tests, drawn on the device)
    x = S.make_x(N_local, C, HW, 1000 + rank, dtype=wl["dtype"], device=dev)
    dz = S.make_dz(N_local, C, HW, 1000 + rank, dtype=wl["dtype"], device=dev)
    prm = S.make_params(C, 0, device=dev)
    g, bt, rm, rv = prm.gamma, prm.beta, prm.running_mean, prm.running_var
    st = torch.cuda.current_stream()

    # keep the repeated in-place application bounded: re-standardise x and dz once
    # outside the timed region if they drift (z of a layer is the next layer's input)
    fl = {"auto": 0, "streaming": L.FORCE_STREAMING, "fused": L.FORCE_FUSED}[args.schedule]
    if world > 1 and args.sync == "fused":
        fl |= L.SYNC_FUSED

    def step():
        z, sm, sv = P.forward(x, g, bt, rm, rv, comm=comm, flags=fl)
        P.backward(z, dz, g, bt, sv, comm=comm, flags=fl)

    fits_l2 = 2 * E * b < 2 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if fits_l2 else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    def timed():
        K = args.steps
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = L.launch_count()
        t_start.record(st)
        step_ms = []
        for i in range(K):
            if flush is not None:  # L2-resident workload: flush, time the step alone
                flush.add_(1.0)
            evs[i][0].record(st)
            z, sm, sv = P.forward(x, g, bt, rm, rv, comm=comm, flags=fl)
            evs[i][1].record(st)
            P.backward(z, dz, g, bt, sv, comm=comm, flags=fl)
            evs[i][2].record(st)
        t_end.record(st)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches = L.launch_count() - launches0
        fwd = [a.elapsed_time(bb) for a, bb, _ in evs]
        bwd = [bb.elapsed_time(c) for _, bb, c in evs]
        if flush is not None:
            total = sum(f + w for f, w in zip(fwd, bwd))
        else:
            total = t_start.elapsed_time(t_end)
        return total, fwd, bwd, launches

    with ClockSampler(local) as clk:
        total_ms, fwd, bwd, launches = timed()
    rejected = None
    if clk.bad():
        rejected = clk.summary()
        with ClockSampler(local) as clk:
            total_ms, fwd, bwd, launches = timed()

    # max over ranks
    total_ms, fwd_sum, bwd_sum = max_over_ranks([total_ms, sum(fwd), sum(bwd)], dev, dist, world)
    K = args.steps
    ms_per_step = total_ms / K
    bytes_step_all = 5 * E_all * b
    value = bytes_step_all / (ms_per_step * 1e-3) / 1e9
    peak, peak_src = load_peak()

    # dominant kernel: the backward (3*E*b algorithmic bytes per launch)
    bwd_ms = bwd_sum / K
    fwd_ms = fwd_sum / K
    qfl = fl if world == 1 or args.sync == "fused" else L.FORCE_STREAMING
    s_f, k_f = L.query_schedule(L.desc(N_local, C, HW, L.BF16 if b == 2 else L.F32, L.NCHW), 0,
                                qfl)
    s_b, k_b = L.query_schedule(L.desc(N_local, C, HW, L.BF16 if b == 2 else L.F32, L.NCHW), 1,
                                qfl)
    bwd_bytes = 3 * E * b
    achieved = bwd_bytes / (bwd_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config) if world == 1 else None

    # ---- end to end: pinned host buffers in, results out, every step
    e2e = None
    if args.e2e_steps > 0:
        # End to end through the public API with host buffers, pipelined the way a data
        # loader would: copies in on one stream, compute on the main stream, results out
        # on a third (PCIe is full duplex), device input buffers double-buffered so step
        # i+1's upload overlaps step i's download.  Every step still uploads x and dz from
        # pinned host memory and downloads z, dx, dgamma and dbeta.
        dt = {2: torch.bfloat16, 4: torch.float32}[b]
        xh = torch.empty(x.shape, dtype=dt, pin_memory=True)
        dzh = torch.empty(dz.shape, dtype=dt, pin_memory=True)
        xh.copy_(x)
        dzh.copy_(dz)
        zh = torch.empty_like(xh, pin_memory=True)
        dxh = torch.empty_like(dzh, pin_memory=True)
        pg = torch.empty(2 * C, dtype=torch.float32, pin_memory=True)
        xs = [x, torch.empty_like(x)]
        dzs = [dz, torch.empty_like(dz)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev = lambda: torch.cuda.Event()  # noqa: E731
        out_done = [None, None]  # step i's downloads of slot i % 2 finished

        def e2e_step(i):
            k = i % 2
            xd, dzd = xs[k], dzs[k]
            with torch.cuda.stream(s_in):
                if out_done[k] is not None:
                    s_in.wait_event(out_done[k])  # slot k's previous results are out
                xd.copy_(xh, non_blocking=True)
                x_in = ev()
                x_in.record(s_in)
                dzd.copy_(dzh, non_blocking=True)
                dz_in = ev()
                dz_in.record(s_in)
            st.wait_event(x_in)
            z, sm, sv = P.forward(xd, g, bt, rm, rv, comm=comm)
            f_done = ev()
            f_done.record(st)
            st.wait_event(dz_in)
            dx, dgam, dbet = P.backward(z, dzd, g, bt, sv, comm=comm)
            b_done = ev()
            b_done.record(st)
            with torch.cuda.stream(s_out):
                s_out.wait_event(f_done)
                zh.copy_(z, non_blocking=True)
                s_out.wait_event(b_done)
                dxh.copy_(dx, non_blocking=True)
                pg[:C].copy_(dgam, non_blocking=True)
                pg[C:].copy_(dbet, non_blocking=True)
                out_done[k] = ev()
                out_done[k].record(s_out)

        e2e_step(0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s_in)
        for i in range(args.e2e_steps):
            e2e_step(i + 1)
        c.record(s_out)
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(c) / args.e2e_steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = te.item()
        e2e = {"value": round(bytes_step_all / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": 2 * E * b, "d2h_bytes_per_step": 2 * E * b + 2 * C * 4,
               "ms_per_step": round(e2e_ms, 3), "steps": args.e2e_steps,
               "path": "pinned host -> HBM (copy stream), iabn_forward + iabn_backward (C ABI), "
                       "HBM -> pinned host (copy stream); uploads of step i+1 overlap downloads of step i"}

    # all-reduce overhead of the sync variant (same message sizes, NCCL, device-timed)
    allreduce = None
    if world > 1:
        msgs = {"forward_stats_fp64": 3 * C, "backward_sums_fp64": 2 * C + 1}
        allreduce = {}
        for name, n in msgs.items():
            buf = torch.zeros(n, dtype=torch.float64, device=dev)
            for _ in range(5):
                dist.all_reduce(buf)
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(50):
                dist.all_reduce(buf)
            c.record(st)
            torch.cuda.synchronize()
            tt = torch.tensor([a.elapsed_time(c) / 50 * 1e3], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            allreduce[name] = {"bytes": n * 8, "us": round(tt.item(), 2),
                               "pct_of_step": round(100 * tt.item() * 1e-3 / ms_per_step, 2)}

    # synchronized variant on one GPU: the fused-collective kernels over G virtual ranks
    # (the G shards of this workload, records exchanged through the peer-record protocol)
    sync_emu = None
    G = args.sync_emulated
    if world == 1 and G > 1 and wl["N"] % G == 0 and wl["layout"] == "NCHW":
        def emu_step():
            z, _, sv = P.forward_sync_emulated(x, G, g, bt, rm, rv)
            P.backward_sync_emulated(z, dz, G, g, bt, sv)
            return sv
        for _ in range(3):
            emu_step()
        torch.cuda.synchronize()
        ne = max(1, min(args.steps, 50))
        fe, be = [], []
        for _ in range(ne):
            if flush is not None:
                flush.add_(1.0)
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(st)
            z, _, sv = P.forward_sync_emulated(x, G, g, bt, rm, rv)
            e1.record(st)
            P.backward_sync_emulated(z, dz, G, g, bt, sv)
            e2.record(st)
            torch.cuda.synchronize()
            fe.append(e0.elapsed_time(e1))
            be.append(e1.elapsed_time(e2))
        ems = (sum(fe) + sum(be)) / ne
        ev_ = bytes_step_all / (ems * 1e-3) / 1e9
        sync_emu = {"virtual_ranks": G, "N_per_rank": wl["N"] // G, "value": round(ev_, 2),
                    "unit": "GB/s", "pct_of_peak": round(100 * ev_ / peak, 2),
                    "ms_per_step": round(ems, 4), "fwd_ms": round(sum(fe) / ne, 4),
                    "bwd_ms": round(sum(be) / ne, 4), "steps": ne,
                    "path": "iabn_forward_sync_emulated + iabn_backward_sync_emulated: one "
                            "cooperative launch per pass, G ranks' channel records exchanged "
                            "in-kernel (no NCCL launch); 5*E*b bytes"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": K, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": f"{args.config}: {wl['desc']}", "global_batch": wl["N"],
                       "N_local": N_local, "C": C, "HW": HW, "layout": wl["layout"],
                       "parallelism": f"dp{world}" + (f"+sync-stats({args.sync})" if world > 1 else ""),
                       "l2": ("inputs larger than L2 (x, dz %.2f GB each)" % (E * b / 1e9))
                       if flush is None else "L2 flushed before every timed step",
                       "schedule": {"forward": SCHEDULES[s_f] + (f" K={k_f}" if s_f == 1 else ""),
                                    "backward": SCHEDULES[s_b] + (f" K={k_b}" if s_b == 1 else "")},
                       "algorithmic_bytes_per_step": bytes_step_all},
            "pct_of_peak": round(100 * value / peak, 2),
            "elements_per_s": round(E_all / (ms_per_step * 1e-3), 1),
            "effective_8Eb_GBps": round(8 * E_all * b / (ms_per_step * 1e-3) / 1e9, 2),
            "fwd_ms": round(fwd_ms, 4), "bwd_ms": round(bwd_ms, 4),
            "roofline": {"bound": "hbm", "kernel": "fused_bwd_kernel" if s_b else "backward pass",
                         "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "algorithmic_bytes_per_launch": bwd_bytes, "peak_source": peak_src,
                         "forward": {"kernel": "fused_fwd_kernel" if s_f else "forward pass",
                                     "achieved": round(2 * E * b / (fwd_ms * 1e-3) / 1e9, 2),
                                     "frac": round(2 * E * b / (fwd_ms * 1e-3) / 1e9 / peak, 4),
                                     "algorithmic_bytes_per_launch": 2 * E * b}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if rejected:
            line["clocks_rejected_first_run"] = rejected
        if allreduce:
            line["allreduce"] = allreduce
        if sync_emu:
            line["sync_emulated"] = sync_emu
        print(json.dumps(line), flush=True)

    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
