#!/usr/bin/env python
"""Benchmark of the InPlace-ABN hot path on B200 (BASELINE.json metric:
"InPlace-ABN fwd+bwd achieved HBM GB/s (% of peak) at 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config wrn38|r50s3|tiny]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

A step = one forward (Alg. 1: statistics, normalise/affine/leaky-ReLU, z written
over x) + one backward (Alg. 2 from z and dz only -- variant II (BN-dagger) in the
channel-resident kernels, I in the streaming ones; dx written over dz) of one
BN+Act layer on a synthetic batch resident in HBM.  Default workload
(BASELINE.json configs[3], the one quoted "at 1/2/4/8 B200"): WideResNet-38
segmentation crops, global batch 16 x 4096 x 112 x 112, bf16, NCHW; strong
scaling -- rank r holds its share of the 16 crops and, for N > 1, the batch
statistics and gradient sums are exchanged across GPUs inside the library
(InPlace-ABN^sync): the reduce / ncclAllReduce / apply path is timed
first (with per-phase device times from iabn_comm_phase_ms), then the fused-collective
kernels (per-channel records over NVLink inside the channel-resident kernels), which
are headlined only if a child-process preflight passed on every rank and their z and
dx agree with the NCCL path's.  ``pct_of_peak`` divides the aggregate GB/s by
N x the per-GPU peak.

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
    ap.add_argument("--e2e-steps", type=int, default=24)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--schedule", choices=["auto", "streaming", "fused"], default="auto",
                    help="schedule override (IABN_FORCE_*), for experiments")
    ap.add_argument("--sync", choices=["auto", "nccl", "fused"], default="auto",
                    help="N > 1: the reduce / ncclAllReduce / apply path is always timed "
                         "first (the checker); with auto (= fused) the fused-collective "
                         "kernels (IABN_SYNC_FUSED: record exchange over NVLink inside the "
                         "channel-resident kernels) are then preflighted in a child process, "
                         "checked against it and, if they agree, headlined; nccl skips them")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="dry run of the N > 1 path on ONE GPU: G ranks as threads, the "
                         "library's NCCL = the test NCCL (tests/nccl_shim)")
    ap.add_argument("--preflight-fused", action="store_true", help=argparse.SUPPRESS)
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
    # calibrate on a few channels, then size the sample to ~seconds/3 per step
    nc = min(wl["C"], 16)
    one = oracle_sample(wl, nc)
    oracle_step(o, one)
    t0 = time.perf_counter()
    oracle_step(o, one)
    t1 = max(time.perf_counter() - t0, 1e-5) / nc
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
    out = {"value": round(5 * E * b / t / 1e9, 4), "unit": "GB/s", "cores": cpu_cores(),
           "kind": "oracle",
           "sample": f"{ch} of {wl['C']} channels ({wl['N']}x{ch}x{wl['HW']}, {E} elements, "
                     f"{wl['dtype']} values widened to fp64), oracle forward + stored-x backward, "
                     f"median of {len(times)} runs, {t:.3f} s each",
           "elements_per_s": round(E / t, 1), "cpu_model": cpu_model()}
    # the same oracle on ONE thread (OpenMP over channels switched to 1), a smaller sample
    try:
        import ctypes
        gomp = ctypes.CDLL("libgomp.so.1")
        n0 = gomp.omp_get_max_threads()
        gomp.omp_set_num_threads(1)
        try:
            ch1 = max(1, ch // max(cpu_cores(), 1))
            s1 = oracle_sample(wl, ch1)
            oracle_step(o, s1)
            t1 = []
            for _ in range(2):
                t0 = time.perf_counter()
                oracle_step(o, s1)
                t1.append(time.perf_counter() - t0)
        finally:
            gomp.omp_set_num_threads(n0)
        E1 = wl["N"] * ch1 * wl["HW"]
        out["one_thread"] = {"value": round(5 * E1 * b / min(t1) / 1e9, 4), "unit": "GB/s",
                             "cores": 1, "sample": f"{ch1} channels, best of 2"}
    except Exception as e:  # noqa: BLE001
        out["one_thread"] = {"unavailable": str(e)[:200]}
    return out


def cpu_model() -> str | None:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


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


# ---------------------------------------------------------------- rank plumbing
class DistPlumb:
    """One process per GPU (torchrun): barrier and max-over-ranks through torch.distributed."""

    def __init__(self, rank, world, dev):
        self.rank, self.world, self.dev = rank, world, dev

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()

    def allmax(self, values):
        import torch
        import torch.distributed as dist
        t = torch.tensor(values, dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()


class ThreadPlumb:
    """Dry run of the N > 1 code path on ONE GPU (--emulate-ranks G): G ranks as threads,
    the library's NCCL being the test NCCL of tests/nccl_shim.  Validates the sharding,
    the reduce / all-reduce / apply calls, phase timing and the JSON line; its numbers
    are not a scaling measurement (the ranks share one GPU)."""

    def __init__(self, rank, world, dev, shared):
        self.rank, self.world, self.dev, self.sh = rank, world, dev, shared

    def barrier(self):
        self.sh["barrier"].wait()

    def allmax(self, values):
        self.sh["slots"][self.rank] = list(values)
        self.sh["barrier"].wait()
        out = [max(v[i] for v in self.sh["slots"]) for i in range(len(values))]
        self.sh["barrier"].wait()
        return out


def chan_err(a, b, layout_axis=1):
    """Per-channel normwise relative difference of two device tensors [N, C, HW]."""
    import torch
    d = (a.double() - b.double()).abs().amax(dim=(0, 2))
    r = b.double().abs().amax(dim=(0, 2)).clamp_min(1e-30)
    return float((d / r).max().item()) if d.numel() else 0.0


# ---------------------------------------------------------------- fused-collective preflight
def preflight_child(args, wl):
    """--preflight-fused (internal): run once in a child process per rank, on the bench's
    shard shape, the reduce / all-reduce / apply path and the fused-collective path, and
    compare z and dx.  A fault (or the ~20 s peer-wait trap) kills only this child."""
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    import synth_inputs as S
    comm = P.Comm.from_process_group()
    n = shard_sizes(wl["N"], world)[rank]
    x = S.make_x(n, wl["C"], wl["HW"], 2000 + rank, dtype=wl["dtype"], device=dev)
    dz = S.make_dz(n, wl["C"], wl["HW"], 2000 + rank, dtype=wl["dtype"], device=dev)
    prm = S.make_params(wl["C"], 0, device=dev)
    outs = []
    for fl in (0, L.SYNC_FUSED):
        rm, rv = prm.running_mean.clone(), prm.running_var.clone()
        z, _, sv = P.forward(x.clone(), prm.gamma, prm.beta, rm, rv, comm=comm, flags=fl)
        dx, dg, db = P.backward(z, dz.clone(), prm.gamma, prm.beta, sv, comm=comm, flags=fl)
        torch.cuda.synchronize()
        outs.append((z, dx))
    err = max(chan_err(outs[1][0], outs[0][0]), chan_err(outs[1][1], outs[0][1]))
    e = torch.tensor([err], dtype=torch.float64, device=dev)
    dist.all_reduce(e, op=dist.ReduceOp.MAX)
    comm.close()
    dist.destroy_process_group()
    tol = 1e-2 if wl["dtype"] == "bf16" else 1e-4
    print(f"PREFLIGHT err={e.item():.3e} tol={tol}", flush=True)
    sys.exit(0 if e.item() <= tol else 3)


def preflight_env(environ) -> dict:
    """Environment of a preflight child: a fresh rendezvous on another port; torchrun's
    agent store (which the parent's process group uses when TORCHELASTIC_USE_AGENT_STORE is
    set) must not be reused."""
    env = {k: v for k, v in environ.items() if not k.startswith("TORCHELASTIC")}
    env["MASTER_PORT"] = str(int(environ.get("MASTER_PORT", "29500")) + 17)
    return env


def preflight_fused(args, pl) -> tuple[bool, str]:
    """Every rank runs preflight_child in a subprocess (its own NCCL group on another
    port); the fused path is used only if every child exits 0."""
    import subprocess
    env = preflight_env(os.environ)
    cmd = [sys.executable, os.path.abspath(__file__), "--preflight-fused", "--config", args.config]
    try:
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
        ok, why = r.returncode == 0, (r.stdout + r.stderr).strip().splitlines()[-1:] or [""]
        why = f"rc={r.returncode} {why[0][:200]}"
    except subprocess.TimeoutExpired:
        ok, why = False, "timeout"
    bad = pl.allmax([0.0 if ok else 1.0])[0]
    return bad == 0.0, why


# ---------------------------------------------------------------- GPU arm
def run_rank(args, wl, pl, make_comm, emulated: bool):
    import torch

    import paper_1712_02616_b200 as P
    from paper_1712_02616_b200 import _lib as L
    import synth_inputs as S

    rank, world, dev = pl.rank, pl.world, pl.dev
    torch.cuda.set_device(dev)
    N_local = shard_sizes(wl["N"], world)[rank]
    C, HW = wl["C"], wl["HW"]
    b = 2 if wl["dtype"] == "bf16" else 4
    E = N_local * C * HW
    E_all = wl["N"] * C * HW
    comm = make_comm() if world > 1 else None

    # inputs resident in HBM (same recipe as the parity tests, drawn on the device)
    x = S.make_x(N_local, C, HW, 1000 + rank, dtype=wl["dtype"], device=dev)
    dz = S.make_dz(N_local, C, HW, 1000 + rank, dtype=wl["dtype"], device=dev)
    prm = S.make_params(C, 0, device=dev)
    g, bt, rm, rv = prm.gamma, prm.beta, prm.running_mean, prm.running_var
    st = torch.cuda.current_stream()
    base_fl = {"auto": 0, "streaming": L.FORCE_STREAMING, "fused": L.FORCE_FUSED}[args.schedule]
    fits_l2 = 2 * E * b < 2 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if fits_l2 else None
    peak, peak_src = load_peak()
    bytes_step_all = 5 * E_all * b

    def timed(fl, K):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pl.barrier()
        torch.cuda.synchronize()
        launches0 = L.launch_count()
        t_start.record(st)
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
        pl.barrier()
        launches = L.launch_count() - launches0
        fwd = [a.elapsed_time(bb) for a, bb, _ in evs]
        bwd = [bb.elapsed_time(c) for _, bb, c in evs]
        total = sum(f + w for f, w in zip(fwd, bwd)) if flush is not None \
            else t_start.elapsed_time(t_end)
        return total, fwd, bwd, launches

    def measure(fl):
        for _ in range(max(args.warmup, 3)):
            z, sm, sv = P.forward(x, g, bt, rm, rv, comm=comm, flags=fl)
            P.backward(z, dz, g, bt, sv, comm=comm, flags=fl)
        torch.cuda.synchronize()
        with ClockSampler(dev.index) as clk:
            r = timed(fl, args.steps)
        rejected = None
        if clk.bad():
            rejected = clk.summary()
            with ClockSampler(dev.index) as clk:
                r = timed(fl, args.steps)
        total_ms, fwd, bwd, launches = r
        total_ms, fwd_sum, bwd_sum = pl.allmax([total_ms, sum(fwd), sum(bwd)])
        K = args.steps
        return dict(ms_per_step=total_ms / K, fwd_ms=fwd_sum / K, bwd_ms=bwd_sum / K,
                    launches=launches, clocks=clk.summary(), rejected=rejected)

    def phases(fl, reps=5):
        """Library-recorded device time per phase (iabn_comm_phase_ms), median of reps
        calls, max over ranks."""
        comm.set_timing(True)
        rows = []
        for _ in range(reps):
            pl.barrier()
            z, sm, sv = P.forward(x, g, bt, rm, rv, comm=comm, flags=fl)
            P.backward(z, dz, g, bt, sv, comm=comm, flags=fl)
            ph = comm.phase_ms()
            rows.append([ph[p_][k] for p_ in ("forward", "backward")
                         for k in ("reduce", "allreduce", "apply")])
        comm.set_timing(False)
        med = [statistics.median(r[i] for r in rows) for i in range(6)]
        med = pl.allmax(med)
        names = ("reduce", "allreduce", "apply")
        out = {p_: {k: round(med[3 * i + j], 4) for j, k in enumerate(names)}
               for i, p_ in enumerate(("forward", "backward"))}
        ar_ms = med[1] + med[4]
        out["allreduce_ms_per_step"] = round(ar_ms, 4)
        out["allreduce_pct_of_step"] = round(100 * ar_ms / max(sum(med), 1e-9), 2)
        out["messages_bytes"] = {"forward_stats_fp64": 24 * C, "backward_sums_fp64": 8 * (2 * C + 1)}
        if not emulated:
            # context: a standalone NCCL all-reduce of the same messages (torch.distributed,
            # same process group, device-timed, max over ranks)
            import torch.distributed as dist
            sa = {}
            for name, n in (("forward_stats_fp64", 3 * C), ("backward_sums_fp64", 2 * C + 1)):
                buf = torch.zeros(n, dtype=torch.float64, device=dev)
                for _ in range(5):
                    dist.all_reduce(buf)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(50):
                    dist.all_reduce(buf)
                e1.record(st)
                torch.cuda.synchronize()
                sa[name] = round(pl.allmax([e0.elapsed_time(e1) / 50 * 1e3])[0], 2)
            out["nccl_standalone_us"] = sa
        return out

    def result(m):
        v = bytes_step_all / (m["ms_per_step"] * 1e-3) / 1e9
        return dict(value=round(v, 2), pct_of_peak=round(100 * v / (world * peak), 2),
                    ms_per_step=round(m["ms_per_step"], 4), fwd_ms=round(m["fwd_ms"], 4),
                    bwd_ms=round(m["bwd_ms"], 4))

    # ---- the timed step: one schedule at N = 1; at N > 1 the reduce / ncclAllReduce /
    # apply path first (the checker), then the fused-collective kernels if every rank's
    # preflight passed and they agree with it on this workload
    sync_paths, head_fl, head_name, note = {}, base_fl, "local", None
    if world == 1:
        head = measure(base_fl)
    else:
        nccl = measure(base_fl)
        sync_paths["nccl"] = dict(result(nccl), phases=phases(base_fl))
        head, head_name = nccl, "nccl"
        fused_ok, why = (False, "disabled (--sync nccl)") if args.sync == "nccl" else \
            (False, "ranks share one GPU (dry run)") if emulated else preflight_fused(args, pl)
        if fused_ok:
            fl_f = base_fl | L.SYNC_FUSED
            outs = []
            for fl in (base_fl, fl_f):
                z, _, sv = P.forward(x.clone(), g, bt, rm.clone(), rv.clone(), comm=comm, flags=fl)
                dx, _, _ = P.backward(z, dz.clone(), g, bt, sv, comm=comm, flags=fl)
                torch.cuda.synchronize()
                outs.append((z, dx))
            err = pl.allmax([max(chan_err(outs[1][0], outs[0][0]),
                                 chan_err(outs[1][1], outs[0][1]))])[0]
            del outs
            tol = 1e-2 if b == 2 else 1e-4
            fused = measure(fl_f)
            sync_paths["fused"] = dict(result(fused), phases=phases(fl_f),
                                       max_chan_err_vs_nccl=err, tol=tol)
            if err <= tol:
                head, head_fl, head_name = fused, fl_f, "fused"
            else:
                note = f"fused-collective path disagrees with the NCCL path ({err:.2e} > {tol})"
        else:
            sync_paths["fused"] = {"skipped": why}

    ms_per_step = head["ms_per_step"]
    value = bytes_step_all / (ms_per_step * 1e-3) / 1e9
    bwd_ms, fwd_ms = head["bwd_ms"], head["fwd_ms"]
    qfl = head_fl if (world == 1 or head_name == "fused") else L.FORCE_STREAMING
    dsc = L.desc(N_local, C, HW, L.BF16 if b == 2 else L.F32, L.NCHW)
    s_f, k_f = L.query_schedule(dsc, 0, qfl)
    s_b, k_b = L.query_schedule(dsc, 1, qfl)
    bwd_bytes = 3 * E * b
    achieved = bwd_bytes / (bwd_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config) if world == 1 else None

    # ---- strong scaling: t(1) of the whole global batch on one GPU (rank 0, non-sync path)
    strong = None
    if world > 1 and not emulated:
        t1 = [0.0]
        if rank == 0:
            xa = S.make_x(wl["N"], C, HW, 3000, dtype=wl["dtype"], device=dev)
            dza = S.make_dz(wl["N"], C, HW, 3000, dtype=wl["dtype"], device=dev)
            for _ in range(3):
                z, sm, sv = P.forward(xa, g, bt, rm, rv, flags=base_fl)
                P.backward(z, dza, g, bt, sv, flags=base_fl)
            a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K1 = max(5, min(args.steps, 50))
            a.record(st)
            for _ in range(K1):
                z, sm, sv = P.forward(xa, g, bt, rm, rv, flags=base_fl)
                P.backward(z, dza, g, bt, sv, flags=base_fl)
            c.record(st)
            torch.cuda.synchronize()
            t1 = [a.elapsed_time(c) / K1]
            del xa, dza
        t1 = pl.allmax(t1)[0]
        strong = {"t1_ms": round(t1, 4), "tG_ms": round(ms_per_step, 4), "G": world,
                  "t1_over_G_tG": round(t1 / (world * ms_per_step), 4),
                  "note": "SURVEY.md 8(d) item 3 diagnostic: t(1) = the whole global batch "
                          "on one GPU (rank 0), tG = this line's step time"}

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
            z, sm, sv = P.forward(xd, g, bt, rm, rv, comm=comm, flags=head_fl)
            f_done = ev()
            f_done.record(st)
            st.wait_event(dz_in)
            dx, dgam, dbet = P.backward(z, dzd, g, bt, sv, comm=comm, flags=head_fl)
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
        pl.barrier()
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s_in)
        for i in range(args.e2e_steps):
            e2e_step(i + 1)
        c.record(s_out)
        torch.cuda.synchronize()
        e2e_ms = pl.allmax([a.elapsed_time(c) / args.e2e_steps])[0]
        # PCIe alone, each direction on its own (same bytes, same pinned buffers)
        def copy_gbps(dst, src, reps=3):
            a_, c_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(st)
            for _ in range(reps):
                dst.copy_(src, non_blocking=True)
            c_.record(st)
            torch.cuda.synchronize()
            return reps * src.numel() * src.element_size() / (a_.elapsed_time(c_) * 1e-3) / 1e9
        h2d = copy_gbps(xs[1], xh)
        d2h = copy_gbps(zh, xs[1])
        e2e = {"value": round(bytes_step_all / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": 2 * E * b, "d2h_bytes_per_step": 2 * E * b + 2 * C * 4,
               "ms_per_step": round(e2e_ms, 3), "steps": args.e2e_steps,
               "pcie_h2d_GBps_alone": round(h2d, 2), "pcie_d2h_GBps_alone": round(d2h, 2),
               "pcie_per_direction_GBps_in_e2e": round(2 * E * b / (e2e_ms * 1e-3) / 1e9, 2),
               "host_numa": host_numa(dev),
               "path": "pinned host -> HBM (copy stream), iabn_forward + iabn_backward (C ABI), "
                       "HBM -> pinned host (copy stream); uploads of step i+1 overlap downloads "
                       "of step i"}
        del xs, dzs

    # ---- synchronized variant on one GPU: the fused-collective kernels over G virtual ranks
    sync_emu = None
    G = args.sync_emulated
    profiled = any(k in os.environ for k in ("NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                                             "NV_COMPUTE_PROFILER_PERFWORKS_DIR",
                                             "CUDA_INJECTION64_PATH"))
    if profiled and G > 1 and not os.environ.get("IABN_EMU_NONCOOP"):
        # Nsight Compute cannot launch the emulation's cooperative cluster kernels
        sync_emu = {"skipped": "profiler attached (cooperative cluster launch unsupported)"}
    elif world == 1 and G > 1 and wl["N"] % G == 0 and wl["layout"] == "NCHW":
        for _ in range(3):
            z, _, sv = P.forward_sync_emulated(x, G, g, bt, rm, rv)
            P.backward_sync_emulated(z, dz, G, g, bt, sv)
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

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s",
            "n_gpus": 1 if emulated else world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": wl["dtype"], "data": "synthetic",
            "config": {"workload": f"{args.config}: {wl['desc']}", "global_batch": wl["N"],
                       "N_local": N_local, "C": C, "HW": HW, "layout": wl["layout"],
                       "parallelism": f"dp{world}" + (f"+sync-stats({head_name})" if world > 1 else ""),
                       "l2": ("inputs larger than L2 (x, dz %.2f GB each)" % (E * b / 1e9))
                       if flush is None else "L2 flushed before every timed step",
                       "schedule": {"forward": SCHEDULES[s_f] + (f" K={k_f}" if s_f == 1 else ""),
                                    "backward": SCHEDULES[s_b] + (f" K={k_b}" if s_b == 1 else "")},
                       "algorithmic_bytes_per_step": bytes_step_all},
            # aggregate GB/s of all ranks over the aggregate peak of the GPUs used
            "pct_of_peak": round(100 * value / (world * peak), 2),
            "elements_per_s": round(E_all / (ms_per_step * 1e-3), 1),
            "effective_8Eb_GBps": round(8 * E_all * b / (ms_per_step * 1e-3) / 1e9, 2),
            "fwd_ms": round(fwd_ms, 4), "bwd_ms": round(bwd_ms, 4),
            "roofline": {"bound": "hbm", "kernel": "fused_bwd_kernel" if s_b else "backward pass",
                         "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "algorithmic_bytes_per_launch": bwd_bytes, "peak_source": peak_src,
                         "per_gpu": True,
                         "forward": {"kernel": "fused_fwd_kernel" if s_f else "forward pass",
                                     "achieved": round(2 * E * b / (fwd_ms * 1e-3) / 1e9, 2),
                                     "frac": round(2 * E * b / (fwd_ms * 1e-3) / 1e9 / peak, 4),
                                     "algorithmic_bytes_per_launch": 2 * E * b}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(head["launches"]),
            "clocks": head["clocks"],
        }
        if head["rejected"]:
            line["clocks_rejected_first_run"] = head["rejected"]
        if sync_paths:
            line["sync_paths"] = sync_paths
            line["headline_sync_path"] = head_name
        if note:
            line["note"] = note
        if strong:
            line["strong_scaling"] = strong
        if emulated:
            line["dry_run"] = (f"{world} ranks as threads on ONE GPU, library NCCL = the test "
                               "NCCL (tests/nccl_shim): validates the N > 1 code path, not a "
                               "scaling measurement")
        if sync_emu:
            line["sync_emulated"] = sync_emu
    if comm is not None:
        comm.close()
    return line


def host_numa(dev) -> dict:
    """NUMA node of the GPU's PCIe device and of this process's CPUs (e2e context)."""
    out = {}
    try:
        import torch
        pr = torch.cuda.get_device_properties(dev)
        bus = "%04x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
            out["gpu_numa_node"] = int(f.read().strip())
    except Exception:
        out["gpu_numa_node"] = None
    try:
        cpus = sorted(os.sched_getaffinity(0))
        nodes = set()
        import glob
        for d in glob.glob("/sys/devices/system/node/node*/cpulist"):
            node = int(d.split("node")[-1].split("/")[0])
            txt = open(d).read().strip()
            ids = set()
            for part in txt.split(","):
                if "-" in part:
                    lo, hi = part.split("-")
                    ids.update(range(int(lo), int(hi) + 1))
                elif part:
                    ids.add(int(part))
            if ids & set(cpus):
                nodes.add(node)
        out["process_cpu_numa_nodes"] = sorted(nodes)
    except Exception:
        out["process_cpu_numa_nodes"] = None
    return out


def main():
    args = parse()
    wl = WORKLOADS[args.config]
    if args.impl == "reference":
        return run_reference(args, wl)
    if args.preflight_fused:
        return preflight_child(args, wl)

    if args.emulate_ranks > 1:  # dry run of the N > 1 path on one GPU
        from tests import nccl_shim  # test infrastructure: the in-process NCCL
        os.environ["IABN_NCCL_LIB"] = nccl_shim.build()
        import torch
        import paper_1712_02616_b200 as P
        G = args.emulate_ranks
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        uid = P.Comm.unique_id()
        shared = {"barrier": threading.Barrier(G), "slots": [None] * G}
        lines, errs = [None] * G, []

        def th(r):
            try:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(torch.cuda.Stream()):
                    lines[r] = run_rank(args, wl, ThreadPlumb(r, G, dev, shared),
                                        lambda: P.Comm.create(G, r, uid), emulated=True)
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                shared["barrier"].abort()

        ts = [threading.Thread(target=th, args=(r,)) for r in range(G)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        print(json.dumps(lines[0]), flush=True)
        return

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
    line = run_rank(args, wl, DistPlumb(rank, world, dev), P.Comm.from_process_group,
                    emulated=False)
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
