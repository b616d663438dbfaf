"""The CPU oracle (test infrastructure) timed on the host cores over BASELINE.json's configs,
as a baseline only: cfg2 (ResNet-50 stage 3, whole), cfg3 and cfg5 (every ResNeXt-101 /
DenseNet-264 layer shape at N = 32, a bounded channel sample per shape, scaled to the
network's layer counts), cfg4 (WideResNet-38 crops, a channel sample) -- all threads and
one thread.  GB/s for the 5*E*b bytes of the layers (the GPU metric's accounting).

    python tools/cpu_baseline.py [--seconds-per-shape 0.3]
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: a reported baseline, not the product)
import synth_inputs as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seconds-per-shape", type=float, default=0.3)
args = ap.parse_args()
o = oracle.load()
gomp = ctypes.CDLL("libgomp.so.1")
nthreads = gomp.omp_get_max_threads()


def sample(N, C, HW, ch, dtype):
    x = S.make_x(N, ch, HW, 0, dtype=dtype).double().numpy()
    dz = S.make_dz(N, ch, HW, 0, dtype=dtype).double().numpy()
    p = S.make_params(ch, 0)
    return x, dz, p.gamma.double().numpy(), p.beta.double().numpy()


def time_shape(N, C, HW, dtype, budget):
    """seconds per element of one forward + stored-x backward, on a channel sample"""
    ch = max(1, min(C, int(2e6 // (N * HW)) or 1))
    x, dz, g, b = sample(N, C, HW, ch, dtype)
    o.forward(x, g, b)
    o.backward_standard(x, dz, g, b)
    t0, n = time.perf_counter(), 0
    while n < 2 or time.perf_counter() - t0 < budget:
        o.forward(x, g, b)
        o.backward_standard(x, dz, g, b)
        n += 1
    return (time.perf_counter() - t0) / n / (N * ch * HW)


def network(layers, dtype, budget):
    b = 2 if dtype == "bf16" else 4
    shapes = {}
    for c, hw in layers:
        shapes[(c, hw)] = shapes.get((c, hw), 0) + 1
    t_tot, e_tot = 0.0, 0
    for (c, hw), n in shapes.items():
        spe = time_shape(32, c, hw, dtype, budget)
        t_tot += n * spe * 32 * c * hw
        e_tot += n * 32 * c * hw
    return {"GBps": round(5 * e_tot * b / t_tot / 1e9, 4), "seconds_per_pass_pair": round(t_tot, 3),
            "layers": len(layers), "shapes": len(shapes)}


res = {"cpu_model": None, "threads_all": nthreads}
try:
    res["cpu_model"] = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                            if l.startswith("model name"))
except Exception:
    pass
for label, threads in (("all_threads", nthreads), ("one_thread", 1)):
    gomp.omp_set_num_threads(threads)
    bud = args.seconds_per_shape if threads > 1 else args.seconds_per_shape / 2
    r = {}
    spe = time_shape(64, 1024, 196, "f32", bud)
    r["cfg2_r50s3_f32"] = round(5 * 4 / spe / 1e9, 4)
    spe = time_shape(16, 4096, 12544, "bf16", bud)
    r["cfg4_wrn38_bf16"] = round(5 * 2 / spe / 1e9, 4)
    for net, layers in (("cfg3_rx101", S.rx101_layers()), ("cfg5_densenet264", S.densenet264_layers())):
        for dt in ("f32", "bf16"):
            r[f"{net}_{dt}"] = network(layers, dt, bud)
    res[label] = r
    print(label, json.dumps(r), flush=True)
gomp.omp_set_num_threads(nthreads)
print(json.dumps(res))
