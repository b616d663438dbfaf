// iabn.cu -- host side of the C ABI declared in include/iabn.h.
//
// Validation (synchronous, before any launch), schedule selection
// (channel-resident cluster kernels when the per-channel slab fits in the
// shared memory of a <=16-CTA cluster, else the streaming kernels), launches on
// the caller's stream, and the NCCL exchange of the synchronized variant
// (libnccl.so.2 loaded with dlopen, so the library loads without NCCL/GPU).
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <numeric>
#include <utility>
#include <vector>
#include <string>

#include "iabn.h"
#include "kernels_act.cuh"
#include "kernels_gres.cuh"
#include "kernels_fused.cuh"
#include "kernels_nhwc.cuh"
#include "kernels_nhwc_bulk.cuh"
#include "kernels_small.cuh"
#include "kernels_stream.cuh"

using namespace iabn;

// ====================================================================== status / errors
namespace {

thread_local std::string g_err;
unsigned long long* g_trace = nullptr;  // debug trace of the last fused launch
size_t g_trace_n = 0;
uint32_t g_trace_ch = 0;
std::atomic<uint64_t> g_launches{0};

iabn_status fail(iabn_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

iabn_status check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(IABN_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return IABN_OK;
}

#define IABN_TRY(expr)                        \
    do {                                      \
        const iabn_status _s = (expr);        \
        if (_s != IABN_OK) return _s;         \
    } while (0)

// ====================================================================== device facts
struct DevFacts {
    int sms = 0;
    int max_smem_optin = 0;
    bool attrs_set = false;
};
constexpr int kMaxDev = 64;
DevFacts g_dev[kMaxDev];
std::mutex g_dev_mu;

iabn_status device_facts(DevFacts** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(IABN_ERR_CUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
    if (dev < 0 || dev >= kMaxDev) return fail(IABN_ERR_CUDA, "device ordinal %d too large", dev);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    DevFacts& f = g_dev[dev];
    if (f.sms == 0) {
        cudaDeviceGetAttribute(&f.sms, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&f.max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        if (f.sms <= 0) return fail(IABN_ERR_CUDA, "no usable CUDA device");
    }
    if (!f.attrs_set) {
        const int dyn = f.max_smem_optin - 4096;  // leave room for static smem
        const void* fns[] = {(const void*)fused_kernel<float, 0, 2>,
                             (const void*)fused_kernel<__nv_bfloat16, 0, 2>,
                             (const void*)fused_kernel<float, 1, 2>,
                             (const void*)fused_kernel<__nv_bfloat16, 1, 2>,
                             (const void*)fused_kernel<float, 0, 4>,
                             (const void*)fused_kernel<__nv_bfloat16, 0, 4>,
                             (const void*)fused_kernel<float, 1, 4>,
                             (const void*)fused_kernel<__nv_bfloat16, 1, 4>,
                             (const void*)fused_kernel<float, 0, 2, true>,
                             (const void*)fused_kernel<__nv_bfloat16, 0, 2, true>,
                             (const void*)fused_kernel<float, 1, 2, true>,
                             (const void*)fused_kernel<__nv_bfloat16, 1, 2, true>,
                             (const void*)fused_kernel<float, 0, 4, true>,
                             (const void*)fused_kernel<__nv_bfloat16, 0, 4, true>,
                             (const void*)fused_kernel<float, 1, 4, true>,
                             (const void*)fused_kernel<__nv_bfloat16, 1, 4, true>};
        for (const void* fn : fns) {
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        const void* act[] = {(const void*)fused_kernel<float, 0, 2, false, 1>, (const void*)fused_kernel<float, 1, 2, false, 1>,
                             (const void*)fused_kernel<float, 0, 4, false, 1>, (const void*)fused_kernel<float, 1, 4, false, 1>,
                             (const void*)fused_kernel<float, 0, 2, true, 1>, (const void*)fused_kernel<float, 1, 2, true, 1>,
                             (const void*)fused_kernel<float, 0, 4, true, 1>, (const void*)fused_kernel<float, 1, 4, true, 1>,
                             (const void*)fused_kernel<float, 0, 2, false, 2>, (const void*)fused_kernel<float, 1, 2, false, 2>,
                             (const void*)fused_kernel<float, 0, 4, false, 2>, (const void*)fused_kernel<float, 1, 4, false, 2>,
                             (const void*)fused_kernel<float, 0, 2, true, 2>, (const void*)fused_kernel<float, 1, 2, true, 2>,
                             (const void*)fused_kernel<float, 0, 4, true, 2>, (const void*)fused_kernel<float, 1, 4, true, 2>};
        for (const void* fn : act) {  // BN + sigmoid / tanh in the channel-resident kernels
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        }
        const void* nhwc[] = {(const void*)nhwc_fused_kernel<float, 0>,
                              (const void*)nhwc_fused_kernel<__nv_bfloat16, 0>,
                              (const void*)nhwc_fused_kernel<float, 1>,
                              (const void*)nhwc_fused_kernel<__nv_bfloat16, 1>};
        for (const void* fn : nhwc) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        const void* nhwc_act[] = {(const void*)nhwc_fused_kernel<float, 0, 1>, (const void*)nhwc_fused_kernel<float, 1, 1>,
                                  (const void*)nhwc_fused_kernel<float, 0, 2>, (const void*)nhwc_fused_kernel<float, 1, 2>};
        for (const void* fn : nhwc_act) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        const void* nb[] = {(const void*)nhwc_bulk_reduce_kernel<float, 0, false>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, false>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, true>,
                            (const void*)nhwc_bulk_reduce_kernel<__nv_bfloat16, 0, false>,
                            (const void*)nhwc_bulk_reduce_kernel<__nv_bfloat16, 1, false>,
                            (const void*)nhwc_bulk_reduce_kernel<__nv_bfloat16, 1, true>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, false, 1>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, true, 1>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, false, 2>,
                            (const void*)nhwc_bulk_reduce_kernel<float, 1, true, 2>};
        for (const void* fn : nb) {
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kNbSmem);
            cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        }
        const void* gres[] = {(const void*)gres_kernel<float, 0>,
                              (const void*)gres_kernel<__nv_bfloat16, 0>,
                              (const void*)gres_kernel<float, 1>,
                              (const void*)gres_kernel<__nv_bfloat16, 1>};
        for (const void* fn : gres) {  // static shared memory of these is ~4.2 KB
            cudaFuncAttributes fa = {};
            cudaFuncGetAttributes(&fa, fn);
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 f.max_smem_optin - (int)fa.sharedSizeBytes);
        }
        e = cudaGetLastError();
        if (e != cudaSuccess)
            return fail(IABN_ERR_CUDA, "kernel attribute setup: %s", cudaGetErrorString(e));
        f.attrs_set = true;
    }
    *out = &f;
    return IABN_OK;
}

// ====================================================================== geometry
struct Geom {
    int64_t N, C, HW, m, E;
    int dtype, layout, b;
};

iabn_status make_geom(const iabn_desc* d, Geom* g) {
    if (!d) return fail(IABN_ERR_INVALID_ARG, "desc is NULL");
    if (d->n <= 0 || d->c <= 0 || d->hw <= 0)
        return fail(IABN_ERR_INVALID_ARG, "empty input: n=%lld c=%lld hw=%lld", (long long)d->n,
                    (long long)d->c, (long long)d->hw);
    if (d->dtype != IABN_F32 && d->dtype != IABN_BF16)
        return fail(IABN_ERR_UNSUPPORTED, "unknown dtype %d", d->dtype);
    if (d->layout != IABN_NCHW && d->layout != IABN_NHWC)
        return fail(IABN_ERR_UNSUPPORTED, "unknown layout %d", d->layout);
    g->N = d->n;
    g->C = d->c;
    g->HW = d->hw;
    if (g->N > (1ll << 31) / g->HW)
        return fail(IABN_ERR_UNSUPPORTED, "n*hw = %lld values per channel exceeds 2^31",
                    (long long)(g->N * g->HW));
    g->m = g->N * g->HW;
    if (g->C > (1ll << 31) / g->HW)
        return fail(IABN_ERR_UNSUPPORTED, "c*hw exceeds 2^31 (one sample too large)");
    if (g->C > (1ll << 40) / g->m) return fail(IABN_ERR_UNSUPPORTED, "tensor too large");
    g->E = g->m * g->C;
    g->dtype = d->dtype;
    g->layout = d->layout;
    g->b = d->dtype == IABN_F32 ? 4 : 2;
    return IABN_OK;
}

bool vec_ok(const Geom& g) {
    return g.layout == IABN_NCHW ? (g.HW * g.b) % 16 == 0 : (g.C * g.b) % 16 == 0;
}

// Split count of the streaming reductions: independent of the device so that
// workspace sizes and reduction trees (hence results) are fixed per shape.
#ifndef IABN_TARGET_WAVES
#define IABN_TARGET_WAVES 1
#endif
constexpr int64_t kTargetCtas = 148 * 8 * IABN_TARGET_WAVES;
// NHWC streaming reductions through the bulk ring (kernels_nhwc_bulk.cuh): 16-byte rows
// of <= 512 vectors; CTAs own whole row ranges, at most 2 per SM of a 148-SM B200 (a
// device constant: workspace sizes must not depend on the device), at least one 16 KB
// stage each.  0 = not applicable.
int env_int(const char* name, int dflt);
int nb_grid(const Geom& g) {
    if (g.layout != IABN_NHWC || !vec_ok(g) || env_int("IABN_NHWC_BULK", 1) == 0) return 0;
    if (g.C * g.b > 4096) return 0;  // <= 256 vectors per row
    const int64_t bytes = g.m * g.C * g.b;  // one input
    // 32 clusters of 8: resident at once (2 CTAs per SM; cudaOccupancyMaxActiveClusters
    // reports 33 on a 148-SM B200 -- 37 clusters ran a second wave of 4)
    int64_t G = std::min<int64_t>(256, bytes / kNbStageBytes);
    G = std::min<int64_t>(G, g.m) / kNbCluster * kNbCluster;  // whole clusters
    return (int)(G / kNbCluster);  // records: one per cluster
}

int stat_splits_ldg(const Geom& g);
int stat_splits(const Geom& g) {
    if (const int G = nb_grid(g)) return G;
    return stat_splits_ldg(g);
}
// splits of the LDG reduction kernels (the workspace holds max(S, 296) NHWC records)
int stat_splits_ldg(const Geom& g) {
    const int64_t target = kTargetCtas;
    int64_t units, per_unit_min, work;
    if (g.layout == IABN_NCHW) {
        units = g.C;
        work = g.m;
        per_unit_min = 4096;
    } else {
        const int64_t V = vec_ok(g) ? 16 / g.b : 1;
        units = (g.C + 16 * V - 1) / (16 * V);
        work = g.m;  // rows
        per_unit_min = 16 * 16;
    }
    int64_t S = (target + units - 1) / units;
    S = std::min<int64_t>(S, std::max<int64_t>(1, work / per_unit_min));
    // small NHWC layers: at least one CTA per SM when the rows allow >= 32 each (the
    // reduction is a chain of load latencies per CTA; measured on DenseNet-264 NHWC)
    if (g.layout == IABN_NHWC && units * S < 148)
        S = std::max<int64_t>(S, std::min<int64_t>((148 + units - 1) / units, work / 32));
    S = std::max<int64_t>(1, std::min<int64_t>(S, 65535));
    return (int)S;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct WsLayout {
    size_t part, stats, sums_loc, sums_glob, coef, bar, total;
};
// grid-resident NHWC schedule: at most this many CTAs (2 per SM of a 148-SM B200; a
// device constant so that workspace sizes do not depend on the device)
constexpr int64_t kGresMaxG = 296;

WsLayout ws_layout(const Geom& g, int S) {
    WsLayout w;
    size_t off = 0;
    w.part = off;
    const int64_t rec = g.layout == IABN_NHWC ? std::max<int64_t>(S, kGresMaxG) : S;
    off += align256((size_t)rec * g.C * 3 * sizeof(double));
    w.stats = off;
    off += align256((size_t)g.C * 3 * sizeof(double));
    w.sums_loc = off;
    off += align256((size_t)(2 * g.C + 1) * sizeof(double));
    w.sums_glob = off;
    off += align256((size_t)(2 * g.C + 1) * sizeof(double));
    w.coef = off;
    off += align256((size_t)g.C * sizeof(float4));
    w.bar = off;  // grid-barrier counter of the one-launch schedule
    off += 256;
    w.total = off;
    return w;
}

// ====================================================================== argument checks
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

iabn_status check_scalars(float eps, float slope) {
    if (!(eps > 0.f) || !std::isfinite(eps))
        return fail(IABN_ERR_INVALID_ARG, "eps must be finite and > 0 (got %g)", (double)eps);
    if (!(slope > 0.f && slope <= 1.f))
        return fail(IABN_ERR_INVALID_ARG, "slope must be in (0, 1] (got %g)", (double)slope);
    return IABN_OK;
}

iabn_status check_momentum(float momentum) {
    if (!(momentum >= 0.f && momentum <= 1.f))
        return fail(IABN_ERR_INVALID_ARG, "momentum must be in [0, 1] (got %g)", (double)momentum);
    return IABN_OK;
}

iabn_status check_act(const char* name, const void* p) {
    if (!p) return fail(IABN_ERR_INVALID_ARG, "%s is NULL", name);
    if (!aligned16(p))
        return fail(IABN_ERR_UNSUPPORTED, "%s is not 16-byte aligned", name);
    return IABN_OK;
}

// a and b must be equal or disjoint ranges of `bytes`
iabn_status check_same_or_disjoint(const char* an, const void* a, const char* bn, const void* b,
                                   size_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    if (x == y) return IABN_OK;
    if (x < y + bytes && y < x + bytes)
        return fail(IABN_ERR_ALIAS, "%s and %s partially overlap", an, bn);
    return IABN_OK;
}
iabn_status check_disjoint(const char* an, const void* a, const char* bn, const void* b,
                           size_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    if (x < y + bytes && y < x + bytes) return fail(IABN_ERR_ALIAS, "%s and %s overlap", an, bn);
    return IABN_OK;
}

iabn_status check_ws(const Geom& g, void* ws, size_t ws_bytes, const WsLayout& w) {
    if (!ws) return fail(IABN_ERR_WORKSPACE, "workspace is NULL");
    if (!aligned16(ws)) return fail(IABN_ERR_WORKSPACE, "workspace not 16-byte aligned");
    if (ws_bytes < w.total)
        return fail(IABN_ERR_WORKSPACE, "workspace %zu bytes < required %zu", ws_bytes, w.total);
    (void)g;
    return IABN_OK;
}

// ====================================================================== fused planning
// Experiment overrides (IABN_*), read once per process: no getenv on the hot path.
int env_int(const char* name, int dflt) {
    struct Entry {
        const char* name;
        bool set;
        int val;
    };
    static std::mutex mu;
    static Entry cache[32];
    static int n = 0;
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n; ++i)
        if (cache[i].name == name || strcmp(cache[i].name, name) == 0)
            return cache[i].set ? cache[i].val : dflt;
    const char* s = getenv(name);
    if (n < 32) cache[n++] = Entry{name, s != nullptr, s ? atoi(s) : 0};
    return s ? atoi(s) : dflt;
}

// Kernel launch with programmatic stream serialisation (PDL): the kernel may be
// scheduled while the previous kernel on the stream drains; it waits in pdl_wait()
// before touching global memory.  IABN_PDL=0 launches plainly (experiments).
bool pdl_enabled() {
    static const bool on = env_int("IABN_PDL", 1) != 0;
    return on;
}
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);  // errors: check_launch
}

// Shared-memory budget per CTA for the slab ring: ~100 KB keeps two CTAs per SM.
size_t fused_budget_bytes() {
    static const size_t budget = (size_t)std::max(8, env_int("IABN_FUSED_SMEM_KB", 100)) * 1024;
    return budget;
}


struct FusedPlan {
    bool ok = false;
    int K = 0;           // CTAs per cluster (per channel)
    int clusters = 0;    // persistent clusters in the grid
    int max_clusters = 0;  // clusters that can be co-resident
    uint32_t cap = 0;    // vectors per input per buffer
    uint32_t chunk_vecs = 0;
    int nbuf = 0;
    size_t smem = 0;
    int minb = 2;        // kernel variant: CTAs per SM its registers allow (2 or 4)
    bool mis = false;    // planes not 16-byte aligned: covering-range kernels
    uint32_t mis_w = 0;  // 16-byte slots per plane (MIS)
};

template <bool MIS>
const void* fused_fn_t(int pass, int dtype, int minb) {
    if (minb == 4) {
        if (pass == 0)
            return dtype == IABN_F32 ? (const void*)fused_kernel<float, 0, 4, MIS>
                                     : (const void*)fused_kernel<__nv_bfloat16, 0, 4, MIS>;
        return dtype == IABN_F32 ? (const void*)fused_kernel<float, 1, 4, MIS>
                                 : (const void*)fused_kernel<__nv_bfloat16, 1, 4, MIS>;
    }
    if (pass == 0)
        return dtype == IABN_F32 ? (const void*)fused_kernel<float, 0, 2, MIS>
                                 : (const void*)fused_kernel<__nv_bfloat16, 0, 2, MIS>;
    return dtype == IABN_F32 ? (const void*)fused_kernel<float, 1, 2, MIS>
                             : (const void*)fused_kernel<__nv_bfloat16, 1, 2, MIS>;
}
const void* fused_fn(int pass, int dtype, int minb, bool mis) {
    return mis ? fused_fn_t<true>(pass, dtype, minb) : fused_fn_t<false>(pass, dtype, minb);
}

// Co-resident clusters of K CTAs with `smem` bytes of dynamic shared memory (cached).
int max_active_clusters(int pass, int dtype, int K, size_t smem, int minb, bool mis) {
    static std::mutex mu;
    struct Key {
        int dev, pass, dtype, K;
        size_t smem;
        int minb;
        bool mis;
        int val;
    };
    static Key cache[512];
    static int ncache = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < ncache; ++i)
        if (cache[i].dev == dev && cache[i].pass == pass && cache[i].dtype == dtype &&
            cache[i].K == K && cache[i].smem == smem && cache[i].minb == minb &&
            cache[i].mis == mis)
            return cache[i].val;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)K, 1, 1);
    cfg.blockDim = dim3(kFusedThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fused_fn(pass, dtype, minb, mis), &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (ncache < 512) cache[ncache++] = Key{dev, pass, dtype, K, smem, minb, mis, n};
    return n;
}

// Choose (K, nbuf): a slice of ceil(mv/K) vectors per CTA, nbuf slab buffers.
// Measured on B200 (profiles/): two ~100 KB CTAs per SM
// beat one ~200 KB CTA (two independent pipelines hide each other's serial
// phases), double buffering beats single when the slice allows it, and clusters
// of <= 8 CTAs pack the GPCs far better than 16.  So: the smallest K whose slice
// double-buffers in the per-CTA budget; else (large channels) the smallest K
// whose slice fits once.
FusedPlan fused_plan(const Geom& g, int pass, const DevFacts& f, uint32_t flags) {
    FusedPlan best;
    if (g.layout != IABN_NCHW) return best;
    // planes not 16-byte aligned: each plane is held as the W aligned 16-byte slots that
    // cover it (bulk copies need 16-byte alignment); needs whole planes per CTA and a
    // tensor whose byte size is a multiple of 16 (the last plane's covering range)
    // (faster than the streaming kernels on the misaligned layers of cfg3/cfg5: bf16
    // 14x14 and 7x7, fp32 7x7 -- whole-network sweeps 8-13 %; env IABN_FUSED_MIS=0 off)
    const bool mis = (g.HW * g.b) % 16 != 0;
    if (mis && ((g.E * g.b) % 16 != 0 ||
                (!(flags & IABN_FORCE_FUSED) && env_int("IABN_FUSED_MIS", 1) == 0)))
        return best;
    const int64_t W = (g.HW * g.b + 15) / 16 + 1;
    const int nin = pass == 0 ? 1 : 2;
    const int64_t mv = mis ? g.N * W : g.m * g.b / 16;
    const size_t cap_bytes = (size_t)f.max_smem_optin - 4096;
    const size_t budget = std::min<size_t>(fused_budget_bytes(), cap_bytes);
    const int kforce = env_int("IABN_FUSED_K", 0);
    const int nforce = env_int("IABN_FUSED_NBUF", 0);
    const int64_t pv = mis ? W : g.HW * g.b / 16;  // vectors (slots) per plane
    const int64_t np = g.N;
    int minb = 2;
    size_t lim = budget;
    auto consider = [&](int K, int nbuf) -> bool {
        // slice: whole planes when N >= K (see cta_slice)
        const bool by_plane = np >= K;
        if (mis && !by_plane) return false;
        // the small-slab variant only with whole planes per CTA: a plane split across CTAs
        // (sub-plane chunks, cursor-addressed apply) loses to the 2-CTA/SM variant with
        // whole planes (fused-collective sync at 2 planes per rank: bwd 1.16 -> 0.97 ms)
        if (minb == 4 && !by_plane) return false;
        const int64_t cap = by_plane ? pv * ((np + K - 1) / K) : (mv + K - 1) / K;
        const size_t bytes = (size_t)cap * 16 * nin * nbuf;
        if (bytes > lim) return false;
        const int cl = max_active_clusters(pass, g.dtype, K, bytes, minb, mis);
        if (cl <= 0) return false;
        best.ok = true;
        best.minb = minb;
        best.K = K;
        best.clusters = (int)std::min<int64_t>(cl, g.C);
        best.max_clusters = cl;
        best.cap = (uint32_t)cap;
        best.nbuf = nbuf;
        best.smem = bytes;
        // chunks: large bulk copies keep the TMA engines efficient (measured: >= 16 KB
        // per input best); whole planes when planes are that large; <= kMaxChunks
        const int64_t env = env_int("IABN_FUSED_CHUNK", 0);
        int64_t cv;
        if (env > 0) {
            cv = env;
        } else if (by_plane) {
            const int64_t per = std::max<int64_t>(1, (1024 + pv - 1) / pv);  // planes per chunk
            cv = pv * per;
        } else {
            cv = 2048 / nin;
        }
        cv = std::max<int64_t>(cv, (cap + kMaxChunks - 1) / kMaxChunks);
        if (mis) cv = (cv + pv - 1) / pv * pv;  // whole planes
        best.chunk_vecs = (uint32_t)std::min<int64_t>(cv, cap);
        best.mis = mis;
        best.mis_w = (uint32_t)W;
        return true;
    };
    {
        // small slabs first: the 4-CTA/SM variant with ~50 KB double-buffered slabs
        // (small layers: more resident pipelines; measured r50s3 52 -> 57 %), else
        // the 2-CTA/SM variant with ~100 KB slabs (large channels, e.g. cfg4)
        const int mforce = env_int("IABN_FUSED_MINB", 0);
        const size_t small = std::min<size_t>(
            (size_t)std::max(8, env_int("IABN_FUSED_SMALL_KB", 50)) * 1024, budget);
        if (kforce || nforce) {
            minb = mforce == 4 ? 4 : 2;
            lim = minb == 4 ? small : budget;
            for (int K = kforce ? kforce : 1; K <= (kforce ? kforce : kMaxCluster) && K <= mv; ++K)
                for (int nb = nforce ? nforce : kMaxBuf; nb >= (nforce ? nforce : 1); --nb)
                    if (consider(K, nb)) goto done;
            goto done;
        }
        if (mforce != 2) {
            minb = 4;
            lim = small;
            for (int K = 1; K <= 8 && K <= mv; ++K)
                if (consider(K, 2)) goto done;
        }
        if (mforce == 4) goto done;
        minb = 2;
        lim = budget;
        for (int K = 1; K <= 8 && K <= mv; ++K)
            if (consider(K, 2)) goto done;
        for (int K = 1; K <= kMaxCluster && K <= mv; ++K)
            if (consider(K, 1)) goto done;
    }
done:
    // small slabs: more of them in flight per CTA when they fit in the same budget (the
    // per-channel latency -- load, record exchange, coefficients -- is then hidden by more
    // channels in flight rather than by bigger ones)
    if (best.ok && best.nbuf == 2 && !env_int("IABN_FUSED_NBUF", 0) &&
        env_int("IABN_FUSED_DEEP", 1)) {
        const FusedPlan keep = best;
        const int K = best.K;
        int nb = kMaxBuf;
        for (; nb > 2; --nb)
            if (consider(K, nb) && best.clusters == keep.clusters) break;
        if (nb == 2) best = keep;
    }
    if (best.ok && env_int("IABN_VERBOSE", 0)) {
        static std::mutex pm;
        static int printed = 0;
        std::lock_guard<std::mutex> lk(pm);
        if (printed++ < 16)
            fprintf(stderr, "[iabn] fused pass=%d C=%lld m=%lld: K=%d nbuf=%d minb=%d clusters=%d smem=%zu cap=%u chunk=%u\n",
                    pass, (long long)g.C, (long long)g.m, best.K, best.nbuf, best.minb, best.clusters,
                    best.smem, best.cap, best.chunk_vecs);
    }
    return best;
}

FastDiv fd32(int64_t d) { return make_fastdiv((uint32_t)d); }

// a.vranks > 1 (one-GPU emulation of the synchronized variant): clusters of different
// virtual ranks wait on one another, so the grid is launched cooperatively (co-resident)
std::atomic<int> g_last_dyn{0};  // test hook: did the last fused launch schedule dynamically

// Counters of the dynamic channel scheduling, one pair per (device, stream): zeroed
// once (stream-ordered), re-armed by each launch's last cluster.  nullptr (static
// scheduling) when the first use on a stream is inside a CUDA-graph capture.
unsigned int* dyn_counters(cudaStream_t st) {
    struct Ent {
        int dev;
        cudaStream_t st;
        unsigned int* p;
    };
    static std::mutex mu;
    static std::vector<Ent> ents;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    for (const Ent& e : ents)
        if (e.dev == dev && e.st == st) return e.p;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
    }
    unsigned int* p = nullptr;  // [kMaxRanks][2]: one pair per (virtual) rank
    if (cudaMalloc(&p, 2 * kMaxRanks * sizeof(unsigned int)) != cudaSuccess ||
        cudaMemsetAsync(p, 0, 2 * kMaxRanks * sizeof(unsigned int), st) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    ents.push_back(Ent{dev, st, p});
    return p;
}

template <typename T, int ACT = 0>
iabn_status launch_fused(int pass, const FusedPlan& p, FusedArgs a, cudaStream_t st) {
    a.dyn = nullptr;
    if (a.qv == 0) {  // plain call: one rank, no exchange
        a.qv = (uint32_t)p.clusters;
        a.vranks = 1;
        a.nranks = 1;
        // dynamic channel scheduling for large slices (the sync variants keep the static
        // order: every rank must process the channels in the same order).  Measured on B200:
        // WideResNet-38 (50-100 KB slices) fwd 0.530 -> 0.491 ms, bwd 0.848 -> 0.799 ms;
        // small slices (ResNet-50 stage 3, <= 25 KB) lose ~5 % to the ticket round trip, so
        // they keep the static order.  Env IABN_FUSED_DYN=0 off, 2 = also small slices.
        const int dyn = env_int("IABN_FUSED_DYN", 1);
        const size_t slice = (size_t)p.cap * 16u * (pass == 0 ? 1u : 2u);
        if (dyn && p.minb == 2 && (int64_t)p.clusters < a.C && (slice >= 32768 || dyn == 2))
            a.dyn = dyn_counters(st);
    } else {
        // synchronized variant, opt-in (env IABN_SYNC_DYN=1): each rank draws its channels
        // from its own counter in increasing order, which keeps the cross-rank waits
        // deadlock-free (the smallest channel not yet finished everywhere has been drawn and
        // published by every rank).  Measured slower than the static
        // order at G >= 2 (WideResNet-38 emulated G = 2/4/8: 86.5/86.8/84.3 -> 83.7/80.5/
        // 75.2 %): with identical static orders the ranks reach a channel at about the same
        // time; with per-rank dynamic orders a channel's records wait for the slowest rank's
        // cluster that happens to draw it.
        // (one rank -- the G = 1 emulation -- has no cross-rank waits: dynamic as above)
        const int dyn = a.nranks <= 1 ? env_int("IABN_FUSED_DYN", 1) : env_int("IABN_SYNC_DYN", 0);
        const size_t slice = (size_t)p.cap * 16u * (pass == 0 ? 1u : 2u);
        if (dyn && p.minb == 2 && (int64_t)a.qv < a.C && (slice >= 32768 || dyn == 2))
            a.dyn = dyn_counters(st);
    }
    g_last_dyn.store(a.dyn != nullptr ? 1 : 0);
    a.cap = p.cap;
    a.chunk_vecs = p.chunk_vecs;
    a.nbuf = (uint32_t)p.nbuf;
    // single-buffered slices (the backward of large channels): the refill waits for the
    // apply, so the slice is prefetched into L2 first (cfg4 backward 0.90 -> 0.85 ms).
    // Double-buffered slices of large planes (>= 16 KB: one prefetch per plane) too: the
    // fused-collective sync over 2-8 ranks on cfg4 (one plane per CTA) 77-79 -> 82-85 %
    // of peak; small planes (r50s3, 14x14 bf16) measured slower with it (tools/gpu_exp122.sh)
    {
        const int pf = env_int("IABN_FUSED_PREFETCH", -1);  // -1 auto, 0 off, 1 on, 2 bwd only
        const bool big_planes = a.HW * (int64_t)sizeof(T) >= 16384;
        a.prefetch = pf < 0    ? (p.nbuf == 1 || big_planes ? 1u : 0u)
                     : pf == 2 ? (uint32_t)(pass == 1)
                               : (uint32_t)pf;
        // L2 cache hints: bit 1 = the prefetch marks its lines evict_last (they must survive
        // until the refill), bit 2 = the refill copies mark them evict_first (used once);
        // measured: backward 0.848 -> 0.834 ms, DRAM reads 3.45 -> 3.32 GB (3.29 GB minimum)
        if (a.prefetch) a.prefetch |= (uint32_t)env_int("IABN_FUSED_PF_HINT", 3) << 1;
        // experiments: bit 3 = every bulk copy of the slices evict_first
        a.prefetch |= (uint32_t)env_int("IABN_FUSED_LOAD_EVICT_FIRST", 0) << 3;
    }
    a.debug = (uint32_t)env_int("IABN_FUSED_DEBUG", 0);
    a.trace = nullptr;
    a.trace_ch = 0;
    if (a.debug & 4u) {  // experiments only: phase timestamps, dumped by iabn_debug_trace
        static unsigned long long* buf = nullptr;
        static size_t cap = 0;
        const uint32_t per = (uint32_t)((a.C + a.qv - 1) / a.qv);
        const size_t need = (size_t)a.vranks * a.qv * p.K * per * kTraceFields;
        if (need > cap) {
            if (buf) cudaFree(buf);
            cudaMalloc(&buf, need * sizeof(unsigned long long));
            cap = need;
        }
        cudaMemsetAsync(buf, 0, need * sizeof(unsigned long long), st);
        a.trace = buf;
        a.trace_ch = per;
        g_trace = buf;
        g_trace_n = need;
        g_trace_ch = per;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.vranks * a.qv * (unsigned)p.K, 1, 1);
    cfg.blockDim = dim3(kFusedThreads, 1, 1);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[3];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = p.K;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    // IABN_EMU_NONCOOP=1 (experiments only): a plain launch of the emulation -- Nsight
    // Compute cannot launch a cooperative cluster kernel ("LaunchFailed"); under its
    // kernel replay the grid (<= the co-resident clusters) runs alone, so it is resident
    if (a.vranks > 1 && !env_int("IABN_EMU_NONCOOP", 0)) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na].val.cooperative = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    cudaError_t e;
    a.mis_w = p.mis_w;
    a.hwb = (uint32_t)(a.HW * (int64_t)sizeof(T));
    a.fd_w = fd32(p.mis ? p.mis_w : 1);
    if (p.mis) {
        if (p.minb == 4)
            e = pass == 0 ? cudaLaunchKernelEx(&cfg, fused_kernel<T, 0, 4, true, ACT>, a)
                          : cudaLaunchKernelEx(&cfg, fused_kernel<T, 1, 4, true, ACT>, a);
        else
            e = pass == 0 ? cudaLaunchKernelEx(&cfg, fused_kernel<T, 0, 2, true, ACT>, a)
                          : cudaLaunchKernelEx(&cfg, fused_kernel<T, 1, 2, true, ACT>, a);
    } else if (p.minb == 4) {
        e = pass == 0 ? cudaLaunchKernelEx(&cfg, fused_kernel<T, 0, 4, false, ACT>, a)
                      : cudaLaunchKernelEx(&cfg, fused_kernel<T, 1, 4, false, ACT>, a);
    } else {
        e = pass == 0 ? cudaLaunchKernelEx(&cfg, fused_kernel<T, 0, 2, false, ACT>, a)
                      : cudaLaunchKernelEx(&cfg, fused_kernel<T, 1, 2, false, ACT>, a);
    }
    if (e != cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return fail(IABN_ERR_CUDA, "fused launch: %s", cudaGetErrorString(e));
    }
    return check_launch(pass == 0 ? "fused_kernel<fwd>" : "fused_kernel<bwd>");
}

// ====================================================================== NHWC channel groups
// kernels_nhwc.cuh: a cluster of K CTAs holds the g-channel column group of all rows in
// shared memory (2-D TMA boxes), reduces, exchanges over DSMEM and applies in place.
struct NhwcPlan {
    bool ok = false;
    uint32_t g = 0, cols = 0, K = 0, rows_cta = 0, box_rows = 0, ngroups = 0;
    uint32_t slab = 0, red_off = 0, rec_off = 0, coef_off = 0, bar_off = 0;
    size_t smem = 0;
    int clusters = 0;  // launched (persistent over ngroups)
    double est_us = 0;
};

int nhwc_max_clusters(int pass, int dtype, int K, size_t smem) {
    static std::mutex mu;
    struct Key {
        int dev, pass, dtype, K;
        size_t smem;
        int val;
    };
    static std::vector<Key> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    for (const Key& k : cache)
        if (k.dev == dev && k.pass == pass && k.dtype == dtype && k.K == K && k.smem == smem)
            return k.val;
    const void* fn = dtype == IABN_F32
                         ? (pass == 0 ? (const void*)nhwc_fused_kernel<float, 0>
                                      : (const void*)nhwc_fused_kernel<float, 1>)
                         : (pass == 0 ? (const void*)nhwc_fused_kernel<__nv_bfloat16, 0>
                                      : (const void*)nhwc_fused_kernel<__nv_bfloat16, 1>);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)K, 1, 1);
    cfg.blockDim = dim3(kNhwcThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    if (cache.size() < 4096) cache.push_back(Key{dev, pass, dtype, K, smem, n});
    return n;
}

// test hooks (iabn_debug_nhwc_plan): forced g, K and launched clusters, 0 = automatic
std::atomic<int> g_nhwc_force_g{0}, g_nhwc_force_k{0}, g_nhwc_force_clusters{0};

// (g, K) from measurements on B200 (tools/nhwc_tune.py, profiles/r02_nhwc_tune_*.json):
// 2-D TMA boxes of narrow rows move few bytes per request, so the per-CTA chain (load,
// reduce, exchange, apply, store) is short only for small slabs and many CTAs: group rows
// of 32 bytes (then 64, then 16), K = ceil(128 / groups) CTAs per group (at least 128 CTAs
// when the channels allow; ~96 for <= 16 groups; at most 8 per cluster), raised while a backward CTA would hold
// more than 80 KB, all groups in one wave of co-resident clusters.  Layers with more than
// 32768 rows (N*HW; the 56x56 and 112x112 layers at N = 32) keep the streaming schedule:
// their groups do not fit on chip at a useful width.  Env IABN_NHWC_G (channels) /
// IABN_NHWC_K (or the iabn_debug_nhwc_plan hook) force a choice.
NhwcPlan nhwc_plan(const Geom& g, int pass, const DevFacts& f, uint32_t flags) {
    NhwcPlan best;
    if (g.layout != IABN_NHWC || (flags & IABN_EVAL)) return best;
    if ((g.C * g.b) % 16 != 0 || g.m >= (1ll << 31) || g.C >= (1ll << 31)) return best;
    if (!(flags & IABN_FORCE_FUSED) && env_int("IABN_NHWC_FUSED", 1) == 0) return best;
    const int nin = pass == 0 ? 1 : 2, NR = pass == 0 ? 3 : 2;
    const size_t budget = (size_t)f.max_smem_optin - 2048;
    const int gforce = g_nhwc_force_g.load() ? g_nhwc_force_g.load() : env_int("IABN_NHWC_G", 0);
    const int kforce = g_nhwc_force_k.load() ? g_nhwc_force_k.load() : env_int("IABN_NHWC_K", 0);
    const bool forced = gforce || kforce;
    if (!forced && !(flags & IABN_FORCE_FUSED) && g.m > env_int("IABN_NHWC_MAX_ROWS", 32768))
        return best;
    // the plan of (group bytes gb, K), or !ok if it does not fit
    auto make = [&](int gb, int K) -> NhwcPlan {
        NhwcPlan p;
        const uint32_t gch = (uint32_t)(gb / g.b);
        const uint32_t cols = (uint32_t)gb / 16, rs = kNhwcThreads / cols;
        // rows per CTA in nbox boxes of <= 256 rows (TMA box limit), each a multiple of
        // the block's row sweep; boxes sized to the rows, not to 256 (less padding)
        const uint32_t r0 = (uint32_t)((g.m + K - 1) / K);
        const uint32_t nb0 = (r0 + 255) / 256;
        const uint32_t box = std::min<uint32_t>(256, ((r0 + nb0 - 1) / nb0 + rs - 1) / rs * rs);
        const uint32_t nbox = (r0 + box - 1) / box;
        const uint32_t rows_cta = nbox * box;
        if (nbox > (uint32_t)kNhwcMaxBoxes) return p;
        const size_t slab = align256((size_t)rows_cta * gb);
        size_t off = slab * nin;
        const size_t red_off = off;
        off = align256(off + (size_t)(kNhwcThreads / 32) * gch * NR * 8);
        const size_t rec_off = off;
        off = align256(off + (size_t)2 * K * gch * NR * 8);
        const size_t coef_off = off;
        off = align256(off + (size_t)gch * 14 * 4);  // coefficients [g][8] + 6 params [g]
        const size_t bar_off = off;
        off += (size_t)nbox * 8;
        if (off > budget) return p;
        const int mc = nhwc_max_clusters(pass, g.dtype, K, off);
        if (mc <= 0) return p;
        p.ngroups = (uint32_t)((g.C + gch - 1) / gch);
        int clusters = (int)std::min<int64_t>(mc, p.ngroups);
        if (const int fc = g_nhwc_force_clusters.load()) clusters = std::min(clusters, fc);
        p.ok = true;
        p.g = gch;
        p.cols = cols;
        p.K = (uint32_t)K;
        p.rows_cta = rows_cta;
        p.box_rows = box;
        p.slab = (uint32_t)slab;
        p.red_off = (uint32_t)red_off;
        p.rec_off = (uint32_t)rec_off;
        p.coef_off = (uint32_t)coef_off;
        p.bar_off = (uint32_t)bar_off;
        p.smem = off;
        p.clusters = clusters;
        p.est_us = std::ceil((double)p.ngroups / clusters);  // waves
        return p;
    };
    if (forced) {
        for (int gb = 256; gb >= 16; gb /= 2) {
            if (gforce && gb / g.b != gforce) continue;
            if (!gforce && gb / g.b > g.C && gb > 16) continue;
            for (int K = 1; K <= kNhwcMaxK; ++K) {
                if (kforce && K != kforce) continue;
                const NhwcPlan p = make(gb, K);
                if (p.ok) {
                    best = p;
                    goto done;
                }
            }
        }
        goto done;
    }
    for (const int gb : {32, 64, 16}) {
        if (gb / g.b > g.C && gb > 16) continue;
        const int64_t groups = (g.C * g.b + gb - 1) / gb;
        // ~128 CTAs; ~96 when the groups are few (<= 16: K = 6 at 16 groups measured 8-12 %
        // faster than 8, r02: bf16 256x14^2 18.5 -> 16.4 us, fp32 128x14^2 16.0 -> 14.2 us)
        const int64_t tgt = groups <= 16 ? (96 + groups / 2) / groups : (128 + groups - 1) / groups;
        int K = (int)std::min<int64_t>(kNhwcMaxK, std::max<int64_t>(1, tgt));
        NhwcPlan p;
        for (; K <= kNhwcMaxK; ++K) {  // the first one-wave plan from the target K up
            p = make(gb, K);
            if (p.ok && p.est_us <= 1.0) break;
        }
        if (!(p.ok && p.est_us <= 1.0)) continue;
        // backward: at most ~80 KB of slab per CTA while a larger cluster stays one wave
        while (p.K < (uint32_t)kNhwcMaxK && (size_t)p.slab * nin > 80 * 1024) {
            const NhwcPlan q = make(gb, (int)p.K + 1);
            if (!(q.ok && q.est_us <= 1.0)) break;
            p = q;
        }
        best = p;
        break;
    }
done:
    if (best.ok && env_int("IABN_VERBOSE", 0)) {
        static std::mutex pm;
        static int printed = 0;
        std::lock_guard<std::mutex> lk(pm);
        if (printed++ < 32)
            fprintf(stderr, "[iabn] nhwc pass=%d C=%lld m=%lld: g=%u K=%u rows_cta=%u box=%u groups=%u clusters=%d smem=%zu waves=%.0f\n",
                    pass, (long long)g.C, (long long)g.m, best.g, best.K, best.rows_cta,
                    best.box_rows, best.ngroups, best.clusters, best.smem, best.est_us);
    }
    return best;
}

// ====================================================================== small NCHW layers
// kernels_small.cuh: a channel's covering 16-byte slots held in the registers of a team of
// 32*tw threads (<= kSmallR slots per thread), one launch per pass.
struct SmallPlan {
    bool ok = false;
    uint32_t W = 0, tw = 0, R = 0;
    unsigned grid = 0;
};
std::atomic<int> g_small_force{0};  // test hook: 1 on when possible, -1 off, 0 automatic
std::atomic<int> g_small_force_r{0};  // test hook: slots per thread (4 or 8), 0 automatic

SmallPlan small_plan(const Geom& g, uint32_t flags, int sms) {
    SmallPlan p;
    if (g.layout != IABN_NCHW || (flags & IABN_EVAL)) return p;
    const int f = g_small_force.load();
    if (f < 0 || (!f && !env_int("IABN_SMALL", 1))) return p;
    if ((g.E * g.b) % 16 != 0 || g.C >= (1ll << 31)) return p;  // the last plane's covering range
    // measured (tools/small_tune.py, profiles/r02_small_tune_*.log): faster than the
    // channel-resident kernels up to 16 KB per channel (bf16 14x14 and every 7x7 layer at
    // N = 32: -25..-42 % per pass); at 25 KB (fp32 14x14) equal or slower
    // Above 16 KB only when the layer is one wave at the R = 8 kernels' occupancy (2 CTAs
    // per SM): fp32 128x14^2 (25 KB) 7.9 / 7.5 -> 5.4 / 5.4 us, while 512x14^2 (4 waves
    // of channels) stays channel-resident (11.0 / 11.2 vs 11.8 / 12.3 us).
    const bool one_wave = g.m * g.b <= 32 * 1024 && g.C <= 2 * (int64_t)sms;
    if (!f && g.m * g.b > (int64_t)env_int("IABN_SMALL_MAX_KB", 16) * 1024 && !one_wave) return p;
    const int64_t W = (g.HW * g.b + 30) / 16;  // >= the slots covering any plane
    auto fit = [&](uint32_t R, SmallPlan& q) {
        for (uint32_t tw : {1u, 2u, 4u, 8u}) {
            if (g.N * W <= (int64_t)32 * tw * R) {
                q.ok = true;
                q.W = (uint32_t)W;
                q.tw = tw;
                q.R = R;
                const int64_t per = (kSmallThreads / 32) / tw;  // channels per CTA
                q.grid = (unsigned)((g.C + per - 1) / per);
                return true;
            }
        }
        return false;
    };
    // R = 4 (thinner warps, more of them in flight) wherever a team of <= 8 warps holds the
    // channel: measured faster on every 7x7 and bf16 14x14 layer but one (bf16 512x14^2
    // backward +6 %), e.g. bf16 128x14^2 5.9 / 7.4 -> 4.2 / 4.8 us, 2688x7^2 13.7 / 19.1 ->
    // 11.9 / 14.3 us; else R = 8.  Forced R (test hook / IABN_SMALL_R): preferred when it fits.
    const int fr = g_small_force_r.load() ? g_small_force_r.load() : env_int("IABN_SMALL_R", 0);
    if (fr == 8 && fit(8, p)) return p;
    if (fit(4, p)) return p;
    fit(8, p);
    return p;
}

template <typename T, int ACT = 0>
iabn_status launch_small(int pass, const Geom& g, const SmallPlan& p, SmallArgs a, cudaStream_t st) {
    a.C = g.C;
    a.HW = g.HW;
    a.N = (uint32_t)g.N;
    a.W = p.W;
    a.fd_w = fd32(p.W);
    a.tw = p.tw;
    a.inv_n = 1.0 / ((double)g.N * (double)g.HW);
    a.trace = nullptr;
    if (env_int("IABN_SMALL_TRACE", 0)) {  // experiments (a build with -DIABN_PHASE_TRACE)
        static unsigned long long* buf = nullptr;
        static size_t cap = 0;
        const size_t need = (size_t)p.grid * kSmallTrace;
        if (need > cap) {
            if (buf) cudaFree(buf);
            cudaMalloc(&buf, need * sizeof(unsigned long long));
            cap = need;
        }
        a.trace = buf;
        g_trace = buf;
        g_trace_n = need;
        g_trace_ch = (uint32_t)kSmallTrace;
    }
    if (p.R == 4) {
        if (pass == 0) launch_pdl(small_kernel<T, 0, 4, ACT>, p.grid, kSmallThreads, 0, st, a);
        else launch_pdl(small_kernel<T, 1, 4, ACT>, p.grid, kSmallThreads, 0, st, a);
    } else {
        if (pass == 0) launch_pdl(small_kernel<T, 0, 8, ACT>, p.grid, kSmallThreads, 0, st, a);
        else launch_pdl(small_kernel<T, 1, 8, ACT>, p.grid, kSmallThreads, 0, st, a);
    }
    return check_launch(pass == 0 ? "small_kernel<fwd>" : "small_kernel<bwd>");
}

// 2-D tensor map of an NHWC activation: dim 0 = C channels, dim 1 = m rows, box = [g, R]
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
        cudaGetLastError();
    });
    return fn;
}

iabn_status nhwc_tmap(CUtensorMap* tm, const void* ptr, const Geom& g, const NhwcPlan& p) {
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(IABN_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)g.C, (cuuint64_t)g.m};
    const cuuint64_t strides[1] = {(cuuint64_t)(g.C * g.b)};
    const cuuint32_t box[2] = {p.g, p.box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = enc(tm, g.dtype == IABN_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                   : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                           2, const_cast<void*>(ptr), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(IABN_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return IABN_OK;
}

template <typename T, int ACT = 0>
iabn_status launch_nhwc(int pass, const Geom& g, const NhwcPlan& p, NhwcArgs a, const void* in0,
                        const void* in1, void* out, cudaStream_t st) {
    CUtensorMap t0, t1, t2;
    IABN_TRY(nhwc_tmap(&t0, in0, g, p));
    IABN_TRY(nhwc_tmap(&t1, pass == 1 ? in1 : in0, g, p));
    IABN_TRY(nhwc_tmap(&t2, out, g, p));
    a.in0 = in0;
    a.C = g.C;
    a.m = (uint32_t)g.m;
    a.inv_m = 1.0 / (double)g.m;
    a.g = p.g;
    a.cols = p.cols;
    a.ngroups = p.ngroups;
    a.K = p.K;
    a.rows_cta = p.rows_cta;
    a.box_rows = p.box_rows;
    a.slab_bytes = p.slab;
    a.red_off = p.red_off;
    a.rec_off = p.rec_off;
    a.coef_off = p.coef_off;
    a.bar_off = p.bar_off;
    a.prefetch = (uint32_t)env_int("IABN_NHWC_PREFETCH", 1);
    a.trace = nullptr;
    if (env_int("IABN_NHWC_TRACE", 0)) {  // experiments only: phase timestamps
        static unsigned long long* buf = nullptr;
        static size_t cap = 0;
        const size_t need = (size_t)p.clusters * p.K * kNhwcTrace;
        if (need > cap) {
            if (buf) cudaFree(buf);
            cudaMalloc(&buf, need * sizeof(unsigned long long));
            cap = need;
        }
        a.trace = buf;
        g_trace = buf;
        g_trace_n = need;
        g_trace_ch = (uint32_t)kNhwcTrace;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.clusters * p.K), 1, 1);
    cfg.blockDim = dim3(kNhwcThreads, 1, 1);
    cfg.dynamicSmemBytes = p.smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = p.K;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    const cudaError_t e = pass == 0 ? cudaLaunchKernelEx(&cfg, nhwc_fused_kernel<T, 0, ACT>, t0, t1, t2, a)
                                    : cudaLaunchKernelEx(&cfg, nhwc_fused_kernel<T, 1, ACT>, t0, t1, t2, a);
    if (e != cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return fail(IABN_ERR_CUDA, "nhwc launch: %s", cudaGetErrorString(e));
    }
    return check_launch(pass == 0 ? "nhwc_fused_kernel<fwd>" : "nhwc_fused_kernel<bwd>");
}

FastDiv cover_fd(const Geom& g) { return make_fastdiv((uint32_t)(g.HW / (16 / g.b) + 2)); }

// ====================================================================== grid-resident NHWC
// The whole NHWC tensor resident in the grid's shared memory (kernels_gres.cuh):
// returns the grid (0 = not possible): rows split over G CTAs of at most
// IABN_GRES_KB (default 96) KB of input each, 2 CTAs per SM, G <= kGresMaxG.
int gres_grid(const Geom& g, int pass, uint32_t flags, const DevFacts& f) {
    if (g.layout != IABN_NHWC || !vec_ok(g) || g.E >= (1ll << 31)) return 0;
    if (flags & (IABN_FORCE_STREAMING | IABN_FORCE_FUSED | IABN_EVAL))
        return 0;
    // opt-in: measured against the streaming kernels (tools/shape_graph.py, graph replay,
    // DenseNet-like NHWC shapes at N = 32) it wins for bf16 layers of ~13 MB (1.1-1.4x)
    // and loses for tiny and fp32 layers, and whole-network sweeps come out slower
    if (!(flags & IABN_FORCE_RESIDENT) && env_int("IABN_GRES", 0) != 1) return 0;
    const int64_t row_bytes = g.C * g.b * (pass == 0 ? 1 : 2);
    if (g.C * g.b / 16 > kThreads) return 0;  // one 16-byte column per thread at least
    const int64_t per = (int64_t)std::max(8, env_int("IABN_GRES_KB", 96)) * 1024;
    const int64_t maxg = std::min<int64_t>(std::min<int64_t>(kGresMaxG, 2 * (int64_t)f.sms), g.m);
    int64_t G = (g.m * row_bytes + per - 1) / per;
    G = std::max<int64_t>(G, std::min<int64_t>(f.sms, g.m));  // at least one CTA per SM
    if (G > maxg) return 0;
    // the largest slice must fit (rows split as evenly as possible)
    if ((g.m + G - 1) / G * row_bytes > per) return 0;
    return (int)G;
}

// Persistent grid-barrier state, one slot per stream (allocated and zeroed once per
// device; a stream keeps its slot, so launches on one stream are ordered).
GridBar* gres_bar(cudaStream_t st) {
    constexpr int kSlotsPerDev = 256;
    static std::mutex mu;
    static GridBar* base[kMaxDev] = {};
    static cudaStream_t owner[kMaxDev][kSlotsPerDev];
    static int used[kMaxDev] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!base[dev]) {
        GridBar* p = nullptr;
        if (cudaMalloc(&p, kSlotsPerDev * sizeof(GridBar)) != cudaSuccess) return nullptr;
        if (cudaMemset(p, 0, kSlotsPerDev * sizeof(GridBar)) != cudaSuccess) return nullptr;
        base[dev] = p;
    }
    for (int i = 0; i < used[dev]; ++i)
        if (owner[dev][i] == st) return base[dev] + i;
    if (used[dev] == kSlotsPerDev) return nullptr;
    owner[dev][used[dev]] = st;
    return base[dev] + used[dev]++;
}

template <typename T, int PASS>
iabn_status launch_gres(const Geom& g, int G, GresArgs a, cudaStream_t st) {
    a.bar = gres_bar(st);
    if (!a.bar) return fail(IABN_ERR_CUDA, "grid-barrier state unavailable");
    const int64_t row_bytes = g.C * g.b * (PASS == 0 ? 1 : 2);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = (size_t)((g.m + G - 1) / G * row_bytes);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, gres_kernel<T, PASS>, a);
    if (e != cudaSuccess) {
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return fail(IABN_ERR_CUDA, "grid-resident kernel: %s", cudaGetErrorString(e));
    }
    return check_launch(PASS == 0 ? "gres_kernel<fwd>" : "gres_kernel<bwd>");
}

// ====================================================================== streaming launches
template <typename T, int PASS, int ACT = 0>
iabn_status launch_nb(const Geom& g, int S, const void* in0, const void* in1, const float* gamma,
                      const float* beta, float eps, float slope, uint32_t flags, double* part,
                      cudaStream_t st) {
    NbArgs a{};
    a.in0 = in0;
    a.in1 = in1;
    a.gamma = gamma;
    a.beta = beta;
    a.C = g.C;
    a.rows = g.m;
    a.cv = (uint32_t)(g.C * g.b / 16);
    a.rt = std::max<uint32_t>(1, (uint32_t)kThreads / a.cv);
    a.rps = std::max<uint32_t>(1, kNbStageBytes / (PASS == 0 ? 1 : 2) / (a.cv * 16));
    a.eps = eps;
    a.slope = slope;
    a.flags = flags;
    a.part = part;
    a.trace = nullptr;
    if (env_int("IABN_NB_TRACE", 0)) {  // experiments only: phase timestamps
        static unsigned long long* buf = nullptr;
        static size_t cap = 0;
        const size_t need = (size_t)S * kNbCluster * kNbTrace;
        if (need > cap) {
            if (buf) cudaFree(buf);
            cudaMalloc(&buf, need * sizeof(unsigned long long));
            cap = need;
        }
        a.trace = buf;
        g_trace = buf;
        g_trace_n = need;
        g_trace_ch = (uint32_t)kNbTrace;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(S * kNbCluster));
    cfg.blockDim = dim3(a.rt * a.cv);
    cfg.dynamicSmemBytes = kNbSmem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kNbCluster;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    if (a.trace) {  // experiments: residency of this launch
        int nc = -1, nb = -1;
        cudaOccupancyMaxActiveClusters(&nc, (const void*)nhwc_bulk_reduce_kernel<T, PASS, false>, &cfg);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, (const void*)nhwc_bulk_reduce_kernel<T, PASS, false>,
                                                      (int)cfg.blockDim.x, kNbSmem);
        fprintf(stderr, "nb: grid %u block %u smem %zu: max active clusters %d, blocks/SM %d\n",
                cfg.gridDim.x, cfg.blockDim.x, (size_t)kNbSmem, nc, nb);
        cudaGetLastError();
    }
    if (PASS == 0)
        cudaLaunchKernelEx(&cfg, nhwc_bulk_reduce_kernel<T, 0, false>, a);
    else if (flags & IABN_VARIANT_I)
        cudaLaunchKernelEx(&cfg, nhwc_bulk_reduce_kernel<T, 1, false, ACT>, a);
    else
        cudaLaunchKernelEx(&cfg, nhwc_bulk_reduce_kernel<T, 1, true, ACT>, a);
    return check_launch(PASS == 0 ? "nhwc_bulk_reduce<stats>" : "nhwc_bulk_reduce<grad>");
}

template <typename T>
iabn_status launch_stats(const Geom& g, int S, const void* x, double* part, cudaStream_t st) {
    const bool vec = vec_ok(g);
    if (g.layout == IABN_NCHW) {
        const dim3 grid((unsigned)g.C, (unsigned)S);
        const FastDiv fd = fd32(g.HW);
        if (vec)
            launch_pdl(stats_nchw_kernel<T, true>, grid, kThreads, 0, st, (const T*)x, g.C, g.HW,
                                                                  (uint32_t)g.m, fd, part);
        else  // planes not 16-byte aligned: masked covering vectors
            launch_pdl(nchw_cover_kernel<T, 0>, grid, kThreads, 0, st,
                (const T*)x, nullptr, nullptr, nullptr, g.C, g.HW, g.N, g.E, 0.f, 1.f, 1.f, 0u,
                cover_fd(g), part);
    } else if (nb_grid(g)) {
        return launch_nb<T, 0>(g, S, x, nullptr, nullptr, nullptr, 1e-5f, 1.f, 0u, part, st);
    } else {
        const int V = vec ? 16 / g.b : 1;
        const dim3 grid((unsigned)((g.C + 16 * V - 1) / (16 * V)), (unsigned)S);
        if (vec)
            launch_pdl(stats_nhwc_kernel<T, true>, grid, kThreads, 0, st, (const T*)x, g.C, g.m, part);
        else
            launch_pdl(stats_nhwc_kernel<T, false>, grid, kThreads, 0, st, (const T*)x, g.C, g.m, part);
    }
    return check_launch("stats kernel");
}

template <typename T>
iabn_status launch_bwd_reduce(const Geom& g, int S, const void* z, const void* dz,
                              const float* gamma, const float* beta, float eps, float slope,
                              uint32_t flags, double* part, cudaStream_t st) {
    const bool vec = vec_ok(g);
    const float inv_slope = 1.0f / slope;
    if (g.layout == IABN_NCHW) {
        const dim3 grid((unsigned)g.C, (unsigned)S);
        const FastDiv fd = fd32(g.HW);
        if (vec)
            launch_pdl(bwd_reduce_nchw_kernel<T, true>, grid, kThreads, 0, st,
                (const T*)z, (const T*)dz, gamma, beta, g.C, g.HW, (uint32_t)g.m, fd, eps, slope,
                inv_slope, flags, part);
        else  // planes not 16-byte aligned: masked covering vectors
            launch_pdl(nchw_cover_kernel<T, 1>, grid, kThreads, 0, st,
                (const T*)z, (const T*)dz, gamma, beta, g.C, g.HW, g.N, g.E, eps, slope,
                inv_slope, flags, cover_fd(g), part);
    } else if (nb_grid(g)) {
        return launch_nb<T, 1>(g, S, z, dz, gamma, beta, eps, slope, flags, part, st);
    } else {
        const int V = vec ? 16 / g.b : 1;
        const dim3 grid((unsigned)((g.C + 16 * V - 1) / (16 * V)), (unsigned)S);
        if (vec)
            launch_pdl(bwd_reduce_nhwc_kernel<T, true>, grid, kThreads, 0, st,
                (const T*)z, (const T*)dz, gamma, beta, g.C, g.m, eps, slope, inv_slope, flags,
                part);
        else
            launch_pdl(bwd_reduce_nhwc_kernel<T, false>, grid, kThreads, 0, st,
                (const T*)z, (const T*)dz, gamma, beta, g.C, g.m, eps, slope, inv_slope, flags,
                part);
    }
    return check_launch("bwd_reduce kernel");
}

// Elementwise passes in whole-sample chunks of < 2^31 elements whose byte
// offsets stay 16-byte aligned (channel phase is preserved at sample boundaries).
int64_t samples_per_chunk(const Geom& g) {
    const int64_t per = g.C * g.HW;
    int64_t spc = ((1ll << 31) - 1) / per;
    int64_t q = 1;
    while (q < 16 && ((per * g.b * q) % 16) != 0) q *= 2;
    spc = (spc / q) * q;
    return spc;
}

int apply_grid(int64_t E, int b, int sms) {
    const int64_t nvec = E * b / 16;
    const int64_t want = (nvec + (int64_t)kThreads * kUnroll - 1) / ((int64_t)kThreads * kUnroll);
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
}

// NHWC aligned: a grid whose stride (grid * kThreads vectors) is a multiple of the
// C/V vectors of one row, so every thread keeps one channel group (0 = not possible)
// Resident CTAs per SM of a kernel (cached per kernel; 0 if the query fails)
int blocks_per_sm(const void* fn) {
    static std::mutex mu;
    static std::pair<const void*, int> cache[64];
    static int n = 0;
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < n; ++i)
        if (cache[i].first == fn) return cache[i].second;
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kThreads, 0) != cudaSuccess) b = 0;
    cudaGetLastError();
    if (n < 64) cache[n++] = {fn, b};
    return b;
}

// NHWC aligned: a grid whose stride (grid * kThreads vectors) is a multiple of the C/V
// vectors of one row, so every thread keeps one channel group (0 = not possible); one
// batch of kNhwcApplyUnroll vectors per thread, but at most one wave of resident CTAs
// (bpsm per SM) for the bf16 applies: r02 ncu, 784 CTAs at 444 resident ran a 77 % second
// wave (bf16 128x56^2 forward 23.8 -> 21.1 us, 64x112^2 37.7 -> 31.4 us)
int nhwc_grid(const Geom& g, int64_t nvec, int sms, int bpsm = 0) {
    const int64_t cv = g.C * g.b / 16;
    const int64_t q = cv / std::gcd<int64_t>(cv, kThreads);  // grid must be a multiple of q
    int64_t want = std::min<int64_t>((nvec + kThreads * kNhwcApplyUnroll - 1) / (kThreads * kNhwcApplyUnroll),
                                     (int64_t)sms * 64);
    // (only for the register-heavy kernels, <= 3 CTAs per SM: the bf16 applies; with more
    // resident CTAs the waves of fresh CTAs overlap better than a per-thread loop, e.g.
    // fp32 32x256x56^2 forward 50.9 -> 55.1 us with the cap)
    if (bpsm > 0 && bpsm <= 3 && want > (int64_t)sms * bpsm) want = (int64_t)sms * bpsm / q * q;
    if (q > (int64_t)sms * 16) return 0;
    return (int)(std::max<int64_t>(1, (want + q - 1) / q) * q);
}

template <typename T, bool EV>
iabn_status launch_fwd_apply_ev(const Geom& g, const void* x, void* z, const float4* coef,
                                float slope, int sms, cudaStream_t st, const EvalCoef& ev) {
    const int64_t spc = samples_per_chunk(g);
    if (spc <= 0) return fail(IABN_ERR_UNSUPPORTED, "sample too large for the streaming apply");
    const bool al = vec_ok(g);
    const FastDiv fh = fd32(g.HW), fc = fd32(g.C);
    for (int64_t n0 = 0; n0 < g.N; n0 += spc) {
        const int64_t nn = std::min(spc, g.N - n0);
        const int64_t off = n0 * g.C * g.HW;
        const uint32_t E = (uint32_t)(nn * g.C * g.HW);
        const T* xp = (const T*)x + off;
        T* zp = (T*)z + off;
        const int grid = apply_grid(E, g.b, sms);
        if (g.layout == IABN_NCHW && g.HW >= 16 / g.b) {  // any alignment (straddles handled)
            launch_pdl(fwd_apply_rows_kernel<T, EV>, grid, kThreads, 0, st,
                xp, zp, coef, E, (uint32_t)g.HW, (uint32_t)g.C, fh, fc, slope, ev);
        } else if (g.layout == IABN_NCHW) {
            if (al)
                launch_pdl(fwd_apply_kernel<T, 0, true, EV>, grid, kThreads, 0, st, xp, zp, coef, E, fh, fc, slope, ev);
            else
                launch_pdl(fwd_apply_kernel<T, 0, false, EV>, grid, kThreads, 0, st, xp, zp, coef, E, fh, fc, slope, ev);
        } else if (al && nhwc_grid(g, E / (16 / g.b), sms) > 0) {
            const int bp = blocks_per_sm((const void*)fwd_apply_nhwc_kernel<T, EV>);
            launch_pdl(fwd_apply_nhwc_kernel<T, EV>, nhwc_grid(g, E / (16 / g.b), sms, bp), kThreads, 0, st,
                xp, zp, coef, (uint32_t)(E / (16 / g.b)), (uint32_t)(g.C * g.b / 16), slope, ev);
        } else {
            if (al)
                launch_pdl(fwd_apply_kernel<T, 1, true, EV>, grid, kThreads, 0, st, xp, zp, coef, E, fh, fc, slope, ev);
            else
                launch_pdl(fwd_apply_kernel<T, 1, false, EV>, grid, kThreads, 0, st, xp, zp, coef, E, fh, fc, slope, ev);
        }
        IABN_TRY(check_launch("fwd_apply kernel"));
    }
    return IABN_OK;
}
template <typename T>
iabn_status launch_fwd_apply(const Geom& g, const void* x, void* z, const float4* coef,
                             float slope, int sms, cudaStream_t st) {
    return launch_fwd_apply_ev<T, false>(g, x, z, coef, slope, sms, st, EvalCoef{});
}

template <typename T>
iabn_status launch_bwd_apply(const Geom& g, const void* z, const void* dz, void* dx,
                             const float4* coef, float slope, int sms, cudaStream_t st) {
    const int64_t spc = samples_per_chunk(g);
    if (spc <= 0) return fail(IABN_ERR_UNSUPPORTED, "sample too large for the streaming apply");
    const bool al = vec_ok(g);
    const FastDiv fh = fd32(g.HW), fc = fd32(g.C);
    const float inv_slope = 1.0f / slope;
    for (int64_t n0 = 0; n0 < g.N; n0 += spc) {
        const int64_t nn = std::min(spc, g.N - n0);
        const int64_t off = n0 * g.C * g.HW;
        const uint32_t E = (uint32_t)(nn * g.C * g.HW);
        const T* zp = (const T*)z + off;
        const T* dzp = (const T*)dz + off;
        T* dxp = (T*)dx + off;
        const int grid = apply_grid(E, g.b, sms);
        if (g.layout == IABN_NCHW && g.HW >= 16 / g.b) {  // any alignment (straddles handled)
            launch_pdl(bwd_apply_rows_kernel<T>, grid, kThreads, 0, st, zp, dzp, dxp, coef, E, (uint32_t)g.HW,
                                                               (uint32_t)g.C, fh, fc, slope, inv_slope);
        } else if (g.layout == IABN_NCHW) {
            if (al)
                launch_pdl(bwd_apply_kernel<T, 0, true>, grid, kThreads, 0, st, zp, dzp, dxp, coef, E, fh, fc, slope, inv_slope);
            else
                launch_pdl(bwd_apply_kernel<T, 0, false>, grid, kThreads, 0, st, zp, dzp, dxp, coef, E, fh, fc, slope, inv_slope);
        } else if (al && nhwc_grid(g, E / (16 / g.b), sms) > 0) {
            const int bp = blocks_per_sm((const void*)bwd_apply_nhwc_kernel<T>);
            launch_pdl(bwd_apply_nhwc_kernel<T>, nhwc_grid(g, E / (16 / g.b), sms, bp), kThreads, 0, st,
                zp, dzp, dxp, coef, (uint32_t)(E / (16 / g.b)), (uint32_t)(g.C * g.b / 16), slope,
                inv_slope);
        } else {
            if (al)
                launch_pdl(bwd_apply_kernel<T, 1, true>, grid, kThreads, 0, st, zp, dzp, dxp, coef, E, fh, fc, slope, inv_slope);
            else
                launch_pdl(bwd_apply_kernel<T, 1, false>, grid, kThreads, 0, st, zp, dzp, dxp, coef, E, fh, fc, slope, inv_slope);
        }
        IABN_TRY(check_launch("bwd_apply kernel"));
    }
    return IABN_OK;
}

unsigned cgrid(int64_t C) { return (unsigned)((C + 127) / 128); }
// warp-per-channel kernels (combine / coefficients), 128 threads = 4 channels per block
unsigned wgrid(int64_t C) { return (unsigned)((C + 3) / 4); }

// ====================================================================== NCCL (dlopen)
struct Nccl {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;  // optional (fused sync setup)
};
Nccl g_nccl;
std::mutex g_nccl_mu;

Nccl* nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl.tried) {
        g_nccl.tried = true;
        const char* env = getenv("IABN_NCCL_LIB");
        void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            g_nccl.why = dlerror();
        } else {
            g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
            g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
            g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
            g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
            g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
            g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllReduce &&
                        g_nccl.CommDestroy && g_nccl.GetErrorString;
            if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks required symbols";
        }
    }
    return g_nccl.ok ? &g_nccl : nullptr;
}

// Record buffers of the synchronized channel-resident kernels: peer[g] = rank g's buffer
// [2][cap][nranks] PeerRec (mapped into this process), ctr = the call counter.
struct SyncBuf {
    PeerRec* peer[kMaxRanks] = {};
    unsigned long long* ctr = nullptr;
    uint32_t cap = 0;
    int nranks = 0;
};

}  // namespace

// What the ranks agreed on for one (shard geometry, pass) of the fused-collective sync:
// whether every rank can run the channel-resident kernel with the same plan (same
// channel -> cluster mapping, equal shards), and the global count m_G.
struct SyncAgree {
    int64_t n, c, hw;
    int dtype, layout, pass;
    bool fused;
    int64_t m_global;
};

struct iabn_comm_s {
    ncclComm_t comm;
    int nranks, rank;
    // fused-collective sync (IABN_SYNC_FUSED): this rank's record buffer, every rank's
    // buffer mapped through CUDA IPC (peer access over NVLink), the call counter
    SyncBuf sb{};
    void* own = nullptr;
    std::vector<SyncAgree> agree{};
    // phase timing (iabn_comm_set_timing): events [pass][4] around reduce | all-reduce | apply
    bool timing = false;
    bool timed[2] = {false, false};
    cudaEvent_t ev[2][4] = {};
};

namespace {

iabn_status allreduce_f64(double* buf, size_t count, iabn_comm comm, cudaStream_t st) {
    Nccl* n = nccl();
    if (!n) return fail(IABN_ERR_NCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    const ncclResult_t r = n->AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm->comm, st);
    if (r != ncclSuccess) return fail(IABN_ERR_NCCL, "ncclAllReduce: %s", n->GetErrorString(r));
    return IABN_OK;
}

// The fused-collective sync buffers of a communicator (collective: every rank calls it
// at the same call with the same C): allocate [2][cap][nranks] records, export them
// with CUDA IPC, all-gather the handles over NCCL and map every peer's buffer.
iabn_status comm_sync_buf(iabn_comm comm, int64_t C, cudaStream_t st) {
    if (comm->sb.cap >= C) return IABN_OK;
    Nccl* n = nccl();
    if (!n || !n->AllGather) return fail(IABN_ERR_NCCL, "NCCL all-gather unavailable");
    if (comm->nranks > kMaxRanks)
        return fail(IABN_ERR_UNSUPPORTED, "fused sync supports at most %d ranks", kMaxRanks);
    auto cuda = [](cudaError_t e, const char* what) -> iabn_status {
        return e == cudaSuccess ? IABN_OK
                                : fail(IABN_ERR_CUDA, "fused sync setup, %s: %s", what, cudaGetErrorString(e));
    };
    // every rank finished its earlier calls before anyone drops the old buffers
    IABN_TRY(cuda(cudaStreamSynchronize(st), "stream synchronize"));
    const uint32_t cap = (uint32_t)std::max<int64_t>(std::max<int64_t>(C, 2ll * comm->sb.cap), 1024);
    const size_t bytes = (size_t)2 * cap * comm->nranks * sizeof(PeerRec);
    void* nb = nullptr;
    IABN_TRY(cuda(cudaMalloc(&nb, bytes), "cudaMalloc"));
    // stream-ordered initialisation (the caller's stream may be a non-blocking one, which
    // the legacy-stream cudaMemset / cudaMemcpy would not be ordered with)
    IABN_TRY(cuda(cudaMemsetAsync(nb, 0, bytes, st), "cudaMemsetAsync"));
    if (!comm->sb.ctr) {
        static const unsigned long long init[2] = {1ull, 0ull};
        IABN_TRY(cuda(cudaMalloc(&comm->sb.ctr, sizeof(init)), "cudaMalloc"));
        IABN_TRY(cuda(cudaMemcpyAsync(comm->sb.ctr, init, sizeof(init), cudaMemcpyHostToDevice, st),
                      "counter"));
    }
    cudaIpcMemHandle_t h;
    IABN_TRY(cuda(cudaIpcGetMemHandle(&h, nb), "cudaIpcGetMemHandle"));
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    char* dh = nullptr;
    IABN_TRY(cuda(cudaMalloc(&dh, hb * comm->nranks), "cudaMalloc"));
    IABN_TRY(cuda(cudaMemcpyAsync(dh + hb * comm->rank, &h, hb, cudaMemcpyHostToDevice, st), "handle"));
    const ncclResult_t r = n->AllGather(dh + hb * comm->rank, dh, hb, ncclInt8, comm->comm, st);
    if (r != ncclSuccess) return fail(IABN_ERR_NCCL, "ncclAllGather: %s", n->GetErrorString(r));
    std::vector<cudaIpcMemHandle_t> hs(comm->nranks);
    IABN_TRY(cuda(cudaStreamSynchronize(st), "stream synchronize"));
    IABN_TRY(cuda(cudaMemcpy(hs.data(), dh, hb * comm->nranks, cudaMemcpyDeviceToHost), "handles"));
    cudaFree(dh);
    for (int g = 0; g < comm->nranks; ++g) {
        if (g == comm->rank) continue;
        if (comm->sb.peer[g]) cudaIpcCloseMemHandle(comm->sb.peer[g]);
        void* pp = nullptr;
        IABN_TRY(cuda(cudaIpcOpenMemHandle(&pp, hs[g], cudaIpcMemLazyEnablePeerAccess),
                      "cudaIpcOpenMemHandle"));
        comm->sb.peer[g] = (PeerRec*)pp;
    }
    if (comm->own) cudaFree(comm->own);
    comm->own = nb;
    comm->sb.peer[comm->rank] = (PeerRec*)nb;
    comm->sb.cap = cap;
    comm->sb.nranks = comm->nranks;
    return IABN_OK;
}

// Phase boundary k (0..3) of pass `pass` of a timed synchronized call.
void phase_mark(iabn_comm comm, int pass, int k, cudaStream_t st) {
    if (!comm->timing) return;
    if (!comm->ev[pass][k] && cudaEventCreate(&comm->ev[pass][k]) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaEventRecord(comm->ev[pass][k], st);
    if (k == 3) comm->timed[pass] = true;
}

bool sync_fused_wanted(uint32_t flags) {
    return (flags & IABN_SYNC_FUSED) || env_int("IABN_SYNC_FUSED", 0) == 1;
}

// Collective (every rank, same call): do all ranks run the fused-collective kernel for
// this shard geometry and pass?  The kernels of different ranks wait on one another per
// channel, so they must agree -- same shard shape and same plan (K, clusters, nbuf: the
// channel -> cluster order) on every rank -- or all take the reduce / all-reduce / apply
// path.  Decided once per (geometry, pass) by an all-gather of each rank's plan (a host
// synchronisation: the first call of a shape must not be inside a CUDA-graph capture),
// then cached in the communicator.
iabn_status sync_agree(iabn_comm comm, const Geom& g, int pass, const FusedPlan& p,
                       cudaStream_t st, SyncAgree* out) {
    for (const SyncAgree& a : comm->agree)
        if (a.n == g.N && a.c == g.C && a.hw == g.HW && a.dtype == g.dtype &&
            a.layout == g.layout && a.pass == pass) {
            *out = a;
            return IABN_OK;
        }
    Nccl* n = nccl();
    if (!n || !n->AllGather) return fail(IABN_ERR_NCCL, "NCCL all-gather unavailable");
    constexpr int R = 8;
    const int64_t mine[R] = {g.N, g.C, g.HW, (int64_t)g.dtype | ((int64_t)g.layout << 8),
                             p.ok ? 1 : 0, p.K, p.clusters, p.nbuf};
    int64_t* d = nullptr;
    auto cuda = [](cudaError_t e, const char* what) -> iabn_status {
        return e == cudaSuccess ? IABN_OK
                                : fail(IABN_ERR_CUDA, "sync schedule agreement, %s: %s", what,
                                       cudaGetErrorString(e));
    };
    IABN_TRY(cuda(cudaMalloc(&d, sizeof(int64_t) * R * comm->nranks), "cudaMalloc"));
    std::vector<int64_t> all((size_t)R * comm->nranks);
    iabn_status s = cuda(cudaMemcpyAsync(d + R * comm->rank, mine, sizeof(mine),
                                         cudaMemcpyHostToDevice, st), "copy");
    if (s == IABN_OK) {
        const ncclResult_t r = n->AllGather(d + R * comm->rank, d, R, ncclInt64, comm->comm, st);
        if (r != ncclSuccess) s = fail(IABN_ERR_NCCL, "ncclAllGather: %s", n->GetErrorString(r));
    }
    if (s == IABN_OK)
        s = cuda(cudaMemcpyAsync(all.data(), d, sizeof(int64_t) * all.size(), cudaMemcpyDeviceToHost,
                                 st), "copy");
    if (s == IABN_OK) s = cuda(cudaStreamSynchronize(st), "stream synchronize");
    cudaFree(d);
    IABN_TRY(s);
    SyncAgree a{g.N, g.C, g.HW, (int)g.dtype, (int)g.layout, pass, true, 0};
    for (int r = 0; r < comm->nranks; ++r) {
        const int64_t* o = &all[(size_t)R * r];
        a.m_global += o[0] * o[2];
        if (!o[4] || memcmp(o, mine, sizeof(mine)) != 0) a.fused = false;
    }
    comm->agree.push_back(a);
    *out = a;
    return IABN_OK;
}

// ====================================================================== shared call bodies
struct Ctx {
    Geom g;
    DevFacts* dev;
    int S;
    WsLayout w;
    unsigned char* ws;
    cudaStream_t st;
};

// Host-only part of a call: geometry and workspace (no device access, so the
// validation paths run without a GPU).
iabn_status make_ctx(const iabn_desc* desc, void* ws, size_t ws_bytes, void* stream, Ctx* c) {
    IABN_TRY(make_geom(desc, &c->g));
    c->dev = nullptr;
    c->S = stat_splits(c->g);
    c->w = ws_layout(c->g, c->S);
    IABN_TRY(check_ws(c->g, ws, ws_bytes, c->w));
    c->ws = (unsigned char*)ws;
    c->st = (cudaStream_t)stream;
    return IABN_OK;
}

iabn_status attach_device(Ctx& c) { return device_facts(&c.dev); }

template <typename T>
T* wsp(const Ctx& c, size_t off) {
    return (T*)(c.ws + off);
}

iabn_status validate_fwd(const Ctx& c, const void* x, void* z, const float* gamma,
                         const float* beta, float* rm, float* rv, float* sm, float* sv,
                         float momentum, float eps, float slope, uint32_t flags, int64_t m_global) {
    IABN_TRY(check_act("x", x));
    IABN_TRY(check_act("z", z));
    IABN_TRY(check_same_or_disjoint("x", x, "z", z, (size_t)c.g.E * c.g.b));
    if (!gamma || !beta) return fail(IABN_ERR_INVALID_ARG, "gamma/beta is NULL");
    IABN_TRY(check_scalars(eps, slope));
    if (flags & IABN_EVAL) {
        if (!rm || !rv) return fail(IABN_ERR_INVALID_ARG, "eval mode needs running_mean/var");
        return IABN_OK;
    }
    IABN_TRY(check_momentum(momentum));
    if (!sm || !sv) return fail(IABN_ERR_INVALID_ARG, "save_mean/save_var is NULL");
    if ((rm == nullptr) != (rv == nullptr))
        return fail(IABN_ERR_INVALID_ARG, "running_mean and running_var must both be given or both NULL");
    if (m_global < 2)
        return fail(IABN_ERR_DEGENERATE, "training needs >= 2 values per channel (got %lld)",
                    (long long)m_global);
    return IABN_OK;
}

iabn_status validate_bwd(const Ctx& c, const void* z, const void* dz, void* dx,
                         const float* gamma, const float* beta, const float* sv, float* dg,
                         float* db, float eps, float slope) {
    IABN_TRY(check_act("z", z));
    IABN_TRY(check_act("dz", dz));
    IABN_TRY(check_act("dx", dx));
    const size_t bytes = (size_t)c.g.E * c.g.b;
    IABN_TRY(check_same_or_disjoint("dz", dz, "dx", dx, bytes));
    IABN_TRY(check_disjoint("z", z, "dx", dx, bytes));
    if (!gamma || !beta || !sv || !dg || !db)
        return fail(IABN_ERR_INVALID_ARG, "gamma/beta/save_var/dgamma/dbeta is NULL");
    IABN_TRY(check_scalars(eps, slope));
    return IABN_OK;
}

template <typename T>
iabn_status fwd_stream_stats(const Ctx& c, const void* x) {
    return launch_stats<T>(c.g, c.S, x, wsp<double>(c, c.w.part), c.st);
}

template <typename T>
iabn_status fwd_from_partials(const Ctx& c, const double* part, int S, const void* x, void* z,
                              const float* gamma, const float* beta, float* rm, float* rv,
                              float* sm, float* sv, float momentum, float eps, float slope,
                              uint32_t flags) {
    FwdCoefArgs a{part, S, c.g.C, gamma, beta, rm, rv, sm, sv, wsp<float4>(c, c.w.coef),
                  momentum, eps, flags};
    launch_pdl(fwd_coef_kernel, wgrid(c.g.C), 128, 0, c.st, a);
    IABN_TRY(check_launch("fwd_coef kernel"));
    return launch_fwd_apply<T>(c.g, x, z, wsp<float4>(c, c.w.coef), slope, c.dev->sms, c.st);
}

// arguments of the channel-resident kernels (one rank; launch_fused fills the plan)
FusedArgs fused_fwd_args(const Geom& g, const void* x, void* z, const float* gamma,
                         const float* beta, float* rm, float* rv, float* sm, float* sv,
                         float momentum, float eps, float slope, uint32_t flags) {
    FusedArgs a{};
    a.in0 = x;
    a.out = z;
    a.gamma = gamma;
    a.beta = beta;
    a.running_mean = rm;
    a.running_var = rv;
    a.save_mean = sm;
    a.save_var = sv;
    a.C = g.C;
    a.HW = g.HW;
    a.m = (uint32_t)g.m;
    a.fd_hw = fd32(g.HW);
    a.momentum = momentum;
    a.eps = eps;
    a.slope = slope;
    a.inv_slope = 1.0f / slope;
    a.flags = flags;
    return a;
}
FusedArgs fused_bwd_args(const Geom& g, const void* z, const void* dz, void* dx,
                         const float* gamma, const float* beta, const float* sv, float* dg,
                         float* db, float eps, float slope, uint32_t flags) {
    FusedArgs a{};
    a.in0 = z;
    a.in1 = dz;
    a.out = dx;
    a.gamma = gamma;
    a.beta = beta;
    a.save_var = const_cast<float*>(sv);
    a.dgamma = dg;
    a.dbeta = db;
    a.C = g.C;
    a.HW = g.HW;
    a.m = (uint32_t)g.m;
    a.fd_hw = fd32(g.HW);
    a.eps = eps;
    a.slope = slope;
    a.inv_slope = 1.0f / slope;
    a.flags = flags;
    return a;
}

// ====================================================================== in-kernel exchange
void set_sync(FusedArgs& a, const SyncBuf& b, int vranks, int nranks, int rank0, uint32_t qv,
              int64_t vr_elems, double inv_mg) {
    a.qv = qv;
    a.vranks = (uint32_t)vranks;
    a.nranks = (uint32_t)nranks;
    a.rank0 = (uint32_t)rank0;
    a.vr_elems = vr_elems;
    a.sync_ctr = b.ctr;
    a.sync_cap = b.cap;
    a.inv_mg = inv_mg;
    for (int i = 0; i < kMaxRanks; ++i) a.peer[i] = b.peer[i];
}

// One-GPU emulation: the G ranks' buffers in one local allocation, per (device, stream)
// (calls on one stream are ordered; the call counter lives with the buffers).  Grows
// with C; a change of G or C reallocates after synchronising the stream, so the first
// emulated call of a shape must not be inside a CUDA-graph capture.
iabn_status emu_sync_buf(cudaStream_t st, int G, int64_t C, SyncBuf* out) {
    struct Ent {
        int dev;
        cudaStream_t st;
        SyncBuf b;
        void* base;
    };
    static std::mutex mu;
    static std::vector<Ent> ents;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(IABN_ERR_CUDA, "cudaGetDevice failed");
    std::lock_guard<std::mutex> lk(mu);
    Ent* e = nullptr;
    for (auto& x : ents)
        if (x.dev == dev && x.st == st) e = &x;
    if (e && e->b.nranks == G && e->b.cap >= C) {
        *out = e->b;
        return IABN_OK;
    }
    if (!e) {
        ents.push_back(Ent{dev, st, SyncBuf{}, nullptr});
        e = &ents.back();
    } else if (e->base) {
        cudaStreamSynchronize(st);
        cudaFree(e->base);
        e->base = nullptr;
        e->b = SyncBuf{};
    }
    const uint32_t cap = (uint32_t)std::max<int64_t>(C, 256);
    const size_t per = (size_t)2 * cap * G;  // records per rank buffer
    const size_t bytes = 64 + (size_t)G * per * sizeof(PeerRec);
    void* base = nullptr;
    if (cudaMalloc(&base, bytes) != cudaSuccess)
        return fail(IABN_ERR_CUDA, "exchange buffers (%zu bytes): %s", bytes,
                    cudaGetErrorString(cudaGetLastError()));
    static const unsigned long long init[2] = {1ull, 0ull};
    if (cudaMemsetAsync(base, 0, bytes, st) != cudaSuccess ||
        cudaMemcpyAsync(base, init, sizeof(init), cudaMemcpyHostToDevice, st) != cudaSuccess) {
        cudaFree(base);
        return fail(IABN_ERR_CUDA, "exchange buffers init: %s", cudaGetErrorString(cudaGetLastError()));
    }
    e->base = base;
    e->b.ctr = (unsigned long long*)base;
    e->b.cap = cap;
    e->b.nranks = G;
    for (int g = 0; g < G; ++g) e->b.peer[g] = (PeerRec*)((char*)base + 64) + (size_t)g * per;
    *out = e->b;
    return IABN_OK;
}

// ====================================================================== other activations
// BN + sigmoid / tanh (kernels_act.cuh): the streaming schedule only.
uint32_t act_of(uint32_t flags) { return flags & (IABN_ACT_SIGMOID | IABN_ACT_TANH); }

iabn_status check_act_flags(const Geom& g, uint32_t flags) {
    const uint32_t a = act_of(flags);
    if (!a) return IABN_OK;
    if (a == (IABN_ACT_SIGMOID | IABN_ACT_TANH))
        return fail(IABN_ERR_INVALID_ARG, "IABN_ACT_SIGMOID and IABN_ACT_TANH are exclusive");
    if (g.dtype != IABN_F32)
        return fail(IABN_ERR_UNSUPPORTED,
                    "sigmoid / tanh need fp32 storage (their inverse is ill-conditioned on an "
                    "8-bit mantissa)");
    return IABN_OK;
}

template <int ACT>
iabn_status act_elementwise(const Geom& g, int pass, const float* in0, const float* in1,
                            float* out, const float4* coef, int sms, cudaStream_t st) {
    const int64_t spc = samples_per_chunk(g);
    if (spc <= 0) return fail(IABN_ERR_UNSUPPORTED, "sample too large for the streaming apply");
    const FastDiv fh = fd32(g.HW), fc = fd32(g.C);
    for (int64_t n0 = 0; n0 < g.N; n0 += spc) {
        const int64_t nn = std::min(spc, g.N - n0);
        const int64_t off = n0 * g.C * g.HW;
        const uint32_t E = (uint32_t)(nn * g.C * g.HW);
        const int grid = apply_grid(E, 4, sms);
        const bool al = g.layout == IABN_NCHW ? g.HW % 4 == 0 : g.C % 4 == 0;
        const int fixed = g.layout == IABN_NHWC && al
                              ? nhwc_grid(g, E / 4, sms, blocks_per_sm(pass == 0 ? (const void*)act_apply_fixed_kernel<ACT, 0>
                                                                                 : (const void*)act_apply_fixed_kernel<ACT, 1>))
                              : 0;
        const float *a = in0 + off, *b = in1 ? in1 + off : nullptr;
        float* o = out + off;
#define IABN_ACT_LAUNCH(P, LY, AL) \
    launch_pdl(act_apply_kernel<ACT, P, LY, AL>, grid, kThreads, 0, st, a, b, o, coef, E, fh, fc)
        if (pass == 0) {
            if (g.layout == IABN_NCHW) { if (al) IABN_ACT_LAUNCH(0, 0, true); else IABN_ACT_LAUNCH(0, 0, false); }
            else if (fixed) launch_pdl(act_apply_fixed_kernel<ACT, 0>, fixed, kThreads, 0, st, a, b, o, coef, E, fh, fc);
            else { if (al) IABN_ACT_LAUNCH(0, 1, true); else IABN_ACT_LAUNCH(0, 1, false); }
        } else {
            if (g.layout == IABN_NCHW) { if (al) IABN_ACT_LAUNCH(1, 0, true); else IABN_ACT_LAUNCH(1, 0, false); }
            else if (fixed) launch_pdl(act_apply_fixed_kernel<ACT, 1>, fixed, kThreads, 0, st, a, b, o, coef, E, fh, fc);
            else { if (al) IABN_ACT_LAUNCH(1, 1, true); else IABN_ACT_LAUNCH(1, 1, false); }
        }
#undef IABN_ACT_LAUNCH
        IABN_TRY(check_launch(pass == 0 ? "act_fwd_apply kernel" : "act_bwd_apply kernel"));
    }
    return IABN_OK;
}

template <int ACT>
iabn_status act_reduce(const Geom& g, int S, const float* z, const float* dz, const float* gamma,
                       const float* beta, float eps, uint32_t flags, double* part, cudaStream_t st) {
    if (g.layout == IABN_NCHW && g.HW % 4 == 0)
        launch_pdl(act_bwd_reduce_nchw_kernel<ACT, true>, dim3((unsigned)g.C, (unsigned)S), kThreads, 0, st,
            z, dz, gamma, beta, g.C, (uint32_t)g.HW, (uint32_t)g.m, fd32(g.HW / 4), eps, flags, part);
    else if (g.layout == IABN_NCHW)
        launch_pdl(act_bwd_reduce_nchw_kernel<ACT, false>, dim3((unsigned)g.C, (unsigned)S), kThreads, 0, st,
            z, dz, gamma, beta, g.C, (uint32_t)g.HW, (uint32_t)g.m, fd32(g.HW), eps, flags, part);
    else if (g.C % 4 == 0)
        launch_pdl(act_bwd_reduce_nhwc_kernel<ACT>, dim3((unsigned)((g.C + 63) / 64), (unsigned)S), kThreads, 0, st,
            z, dz, gamma, beta, g.C, g.m, eps, flags, part);
    else
        launch_pdl(act_bwd_reduce_nhwc_scalar_kernel<ACT>, dim3((unsigned)((g.C + 31) / 32), (unsigned)S), kThreads, 0, st,
            z, dz, gamma, beta, g.C, g.m, eps, flags, part);
    return check_launch("act_bwd_reduce kernel");
}

template <typename T>
iabn_status bwd_from_sums(const Ctx& c, const double* glob, int Sg, const double* loc, int Sl,
                          const double* count_ptr, double count, const void* z, const void* dz,
                          void* dx, const float* gamma, const float* beta, const float* sv,
                          float* dg, float* db, float eps, float slope, uint32_t flags) {
    BwdCoefArgs a{glob, Sg, loc, Sl, count_ptr, count, c.g.C, gamma, beta, sv, dg, db,
                  wsp<float4>(c, c.w.coef), eps, flags};
    launch_pdl(bwd_coef_kernel, wgrid(c.g.C), 128, 0, c.st, a);
    IABN_TRY(check_launch("bwd_coef kernel"));
    return launch_bwd_apply<T>(c.g, z, dz, dx, wsp<float4>(c, c.w.coef), slope, c.dev->sms, c.st);
}

// One dispatch for every activation (ACT 0 leaky ReLU, 1 sigmoid, 2 tanh; ACT != 0 only
// with T = float): register-resident small layers -> channel-resident clusters (NCHW) ->
// channel groups (NHWC) -> [leaky: grid-resident NHWC, opt-in] -> streaming.
template <typename T, int ACT>
iabn_status forward_sched(const Ctx& c, const void* x, void* z, const float* gamma,
                          const float* beta, float* rm, float* rv, float* sm, float* sv,
                          float momentum, float eps, float slope, uint32_t flags) {
    if (flags & IABN_EVAL) {
        if constexpr (ACT == 0) {  // one launch: the apply derives its coefficients (EvalCoef)
            return launch_fwd_apply_ev<T, true>(c.g, x, z, nullptr, slope, c.dev->sms, c.st,
                                                 EvalCoef{gamma, beta, rm, rv, eps, flags});
        } else {
            float4* coef = wsp<float4>(c, c.w.coef);
            launch_pdl(eval_coef_kernel, cgrid(c.g.C), 128, 0, c.st, c.g.C, gamma, beta, rm, rv,
                       eps, flags, coef);
            IABN_TRY(check_launch("eval_coef kernel"));
            return act_elementwise<ACT>(c.g, 0, (const float*)x, nullptr, (float*)z, coef,
                                        c.dev->sms, c.st);
        }
    }
    if (!(flags & (IABN_FORCE_STREAMING | IABN_FORCE_FUSED | IABN_FORCE_RESIDENT))) {
        const SmallPlan sp = small_plan(c.g, flags, c.dev->sms);
        if (sp.ok) {
            SmallArgs a{};
            a.in0 = x;
            a.out = z;
            a.gamma = gamma;
            a.beta = beta;
            a.running_mean = rm;
            a.running_var = rv;
            a.save_mean = sm;
            a.save_var = sv;
            a.momentum = momentum;
            a.eps = eps;
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.flags = flags;
            return launch_small<T, ACT>(0, c.g, sp, a, c.st);
        }
    }
    FusedPlan p;
    if (!(flags & IABN_FORCE_STREAMING)) p = fused_plan(c.g, 0, *c.dev, flags);
    if ((flags & IABN_FORCE_FUSED) && !p.ok && c.g.layout != IABN_NHWC)
        return fail(IABN_ERR_UNSUPPORTED, "channel-resident forward not possible for this shape");
    if (p.ok)
        return launch_fused<T, ACT>(0, p,
                                    fused_fwd_args(c.g, x, z, gamma, beta, rm, rv, sm, sv,
                                                   momentum, eps, slope, flags),
                                    c.st);
    if (!(flags & (IABN_FORCE_STREAMING | IABN_FORCE_RESIDENT))) {
        const NhwcPlan np = nhwc_plan(c.g, 0, *c.dev, flags);
        if (np.ok) {
            NhwcArgs a{};
            a.gamma = gamma;
            a.beta = beta;
            a.running_mean = rm;
            a.running_var = rv;
            a.save_mean = sm;
            a.save_var = sv;
            a.momentum = momentum;
            a.eps = eps;
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.flags = flags;
            return launch_nhwc<T, ACT>(0, c.g, np, a, x, nullptr, z, c.st);
        }
        if (flags & IABN_FORCE_FUSED)
            return fail(IABN_ERR_UNSUPPORTED, "channel-group NHWC forward not possible for this shape");
    }
    if constexpr (ACT == 0) {
        if (const int G = gres_grid(c.g, 0, flags, *c.dev)) {
            GresArgs a{};
            a.in0 = x;
            a.out = z;
            a.C = c.g.C;
            a.rows = c.g.m;
            a.cv = (uint32_t)(c.g.C * c.g.b / 16);
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.eps = eps;
            a.flags = flags;
            a.part = wsp<double>(c, c.w.part);
            a.coef = wsp<float4>(c, c.w.coef);
            a.fwd = FwdCoefArgs{a.part, G, c.g.C, gamma, beta, rm, rv, sm, sv, a.coef, momentum,
                                eps, flags};
            return launch_gres<T, 0>(c.g, G, a, c.st);
        }
    }
    IABN_TRY(fwd_stream_stats<T>(c, x));
    if constexpr (ACT == 0) {
        return fwd_from_partials<T>(c, wsp<double>(c, c.w.part), c.S, x, z, gamma, beta, rm, rv,
                                    sm, sv, momentum, eps, slope, flags);
    } else {
        float4* coef = wsp<float4>(c, c.w.coef);
        FwdCoefArgs a{wsp<double>(c, c.w.part), c.S, c.g.C, gamma, beta, rm, rv, sm, sv, coef,
                      momentum, eps, flags};
        launch_pdl(fwd_coef_kernel, wgrid(c.g.C), 128, 0, c.st, a);
        IABN_TRY(check_launch("fwd_coef kernel"));
        return act_elementwise<ACT>(c.g, 0, (const float*)x, nullptr, (float*)z, coef,
                                    c.dev->sms, c.st);
    }
}

template <typename T, int ACT>
iabn_status backward_sched(const Ctx& c, const void* z, const void* dz, void* dx,
                           const float* gamma, const float* beta, const float* sv, float* dg,
                           float* db, float eps, float slope, uint32_t flags) {
    if (!(flags & (IABN_FORCE_STREAMING | IABN_FORCE_FUSED | IABN_FORCE_RESIDENT))) {
        const SmallPlan sp = small_plan(c.g, flags, c.dev->sms);
        if (sp.ok) {
            SmallArgs a{};
            a.in0 = z;
            a.in1 = dz;
            a.out = dx;
            a.gamma = gamma;
            a.beta = beta;
            a.save_var = const_cast<float*>(sv);
            a.dgamma = dg;
            a.dbeta = db;
            a.eps = eps;
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.flags = flags;
            return launch_small<T, ACT>(1, c.g, sp, a, c.st);
        }
    }
    FusedPlan p;
    if (!(flags & IABN_FORCE_STREAMING)) p = fused_plan(c.g, 1, *c.dev, flags);
    if ((flags & IABN_FORCE_FUSED) && !p.ok && c.g.layout != IABN_NHWC)
        return fail(IABN_ERR_UNSUPPORTED, "channel-resident backward not possible for this shape");
    if (p.ok)
        return launch_fused<T, ACT>(1, p,
                                    fused_bwd_args(c.g, z, dz, dx, gamma, beta, sv, dg, db, eps,
                                                   slope, flags),
                                    c.st);
    if (!(flags & (IABN_FORCE_STREAMING | IABN_FORCE_RESIDENT))) {
        const NhwcPlan np = nhwc_plan(c.g, 1, *c.dev, flags);
        if (np.ok) {
            NhwcArgs a{};
            a.gamma = gamma;
            a.beta = beta;
            a.save_var = const_cast<float*>(sv);
            a.dgamma = dg;
            a.dbeta = db;
            a.eps = eps;
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.flags = flags;
            return launch_nhwc<T, ACT>(1, c.g, np, a, z, dz, dx, c.st);
        }
        if (flags & IABN_FORCE_FUSED)
            return fail(IABN_ERR_UNSUPPORTED, "channel-group NHWC backward not possible for this shape");
    }
    double* part = wsp<double>(c, c.w.part);
    if constexpr (ACT == 0) {
        if (const int G = gres_grid(c.g, 1, flags, *c.dev)) {
            GresArgs a{};
            a.in0 = z;
            a.in1 = dz;
            a.out = dx;
            a.C = c.g.C;
            a.rows = c.g.m;
            a.cv = (uint32_t)(c.g.C * c.g.b / 16);
            a.slope = slope;
            a.inv_slope = 1.0f / slope;
            a.eps = eps;
            a.flags = flags;
            a.gamma = gamma;
            a.beta = beta;
            a.part = part;
            a.coef = wsp<float4>(c, c.w.coef);
            a.bwd = BwdCoefArgs{part, G, part, G, nullptr, (double)c.g.m, c.g.C, gamma, beta, sv,
                                dg, db, a.coef, eps, flags};
            return launch_gres<T, 1>(c.g, G, a, c.st);
        }
        IABN_TRY(launch_bwd_reduce<T>(c.g, c.S, z, dz, gamma, beta, eps, slope, flags, part, c.st));
        return bwd_from_sums<T>(c, part, c.S, part, c.S, nullptr, (double)c.g.m, z, dz, dx, gamma,
                                beta, sv, dg, db, eps, slope, flags);
    } else {
        // NHWC: the bulk-ring reduction when it applies (c.S = its cluster records), else
        // the LDG act reductions (NHWC: within the workspace's 296 records)
        int S = c.S;
        if (c.g.layout == IABN_NHWC && nb_grid(c.g)) {
            const iabn_status st = launch_nb<float, 1, ACT>(c.g, S, z, dz, gamma, beta, eps, 1.f,
                                                            flags, part, c.st);
            IABN_TRY(st);
        } else {
            if (c.g.layout == IABN_NHWC) S = (int)std::min<int64_t>(stat_splits_ldg(c.g), kGresMaxG);
            IABN_TRY(act_reduce<ACT>(c.g, S, (const float*)z, (const float*)dz, gamma, beta, eps,
                                     flags, part, c.st));
        }
        float4* coef = wsp<float4>(c, c.w.coef);
        BwdCoefArgs a{part, S, part, S, nullptr, (double)c.g.m, c.g.C, gamma, beta, sv, dg, db,
                      coef, eps, flags};
        launch_pdl(bwd_coef_kernel, wgrid(c.g.C), 128, 0, c.st, a);
        IABN_TRY(check_launch("bwd_coef kernel"));
        return act_elementwise<ACT>(c.g, 1, (const float*)z, (const float*)dz, (float*)dx, coef,
                                    c.dev->sms, c.st);
    }
}

// sigmoid / tanh take slope = 1 (unused by their kernels) and fp32 storage only
// (check_act_flags rejects bf16 before any launch)
template <typename T>
iabn_status forward_impl(const Ctx& c, const void* x, void* z, const float* gamma,
                         const float* beta, float* rm, float* rv, float* sm, float* sv,
                         float momentum, float eps, float slope, uint32_t flags) {
    if constexpr (std::is_same<T, float>::value) {
        if (flags & IABN_ACT_SIGMOID)
            return forward_sched<T, 1>(c, x, z, gamma, beta, rm, rv, sm, sv, momentum, eps, 1.f, flags);
        if (flags & IABN_ACT_TANH)
            return forward_sched<T, 2>(c, x, z, gamma, beta, rm, rv, sm, sv, momentum, eps, 1.f, flags);
    }
    return forward_sched<T, 0>(c, x, z, gamma, beta, rm, rv, sm, sv, momentum, eps, slope, flags);
}

template <typename T>
iabn_status backward_impl(const Ctx& c, const void* z, const void* dz, void* dx,
                          const float* gamma, const float* beta, const float* sv, float* dg,
                          float* db, float eps, float slope, uint32_t flags) {
    if constexpr (std::is_same<T, float>::value) {
        if (flags & IABN_ACT_SIGMOID)
            return backward_sched<T, 1>(c, z, dz, dx, gamma, beta, sv, dg, db, eps, 1.f, flags);
        if (flags & IABN_ACT_TANH)
            return backward_sched<T, 2>(c, z, dz, dx, gamma, beta, sv, dg, db, eps, 1.f, flags);
    }
    return backward_sched<T, 0>(c, z, dz, dx, gamma, beta, sv, dg, db, eps, slope, flags);
}

// ====================================================================== fault injection
// Test-of-tests only (iabn_debug_fault, not in include/iabn.h): perturb one output of
// every call by a relative 1e-3 so that the GPU parity harness can be shown to fail.
std::atomic<uint32_t> g_fault{0};
enum : uint32_t { FAULT_DGAMMA = 1, FAULT_Z = 2, FAULT_DX = 4, FAULT_RUNNING_VAR = 8 };

__global__ void fault_scale_kernel(float* v, int64_t n) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) v[i] *= 1.001f;
}
__global__ void fault_act_kernel(void* a, int dtype) {
    if (dtype == IABN_F32) {
        float* f = (float*)a;  // well above the fp32 tolerance plus the R16 allowances
        f[0] = f[0] * 1.01f + 1e-2f;
    } else {
        __nv_bfloat16* h = (__nv_bfloat16*)a;  // bf16 tolerance is 2e-2: a larger step
        const float v = __bfloat162float(h[0]);
        h[0] = __float2bfloat16(v + 0.25f * fabsf(v) + 0.5f);
    }
}
iabn_status fault_after(iabn_status s, int dtype, void* act, float* vec, int64_t n, uint32_t vbit,
                        uint32_t abit, void* stream) {
    const uint32_t f = g_fault.load(std::memory_order_relaxed);
    if (s != IABN_OK || !f) return s;
    const cudaStream_t st = (cudaStream_t)stream;
    if ((f & vbit) && vec) fault_scale_kernel<<<1, 256, 0, st>>>(vec, n);
    if ((f & abit) && act) fault_act_kernel<<<1, 1, 0, st>>>(act, dtype);
    return check_launch("fault injection");
}

#define DISPATCH(dtype, fn, ...) \
    ((dtype) == IABN_F32 ? fn<float>(__VA_ARGS__) : fn<__nv_bfloat16>(__VA_ARGS__))

}  // namespace

// ====================================================================== C ABI
extern "C" {

int iabn_version(void) { return IABN_VERSION; }

const char* iabn_status_string(iabn_status s) {
    switch (s) {
        case IABN_OK: return "IABN_OK";
        case IABN_ERR_INVALID_ARG: return "IABN_ERR_INVALID_ARG";
        case IABN_ERR_UNSUPPORTED: return "IABN_ERR_UNSUPPORTED";
        case IABN_ERR_ALIAS: return "IABN_ERR_ALIAS";
        case IABN_ERR_DEGENERATE: return "IABN_ERR_DEGENERATE";
        case IABN_ERR_WORKSPACE: return "IABN_ERR_WORKSPACE";
        case IABN_ERR_CUDA: return "IABN_ERR_CUDA";
        case IABN_ERR_NCCL: return "IABN_ERR_NCCL";
    }
    return "IABN_ERR_UNKNOWN";
}

const char* iabn_last_error(void) { return g_err.c_str(); }

uint64_t iabn_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

// Experiments only (not in include/iabn.h): copy the phase trace of the last fused
// launch (IABN_FUSED_DEBUG & 4) to host memory; returns the number of values.
IABN_API size_t iabn_debug_trace(unsigned long long* host, size_t n) {
    if (!g_trace) return 0;
    const size_t k = n < g_trace_n ? n : g_trace_n;
    if (host && k) cudaMemcpy(host, g_trace, k * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return g_trace_n;
}
IABN_API uint32_t iabn_debug_trace_channels(void) { return g_trace_ch; }

// Test-of-tests only (not in include/iabn.h): 1 = dgamma x 1.001, 2 = z[0] perturbed,
// 4 = dx[0] perturbed, 8 = running_var x 1.001 on every later call; 0 = off.
IABN_API void iabn_debug_fault(uint32_t mask) { g_fault.store(mask); }

// Test hook only (not in include/iabn.h): force the NHWC channel-group plan -- g channels
// per group, K CTAs per cluster, at most `clusters` clusters launched (persistent loop
// over the groups); 0 = automatic.  Shapes the forced plan cannot take fall back as usual.
// Test hook only (not in include/iabn.h): the register-resident small-layer schedule --
// 1 = whenever the shape allows it (ignoring the size threshold), -1 = never, 0 = automatic.
IABN_API void iabn_debug_small(int on) { g_small_force.store(on); }
// test hook: record count of the NHWC bulk-ring reductions for this shape (0 = LDG kernels)
IABN_API int iabn_debug_nb_records(const iabn_desc* desc) {
    Geom g;
    if (make_geom(desc, &g) != IABN_OK) return -1;
    return nb_grid(g);
}
// ... and its slots per thread (4 or 8; 0 = automatic)
IABN_API void iabn_debug_small_r(int r) { g_small_force_r.store(r); }

// Test hook only (not in include/iabn.h): 1 if the last channel-resident launch drew its
// channels dynamically (ticket counter), 0 if it used the static order.
IABN_API int iabn_debug_last_dynamic(void) { return g_last_dyn.load(); }

IABN_API void iabn_debug_nhwc_plan(int g, int K, int clusters) {
    g_nhwc_force_g.store(g);
    g_nhwc_force_k.store(K);
    g_nhwc_force_clusters.store(clusters);
}

size_t iabn_workspace_bytes(const iabn_desc* desc) {
    Geom g;
    if (make_geom(desc, &g) != IABN_OK) return 0;
    // splits depend on the SM count; size for the largest B200-class count
    // without touching the device (callable without a GPU).
    return ws_layout(g, stat_splits(g)).total;
}

iabn_status iabn_query_schedule(const iabn_desc* desc, int pass, uint32_t flags, int* schedule,
                                int* cluster) {
    Geom g;
    IABN_TRY(make_geom(desc, &g));
    if (!schedule || !cluster) return fail(IABN_ERR_INVALID_ARG, "NULL output");
    if (pass != 0 && pass != 1) return fail(IABN_ERR_INVALID_ARG, "pass must be 0 or 1");
    DevFacts* dev;
    IABN_TRY(device_facts(&dev));
    if (act_of(flags)) {  // sigmoid / tanh: small / channel-resident (NCHW) or streaming
        IABN_TRY(check_act_flags(g, flags));
        if (!(flags & (IABN_FORCE_STREAMING | IABN_EVAL | IABN_FORCE_FUSED)) &&
            small_plan(g, flags, dev->sms).ok) {
            *schedule = 5;
            *cluster = 0;
            return IABN_OK;
        }
        FusedPlan p;
        if (!(flags & (IABN_FORCE_STREAMING | IABN_EVAL))) p = fused_plan(g, pass, *dev, flags);
        *schedule = p.ok ? 1 : 0;
        *cluster = p.ok ? p.K : 0;
        if (!p.ok && !(flags & (IABN_FORCE_STREAMING | IABN_EVAL))) {
            const NhwcPlan np = nhwc_plan(g, pass, *dev, flags);
            if (np.ok) {
                *schedule = 4;
                *cluster = (int)np.K;
            }
        }
        return IABN_OK;
    }
    if (!(flags & (IABN_FORCE_STREAMING | IABN_EVAL | IABN_FORCE_FUSED | IABN_FORCE_RESIDENT))) {
        const SmallPlan sp = small_plan(g, flags, dev->sms);
        if (sp.ok) {
            *schedule = 5;
            *cluster = 0;
            return IABN_OK;
        }
    }
    FusedPlan p;
    if (!(flags & (IABN_FORCE_STREAMING | IABN_EVAL)))
        p = fused_plan(g, pass, *dev, flags);
    *schedule = p.ok ? 1 : 0;
    *cluster = p.ok ? p.K : 0;
    if (!p.ok && !(flags & (IABN_FORCE_STREAMING | IABN_FORCE_RESIDENT))) {
        const NhwcPlan np = nhwc_plan(g, pass, *dev, flags);
        if (np.ok) {
            *schedule = 4;
            *cluster = (int)np.K;
        }
    }
    if (!p.ok && *schedule == 0 && gres_grid(g, pass, flags, *dev) > 0) *schedule = 3;
    return IABN_OK;
}

iabn_status iabn_forward(const iabn_desc* desc, const void* x, void* z, const float* gamma,
                         const float* beta, float* running_mean, float* running_var,
                         float* save_mean, float* save_var, float momentum, float eps,
                         float slope, uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(validate_fwd(c, x, z, gamma, beta, running_mean, running_var, save_mean, save_var,
                          momentum, eps, slope, flags, c.g.m));
    IABN_TRY(check_act_flags(c.g, flags));
    IABN_TRY(attach_device(c));
    return fault_after(DISPATCH(c.g.dtype, forward_impl, c, x, z, gamma, beta, running_mean,
                                running_var, save_mean, save_var, momentum, eps, slope, flags),
                       c.g.dtype, z, running_var, c.g.C, FAULT_RUNNING_VAR, FAULT_Z, stream);
}

iabn_status iabn_backward(const iabn_desc* desc, const void* z, const void* dz, void* dx,
                          const float* gamma, const float* beta, const float* save_mean,
                          const float* save_var, float* dgamma, float* dbeta, float eps,
                          float slope, uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
    (void)save_mean;  // BN* does not depend on mu_B
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(validate_bwd(c, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope));
    IABN_TRY(check_act_flags(c.g, flags));
    IABN_TRY(attach_device(c));
    return fault_after(DISPATCH(c.g.dtype, backward_impl, c, z, dz, dx, gamma, beta, save_var,
                                dgamma, dbeta, eps, slope, flags),
                       c.g.dtype, dx, dgamma, c.g.C, FAULT_DGAMMA, FAULT_DX, stream);
}

// ---------------------------------------------------------------- test time
iabn_status iabn_fold_conv(int64_t cout, int64_t k_per_out, const float* w, const float* bias,
                           const float* running_mean, const float* running_var,
                           const float* gamma, const float* beta, float eps, uint32_t flags,
                           float* w_out, float* bias_out, void* stream) {
    if (cout <= 0 || k_per_out <= 0)
        return fail(IABN_ERR_INVALID_ARG, "cout and k_per_out must be positive");
    if (cout > 0x7fffffffll) return fail(IABN_ERR_UNSUPPORTED, "cout too large");
    if (!w || !w_out || !running_mean || !running_var || !gamma || !beta || !bias_out)
        return fail(IABN_ERR_INVALID_ARG, "NULL required pointer");
    if (!(eps > 0.f) || !std::isfinite(eps))
        return fail(IABN_ERR_INVALID_ARG, "eps must be finite and > 0 (got %g)", (double)eps);
    if (!aligned16(w) || !aligned16(w_out))
        return fail(IABN_ERR_UNSUPPORTED, "w / w_out not 16-byte aligned");
    const size_t wb = (size_t)cout * (size_t)k_per_out * sizeof(float), cb = (size_t)cout * 4;
    IABN_TRY(check_same_or_disjoint("w", w, "w_out", w_out, wb));
    if (bias) IABN_TRY(check_same_or_disjoint("bias", bias, "bias_out", bias_out, cb));
    {
        const uintptr_t a0 = (uintptr_t)w_out, b0 = (uintptr_t)bias_out;
        if (a0 < b0 + cb && b0 < a0 + wb) return fail(IABN_ERR_ALIAS, "w_out and bias_out overlap");
    }
    DevFacts* dev = nullptr;
    IABN_TRY(device_facts(&dev));
    launch_pdl(fold_conv_kernel, (unsigned)cout, kThreads, 0, (cudaStream_t)stream,
        w, bias, running_mean, running_var, gamma, beta, eps, flags, k_per_out, w_out, bias_out);
    return check_launch("fold_conv kernel");
}

// ---------------------------------------------------------------- split phase
iabn_status iabn_forward_reduce(const iabn_desc* desc, const void* x, double* stats, void* ws,
                                size_t ws_bytes, void* stream) {
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(check_act("x", x));
    if (!stats) return fail(IABN_ERR_INVALID_ARG, "stats is NULL");
    IABN_TRY(attach_device(c));
    IABN_TRY(DISPATCH(c.g.dtype, fwd_stream_stats, c, x));
    launch_pdl(combine_kernel<3>, wgrid(c.g.C), 128, 0, c.st, wsp<double>(c, c.w.part), c.S, c.g.C, stats,
                                                      -1.0);
    return check_launch("combine kernel");
}

iabn_status iabn_forward_apply(const iabn_desc* desc, const void* x, void* z,
                               const double* stats_global, const float* gamma, const float* beta,
                               float* running_mean, float* running_var, float* save_mean,
                               float* save_var, float momentum, float eps, float slope,
                               uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    if (!stats_global) return fail(IABN_ERR_INVALID_ARG, "stats_global is NULL");
    // the global count is on the device; only the local one can be checked here
    IABN_TRY(validate_fwd(c, x, z, gamma, beta, running_mean, running_var, save_mean, save_var,
                          momentum, eps, slope, flags & ~(uint32_t)IABN_EVAL, 2));
    IABN_TRY(attach_device(c));
    return DISPATCH(c.g.dtype, fwd_from_partials, c, stats_global, 1, x, z, gamma, beta,
                    running_mean, running_var, save_mean, save_var, momentum, eps, slope, flags);
}

iabn_status iabn_backward_reduce(const iabn_desc* desc, const void* z, const void* dz,
                                 const float* gamma, const float* beta, double* sums, float eps,
                                 float slope, uint32_t flags, void* ws, size_t ws_bytes,
                                 void* stream) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(check_act("z", z));
    IABN_TRY(check_act("dz", dz));
    if (!gamma || !beta || !sums) return fail(IABN_ERR_INVALID_ARG, "gamma/beta/sums is NULL");
    IABN_TRY(check_scalars(eps, slope));
    IABN_TRY(attach_device(c));
    double* part = wsp<double>(c, c.w.part);
    IABN_TRY(DISPATCH(c.g.dtype, launch_bwd_reduce, c.g, c.S, z, dz, gamma, beta, eps, slope,
                      flags, part, c.st));
    launch_pdl(combine_kernel<2>, wgrid(c.g.C), 128, 0, c.st, part, c.S, c.g.C, sums, (double)c.g.m);
    return check_launch("combine kernel");
}

iabn_status iabn_backward_apply(const iabn_desc* desc, const void* z, const void* dz, void* dx,
                                const double* sums_global, const double* sums_local,
                                const float* gamma, const float* beta, const float* save_var,
                                float* dgamma, float* dbeta, float eps, float slope,
                                uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(validate_bwd(c, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope));
    if (!sums_global) return fail(IABN_ERR_INVALID_ARG, "sums_global is NULL");
    IABN_TRY(attach_device(c));
    const double* loc = (flags & IABN_SYNC_GLOBAL_PARAM_GRADS) || !sums_local ? sums_global
                                                                               : sums_local;
    return DISPATCH(c.g.dtype, bwd_from_sums, c, sums_global, 1, loc, 1, sums_global + 2 * c.g.C,
                    0.0, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope, flags);
}

// ---------------------------------------------------------------- synchronized
iabn_status iabn_comm_get_unique_id(unsigned char id[128]) {
    if (!id) return fail(IABN_ERR_INVALID_ARG, "id is NULL");
    Nccl* n = nccl();
    if (!n) return fail(IABN_ERR_NCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    ncclUniqueId u;
    const ncclResult_t r = n->GetUniqueId(&u);
    if (r != ncclSuccess) return fail(IABN_ERR_NCCL, "ncclGetUniqueId: %s", n->GetErrorString(r));
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, u.internal, 128);
    return IABN_OK;
}

iabn_status iabn_comm_init(iabn_comm* out, int nranks, int rank, const unsigned char id[128]) {
    if (!out || !id) return fail(IABN_ERR_INVALID_ARG, "NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(IABN_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
    Nccl* n = nccl();
    if (!n) return fail(IABN_ERR_NCCL, "NCCL unavailable: %s", g_nccl.why.c_str());
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclComm_t comm;
    const ncclResult_t r = n->CommInitRank(&comm, nranks, u, rank);
    if (r != ncclSuccess) return fail(IABN_ERR_NCCL, "ncclCommInitRank: %s", n->GetErrorString(r));
    *out = new iabn_comm_s{comm, nranks, rank};
    return IABN_OK;
}

iabn_status iabn_comm_destroy(iabn_comm comm) {
    if (!comm) return IABN_OK;
    Nccl* n = nccl();
    iabn_status s = IABN_OK;
    if (n) {
        const ncclResult_t r = n->CommDestroy(comm->comm);
        if (r != ncclSuccess) s = fail(IABN_ERR_NCCL, "ncclCommDestroy: %s", n->GetErrorString(r));
    }
    if (comm->own) {
        cudaDeviceSynchronize();
        for (int g = 0; g < comm->nranks; ++g)
            if (g != comm->rank && comm->sb.peer[g]) cudaIpcCloseMemHandle(comm->sb.peer[g]);
        cudaFree(comm->own);
    }
    if (comm->sb.ctr) cudaFree(comm->sb.ctr);
    for (auto& pe : comm->ev)
        for (cudaEvent_t e : pe)
            if (e) cudaEventDestroy(e);
    delete comm;
    return s;
}

iabn_status iabn_comm_set_timing(iabn_comm comm, int on) {
    if (!comm) return fail(IABN_ERR_INVALID_ARG, "comm is NULL");
    comm->timing = on != 0;
    comm->timed[0] = comm->timed[1] = false;
    return IABN_OK;
}

iabn_status iabn_comm_phase_ms(iabn_comm comm, float ms[6]) {
    if (!comm || !ms) return fail(IABN_ERR_INVALID_ARG, "NULL argument");
    for (int pass = 0; pass < 2; ++pass) {
        for (int k = 0; k < 3; ++k) ms[3 * pass + k] = -1.f;
        if (!comm->timed[pass]) continue;
        const cudaError_t e = cudaEventSynchronize(comm->ev[pass][3]);
        if (e != cudaSuccess) return fail(IABN_ERR_CUDA, "cudaEventSynchronize: %s", cudaGetErrorString(e));
        for (int k = 0; k < 3; ++k) {
            float t = 0.f;
            if (cudaEventElapsedTime(&t, comm->ev[pass][k], comm->ev[pass][k + 1]) != cudaSuccess)
                return fail(IABN_ERR_CUDA, "cudaEventElapsedTime failed");
            ms[3 * pass + k] = t;
        }
    }
    return IABN_OK;
}

iabn_status iabn_forward_sync(const iabn_desc* desc, const void* x, void* z, const float* gamma,
                              const float* beta, float* running_mean, float* running_var,
                              float* save_mean, float* save_var, float momentum, float eps,
                              float slope, uint32_t flags, void* ws, size_t ws_bytes,
                              void* stream, iabn_comm comm) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    if (!comm) return fail(IABN_ERR_INVALID_ARG, "comm is NULL");
    if (comm->nranks == 1 || (flags & IABN_EVAL))
        return iabn_forward(desc, x, z, gamma, beta, running_mean, running_var, save_mean,
                            save_var, momentum, eps, slope, flags, ws, ws_bytes, stream);
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    // global count >= nranks * 1 >= 2
    IABN_TRY(validate_fwd(c, x, z, gamma, beta, running_mean, running_var, save_mean, save_var,
                          momentum, eps, slope, flags, c.g.m * comm->nranks));
    IABN_TRY(attach_device(c));
    if (sync_fused_wanted(flags)) {
        // channel-resident kernel with the exchange inside, if every rank can run it with
        // the same plan (else every rank takes the all-reduce path below)
        const FusedPlan p = fused_plan(c.g, 0, *c.dev, flags);
        SyncAgree ag;
        IABN_TRY(sync_agree(comm, c.g, 0, p, c.st, &ag));
        if (ag.fused) {
            IABN_TRY(comm_sync_buf(comm, c.g.C, c.st));
            FusedArgs a = fused_fwd_args(c.g, x, z, gamma, beta, running_mean, running_var,
                                         save_mean, save_var, momentum, eps, slope, flags);
            set_sync(a, comm->sb, 1, comm->nranks, comm->rank, (uint32_t)p.clusters, 0, 0.0);
            phase_mark(comm, 0, 0, c.st);
            IABN_TRY(DISPATCH(c.g.dtype, launch_fused, 0, p, a, c.st));
            for (int k = 1; k <= 3; ++k) phase_mark(comm, 0, k, c.st);
            return fault_after(IABN_OK, c.g.dtype, z, running_var, c.g.C, FAULT_RUNNING_VAR,
                               FAULT_Z, stream);
        }
    }
    double* stats = wsp<double>(c, c.w.stats);
    phase_mark(comm, 0, 0, c.st);
    IABN_TRY(DISPATCH(c.g.dtype, fwd_stream_stats, c, x));
    launch_pdl(combine_kernel<3>, wgrid(c.g.C), 128, 0, c.st, wsp<double>(c, c.w.part), c.S, c.g.C, stats,
                                                      -1.0);
    IABN_TRY(check_launch("combine kernel"));
    phase_mark(comm, 0, 1, c.st);
    IABN_TRY(allreduce_f64(stats, (size_t)c.g.C * 3, comm, c.st));
    phase_mark(comm, 0, 2, c.st);
    IABN_TRY(DISPATCH(c.g.dtype, fwd_from_partials, c, stats, 1, x, z, gamma, beta, running_mean,
                      running_var, save_mean, save_var, momentum, eps, slope, flags));
    phase_mark(comm, 0, 3, c.st);
    return fault_after(IABN_OK, c.g.dtype, z, running_var, c.g.C, FAULT_RUNNING_VAR, FAULT_Z,
                       stream);
}

iabn_status iabn_backward_sync(const iabn_desc* desc, const void* z, const void* dz, void* dx,
                               const float* gamma, const float* beta, const float* save_mean,
                               const float* save_var, float* dgamma, float* dbeta, float eps,
                               float slope, uint32_t flags, void* ws, size_t ws_bytes,
                               void* stream, iabn_comm comm) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    if (!comm) return fail(IABN_ERR_INVALID_ARG, "comm is NULL");
    if (comm->nranks == 1)
        return iabn_backward(desc, z, dz, dx, gamma, beta, save_mean, save_var, dgamma, dbeta,
                             eps, slope, flags, ws, ws_bytes, stream);
    Ctx c;
    IABN_TRY(make_ctx(desc, ws, ws_bytes, stream, &c));
    IABN_TRY(validate_bwd(c, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope));
    IABN_TRY(attach_device(c));
    if (sync_fused_wanted(flags)) {
        const FusedPlan p = fused_plan(c.g, 1, *c.dev, flags);
        SyncAgree ag;
        IABN_TRY(sync_agree(comm, c.g, 1, p, c.st, &ag));
        if (ag.fused) {
            IABN_TRY(comm_sync_buf(comm, c.g.C, c.st));
            FusedArgs a = fused_bwd_args(c.g, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps,
                                         slope, flags);
            set_sync(a, comm->sb, 1, comm->nranks, comm->rank, (uint32_t)p.clusters, 0,
                     1.0 / (double)ag.m_global);
            phase_mark(comm, 1, 0, c.st);
            IABN_TRY(DISPATCH(c.g.dtype, launch_fused, 1, p, a, c.st));
            for (int k = 1; k <= 3; ++k) phase_mark(comm, 1, k, c.st);
            return fault_after(IABN_OK, c.g.dtype, dx, dgamma, c.g.C, FAULT_DGAMMA, FAULT_DX,
                               stream);
        }
    }
    double* part = wsp<double>(c, c.w.part);
    double* loc = wsp<double>(c, c.w.sums_loc);
    double* glob = wsp<double>(c, c.w.sums_glob);
    phase_mark(comm, 1, 0, c.st);
    IABN_TRY(DISPATCH(c.g.dtype, launch_bwd_reduce, c.g, c.S, z, dz, gamma, beta, eps, slope,
                      flags, part, c.st));
    launch_pdl(combine_kernel<2>, wgrid(c.g.C), 128, 0, c.st, part, c.S, c.g.C, loc, (double)c.g.m);
    IABN_TRY(check_launch("combine kernel"));
    const size_t nb = (size_t)(2 * c.g.C + 1) * sizeof(double);
    const cudaError_t e = cudaMemcpyAsync(glob, loc, nb, cudaMemcpyDeviceToDevice, c.st);
    if (e != cudaSuccess) return fail(IABN_ERR_CUDA, "cudaMemcpyAsync: %s", cudaGetErrorString(e));
    phase_mark(comm, 1, 1, c.st);
    IABN_TRY(allreduce_f64(glob, (size_t)(2 * c.g.C + 1), comm, c.st));
    phase_mark(comm, 1, 2, c.st);
    const double* lsrc = (flags & IABN_SYNC_GLOBAL_PARAM_GRADS) ? glob : loc;
    IABN_TRY(DISPATCH(c.g.dtype, bwd_from_sums, c, glob, 1, lsrc, 1, glob + 2 * c.g.C, 0.0, z, dz,
                      dx, gamma, beta, save_var, dgamma, dbeta, eps, slope, flags));
    phase_mark(comm, 1, 3, c.st);
    return fault_after(IABN_OK, c.g.dtype, dx, dgamma, c.g.C, FAULT_DGAMMA, FAULT_DX, stream);
}

// ---------------------------------------------------------------- one-GPU emulation
// nranks shards of one tensor, the fused-collective sync in one cooperative launch
static iabn_status emu_ctx(const iabn_desc* desc, int nranks, void* ws, size_t ws_bytes,
                           void* stream, Ctx* c, Geom* gl) {
    if (!desc) return fail(IABN_ERR_INVALID_ARG, "desc is NULL");
    if (nranks < 1 || nranks > kMaxRanks)
        return fail(IABN_ERR_INVALID_ARG, "nranks must be in [1, %d] (got %d)", kMaxRanks, nranks);
    IABN_TRY(make_geom(desc, gl));
    iabn_desc gd = *desc;
    gd.n = desc->n * nranks;
    IABN_TRY(make_ctx(&gd, ws, ws_bytes, stream, c));
    if (gl->layout != IABN_NCHW)
        return fail(IABN_ERR_UNSUPPORTED, "fused-collective sync: NCHW only");
    return IABN_OK;
}

iabn_status iabn_forward_sync_emulated(const iabn_desc* desc, int nranks, const void* x, void* z,
                                       const float* gamma, const float* beta,
                                       float* running_mean, float* running_var, float* save_mean,
                                       float* save_var, float momentum, float eps, float slope,
                                       uint32_t flags, void* ws, size_t ws_bytes, void* stream) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    Ctx c;
    Geom gl;
    IABN_TRY(emu_ctx(desc, nranks, ws, ws_bytes, stream, &c, &gl));
    if (flags & IABN_EVAL) return fail(IABN_ERR_INVALID_ARG, "eval mode has no exchange");
    IABN_TRY(validate_fwd(c, x, z, gamma, beta, running_mean, running_var, save_mean, save_var,
                          momentum, eps, slope, flags, c.g.m));
    IABN_TRY(attach_device(c));
    const FusedPlan p = fused_plan(gl, 0, *c.dev, flags);
    if (!p.ok || p.max_clusters < nranks)
        return fail(IABN_ERR_UNSUPPORTED, "channel-resident forward not possible for this shard");
    SyncBuf sb;
    IABN_TRY(emu_sync_buf(c.st, nranks, gl.C, &sb));
    FusedArgs a = fused_fwd_args(gl, x, z, gamma, beta, running_mean, running_var, save_mean,
                                 save_var, momentum, eps, slope, flags);
    const uint32_t qv = (uint32_t)std::min<int64_t>(gl.C, p.max_clusters / nranks);
    set_sync(a, sb, nranks, nranks, 0, qv, gl.E, 0.0);
    return fault_after(DISPATCH(gl.dtype, launch_fused, 0, p, a, c.st), gl.dtype, z, running_var,
                       gl.C, FAULT_RUNNING_VAR, FAULT_Z, stream);
}

iabn_status iabn_backward_sync_emulated(const iabn_desc* desc, int nranks, const void* z,
                                        const void* dz, void* dx, const float* gamma,
                                        const float* beta, const float* save_mean,
                                        const float* save_var, float* dgamma, float* dbeta,
                                        float eps, float slope, uint32_t flags, void* ws,
                                        size_t ws_bytes, void* stream) {
    if (act_of(flags)) return fail(IABN_ERR_UNSUPPORTED, "sigmoid / tanh: iabn_forward / iabn_backward only");
    (void)save_mean;
    Ctx c;
    Geom gl;
    IABN_TRY(emu_ctx(desc, nranks, ws, ws_bytes, stream, &c, &gl));
    IABN_TRY(validate_bwd(c, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope));
    IABN_TRY(attach_device(c));
    const FusedPlan p = fused_plan(gl, 1, *c.dev, flags);
    if (!p.ok || p.max_clusters < nranks)
        return fail(IABN_ERR_UNSUPPORTED, "channel-resident backward not possible for this shard");
    SyncBuf sb;
    IABN_TRY(emu_sync_buf(c.st, nranks, gl.C, &sb));
    FusedArgs a = fused_bwd_args(gl, z, dz, dx, gamma, beta, save_var, dgamma, dbeta, eps, slope,
                                 flags);
    const uint32_t qv = (uint32_t)std::min<int64_t>(gl.C, p.max_clusters / nranks);
    set_sync(a, sb, nranks, nranks, 0, qv, gl.E, 1.0 / ((double)gl.m * nranks));
    return fault_after(DISPATCH(gl.dtype, launch_fused, 1, p, a, c.st), gl.dtype, dx, dgamma,
                       gl.C * nranks, FAULT_DGAMMA, FAULT_DX, stream);
}

}  // extern "C"
