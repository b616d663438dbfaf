// kernels_fused.cuh -- channel-resident schedule (NCHW, HW*b a multiple of 16 B).
//
// A persistent grid of thread-block CLUSTERS of K CTAs (K chosen so clusters
// pack onto the GPCs).  Cluster q owns channels c = q, q + Q, ...; CTA r of the
// cluster owns the same channel-space slice [lo_r, hi_r) of each of them (the m
// = N*HW values of a channel are N planes of HW contiguous values, plane stride
// C*HW).  Each CTA is a warp-specialised pipeline:
//
//   producer warp : TMA bulk copies (cp.async.bulk, SASS UBLKCP) of slice t
//                   into slab buffer t % nbuf of a shared-memory ring, one
//                   mbarrier per chunk ("full");
//   reduce warps  : fp32x2 partial sums (FFMA2/FADD2) over the resident slice,
//                   fp64 CTA record, PUSHED into every peer's shared memory
//                   (DSMEM st.shared::cluster + remote mbarrier arrive);
//   exchange warp : waits for the K records of channel s in its own shared
//                   memory, folds them in rank order (deterministic, identical
//                   in every CTA), derives the apply coefficients;
//   apply warps   : outputs of channel s from the still-resident slice with
//                   16-byte stores, then free the slab buffer ("empty").
//
// The exchange never touches L2, so a slice stays in shared memory only for
// load latency + one DSMEM round trip (Little's law: that residence time,
// times the HBM rate, is the shared memory the pipeline needs).
//
// HBM traffic is the minimum the method allows (vs 3*E*b / 5*E*b streaming):
//   forward  (PASS 0): read x once, write z once          = 2*E*b
//   backward (PASS 1): read z and dz once, write dx once   = 3*E*b
#pragma once

#include <type_traits>

#include "common.cuh"
#include "kernels_act.cuh"
#include "kernels_stream.cuh"

namespace iabn {

constexpr int kMaxChunks = 16;  // chunks (mbarriers) per slab buffer
constexpr int kMaxBuf = 4;      // slab buffers per CTA (ring)
constexpr int kMaxCluster = 16; // CTAs per cluster (non-portable size above 8)
constexpr int kSlots = 4;       // in-flight channel records per CTA
constexpr int kMaxRanks = 8;    // ranks of the in-kernel exchange (one node)

// One rank's per-channel record in a peer's exchange buffer (synchronized variant):
// forward (count, sum x, sum x^2), backward (S1, S2 or Q).  Flag-in-word encoding (no
// fences): each double travels as two 8-byte words (32 value bits, 32 flag bits), each
// word stored and loaded as one single-copy-atomic access; a word is current when its
// flag is the call's flag, so the reader needs no release/acquire pair.
struct __align__(16) PeerRec {
    unsigned long long w[6];
};

struct FusedArgs {
    const void* in0;  // forward: x; backward: z
    const void* in1;  // backward: dz
    void* out;        // forward: z; backward: dx
    const float* gamma;
    const float* beta;
    float* running_mean;
    float* running_var;
    float* save_mean;
    float* save_var;  // forward: out; backward: in
    float* dgamma;
    float* dbeta;
    int64_t C, HW;
    uint32_t m;           // values per channel
    FastDiv fd_hw;
    uint32_t cap;         // 16-byte vectors reserved per input per buffer (>= slice)
    uint32_t chunk_vecs;  // vectors per chunk (per input)
    uint32_t nbuf;        // slab buffers in the ring (1..kMaxBuf)
    float momentum, eps, slope, inv_slope;
    uint32_t flags;
    // planes not 16-byte aligned (MIS kernels): each plane of the slice occupies W = mis_w
    // 16-byte slots holding the aligned range that covers it; hwb = HW * sizeof(T)
    uint32_t mis_w, hwb;
    FastDiv fd_w;
    // synchronized variant with the exchange inside the kernel (InPlace-ABN^sync,
    // PAPER.md:315): each rank's cluster record of channel c is stored into every rank's
    // buffer peer[g][(call & 1) * sync_cap + c][rank]; each CTA folds the nranks records
    // in rank order.  vranks > 1: the ranks' shards of one tensor in one launch (one-GPU
    // emulation: cluster i belongs to virtual rank i / qv, whose shard starts vr_elems
    // elements after the previous one); peer[] are then local buffers.
    uint32_t qv;          // clusters per rank in this launch: channel c -> cluster c % qv
    uint32_t vranks;      // ranks in this launch (1, or nranks)
    uint32_t nranks;      // ranks of the exchange (1 = no exchange)
    uint32_t rank0;       // rank of the launch's first virtual rank
    int64_t vr_elems;     // elements between consecutive virtual ranks' shards
    // [0] call number (starts at 1; identical on every rank: each rank makes the same
    // sequence of calls; read from device memory so that graph replays advance it),
    // [1] CTAs finished (the last one advances [0])
    unsigned long long* sync_ctr;
    uint32_t sync_cap;    // channels per parity half of a record buffer
    double inv_mg;        // backward: 1 / global count
    PeerRec* peer[kMaxRanks];
    uint32_t prefetch;  // L2 prefetch of each slice before its buffer frees up
    uint32_t debug;  // experiments only (IABN_FUSED_DEBUG): 4 = record phase timestamps
                     // into `trace`
    unsigned long long* trace;  // [grid][max_ch][8] %globaltimer ns (debug & 4)
    uint32_t trace_ch;          // channels per CTA recorded
    // dynamic channel scheduling: per (virtual) rank [2 vr] ticket counter, [2 vr + 1]
    // clusters finished; zero at launch, reset by the rank's last cluster; nullptr = static
    // (cluster q: q, q + Q, ..)
    unsigned int* dyn;
};
constexpr int kChanRing = 16;  // channel numbers in flight per CTA (dynamic scheduling)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// phase timestamps (debug & 4): 0 producer issued chunk 0, 1 producer issued last chunk,
// 2 reduce got chunk 0, 3 reduce got last chunk, 4 record pushed, 5 exchange gathered,
// 6 apply start, 7 apply end, 8 reduce loop done (thread 0), 9 group partials summed,
// 10 own record slots free (before the push), 11 coefficients published
constexpr int kTraceFields = 12;
#define IABN_TRACE(a, t, slot)                                                              \
    do {                                                                                    \
        if (((a).debug & 4u) && (t) < (a).trace_ch)                                        \
            (a).trace[((size_t)blockIdx.x * (a).trace_ch + (t)) * kTraceFields + (slot)] =  \
                gtimer();                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f64(uint32_t addr, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
// remote asynchronous store of 16 bytes into a peer's shared memory that signals the
// peer's mbarrier with complete_tx (no release fence on the pushing thread)
__device__ __forceinline__ void st_async_f64x2(uint32_t addr, double a, double b, uint32_t mbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(
            addr),
        "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(mbar)
        : "memory");
}
// arrive on a (possibly remote) mbarrier of this cluster.  Relaxed: no ordering of this thread's earlier memory operations (a write-after-read
// release whose reads are complete -- the values are in registers -- needs none, and a
// release would wait for the thread's outstanding global stores)
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr)
                 : "memory");
}
// wait with cluster-scope acquire: peers' DSMEM stores before their arrivals are visible
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAITC_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity), "n"(0x100000)
        : "memory");
}

// ---- cross-rank record exchange (peer memory over NVLink, or local memory in the
// one-GPU emulation): relaxed system-scope 8-byte accesses, flag in every word
__device__ __forceinline__ uint32_t rec_flag(unsigned long long call) {
    return 1u + (uint32_t)(call % 0xfffffffeull);  // never 0 (the buffers start zeroed)
}
template <int NR>
__device__ __forceinline__ void st_rec(PeerRec* d, const double* v, uint32_t flag) {
    const unsigned long long f = (unsigned long long)flag << 32;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        const unsigned long long lo = f | (uint32_t)__double2loint(v[k]);
        const unsigned long long hi = f | (uint32_t)__double2hiint(v[k]);
        asm volatile("st.relaxed.sys.global.v2.b64 [%0], {%1, %2};" ::"l"(d->w + 2 * k), "l"(lo),
                     "l"(hi)
                     : "memory");
    }
}
// all words of the record carry `flag`: decode into v, else false
template <int NR>
__device__ __forceinline__ bool ld_rec(const PeerRec* s, uint32_t flag, double* v) {
    bool ok = true;
#pragma unroll
    for (int k = 0; k < NR; ++k) {
        unsigned long long lo, hi;
        asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];" : "=l"(lo), "=l"(hi)
                     : "l"(s->w + 2 * k)
                     : "memory");
        ok = ok && (uint32_t)(lo >> 32) == flag && (uint32_t)(hi >> 32) == flag;
        v[k] = __hiloint2double((int)(uint32_t)hi, (int)(uint32_t)lo);
    }
    return ok;
}
// Slice of a channel owned by rank r of K, in 16-byte vectors: whole planes when
// there are at least K planes (each plane is then one bulk copy), else an even
// split of the channel's vectors.
__device__ __forceinline__ void cta_slice(uint32_t mv, uint32_t pv, uint32_t r, uint32_t K,
                                          uint32_t& vlo, uint32_t& vhi) {
    const uint32_t np = mv / pv;  // planes (N)
    if (np >= K) {
        vlo = pv * (uint32_t)((uint64_t)np * r / K);
        vhi = pv * (uint32_t)((uint64_t)np * (r + 1) / K);
    } else {
        vlo = (uint32_t)((uint64_t)mv * r / K);
        vhi = (uint32_t)((uint64_t)mv * (r + 1) / K);
    }
}

// Per-channel terms of the coefficients that do not depend on the sums.
struct Terms {
    double g, bet, rstd_b, inv_g;
};

// Per-channel constants of the apply pass (shared memory).
struct ApplyCoef {
    float2 P;   // forward: (A, A) ;           backward: z >= 0 branch (alpha, kappa)
    float2 Q;   // forward: (B', B') ;         backward: z < 0 branch (alpha a, kappa / a)
    float mu;   // forward: mu_hi ;            backward: cc
};

#ifndef IABN_REDUCE_WARPS
#define IABN_REDUCE_WARPS 3
#endif
#ifndef IABN_APPLY_WARPS
#define IABN_APPLY_WARPS 4
#endif
#ifndef IABN_RED_UNROLL
#define IABN_RED_UNROLL 8  // vectors per reduce-loop iteration (shared loads issued first)
#endif
#ifndef IABN_APP_UNROLL
#define IABN_APP_UNROLL 4  // vectors per apply-loop iteration
#endif
constexpr int kReduceWarps = IABN_REDUCE_WARPS;  // stream each resident slice for the channel sums
constexpr int kApplyWarps = IABN_APPLY_WARPS;    // stream it again, one channel behind, for outputs
// Warp roles.  The SMSP arbiter favours higher warp ids, so the order sets the
// priorities: IABN_WARP_ORDER 1 (default) = producer, exchange, apply, reduce (the
// reduce of the resident slice is the critical stage; the polling warps come last);
// 0 = reduce, apply, exchange, producer.
#ifndef IABN_WARP_ORDER
#define IABN_WARP_ORDER 1
#endif
constexpr int kWorkerWarps = kReduceWarps + kApplyWarps;
constexpr int kRU = IABN_RED_UNROLL, kAU = IABN_APP_UNROLL;
constexpr int kProducerWarp = IABN_WARP_ORDER ? 0 : kWorkerWarps + 1;  // TMA bulk copies
constexpr int kExchangeWarp = IABN_WARP_ORDER ? 1 : kWorkerWarps;      // folds the records
constexpr int kApplyWarp0 = IABN_WARP_ORDER ? 2 : kReduceWarps;
constexpr int kReduceWarp0 = IABN_WARP_ORDER ? 2 + kApplyWarps : 0;
constexpr int kFusedThreads = (kWorkerWarps + 2) * 32;

// named barrier over a worker group (id 1: reduce warps, 2: apply warps)
__device__ __forceinline__ void group_sync(uint32_t id, uint32_t nthr) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthr) : "memory");
}
// One warp of a group polls the mbarrier; the rest block on the group's named
// barrier (no issue slots burnt by a whole group of waiting warps).
__device__ __forceinline__ void group_wait(uint64_t* bar, uint32_t parity, bool leader, uint32_t id,
                                           uint32_t nthr) {
    if (leader) mbar_wait(bar, parity);
    group_sync(id, nthr);
}

// A plane of the MIS kernels: byte offset (in the tensor) of the aligned 16-byte range
// covering plane pgi = n*C + c, and the head bytes before the plane's first element.
struct MisPlane {
    uint64_t a0;
    uint32_t h;
};
__device__ __forceinline__ MisPlane mis_plane(uint64_t pgi, uint32_t hwb) {
    const uint64_t B = pgi * hwb;
    return {B & ~(uint64_t)15, (uint32_t)(B & 15)};
}
// element k of 16-byte slot i lies in the plane's bytes [h, h + hwb)
template <typename T>
__device__ __forceinline__ bool mis_valid(uint32_t i, int k, uint32_t h, uint32_t hwb) {
    const uint32_t byte = i * 16u + (uint32_t)k * (uint32_t)sizeof(T);
    return byte >= h && byte < h + hwb;
}

// one element of T from shared memory (byte address)
template <typename T>
__device__ __forceinline__ float lds_elem(uint32_t addr) {
    if constexpr (sizeof(T) == 4) {
        float v;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
        return v;
    } else {
        unsigned short h;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr));
        return __uint_as_float((uint32_t)h << 16);
    }
}

// MINB: CTAs per SM the register allocation must allow -- 2 (up to 113 registers,
// ~100 KB slabs: large channels) or 4 (up to 56 registers, ~50 KB slabs: small
// layers, where more resident pipelines hide the per-channel latency)
// MIS: planes not 16-byte aligned (e.g. bf16 14x14): covering ranges, masked edges
// ACT: 0 leaky ReLU (slope a), 1 sigmoid, 2 tanh (kernels_act.cuh; fp32 only):
// the reduce takes dy = f'(z) dz and y = f^-1(z) per element, the apply z = f(y) /
// dx = alpha dy + kappa y + cc; everything else (slabs, records, coefficients) is shared.
template <typename T, int PASS, int MINB, bool MIS = false, int ACT = 0>
__global__ void __launch_bounds__(kFusedThreads, MINB) fused_kernel(const FusedArgs a) {
    // ACT backward with large slabs (2 CTAs/SM): the reduce warps write (y, dy) back over
    // (z, dz) and the apply warps only combine them -- 32x256x56^2 fp32 sigmoid 76 -> 70 us;
    // with small slabs (4 CTAs/SM) the reduce warps are the bottleneck and the apply warps
    // invert again (the write-back measured 10-20 % slower there)
    constexpr bool WB = ACT != 0 && PASS == 1 && MINB == 2;
    constexpr int NIN = PASS == 0 ? 1 : 2;
    constexpr int NR = PASS == 0 ? 3 : 2;  // doubles per published record
    constexpr int V = Elem<T>::kVec;
    constexpr int NP = Pairs<T>::kN;
    extern __shared__ __align__(128) uint4 smem[];
    __shared__ __align__(8) uint64_t full[kMaxBuf][kMaxChunks];  // TMA -> reduce and apply warps
    __shared__ __align__(8) uint64_t empty[kMaxBuf][kMaxChunks]; // apply warps -> producer
    __shared__ __align__(8) uint64_t gathered[kSlots];           // K peers' records arrived
    __shared__ __align__(8) uint64_t slotfree[kSlots];           // K peers folded my record slot
    __shared__ __align__(8) uint64_t ready[2];                   // exchange -> apply warps
    __shared__ __align__(8) uint64_t freed[2];                   // apply warps -> exchange
    __shared__ __align__(16) double rec[kSlots][kMaxCluster][4];  // pushed by the K peers
    __shared__ double lrec[kSlots][3];                             // sync: this rank's totals
    __shared__ Terms lterm[kSlots];                                // sync: channel terms
    __shared__ double red[2][2][kReduceWarps];
    __shared__ ApplyCoef cs[2];
    __shared__ uint32_t chan_ring[kChanRing];               // channel of slot t (dynamic)
    __shared__ __align__(8) uint64_t chanbar[kChanRing];    // chan_ring[t % R] has landed

    const uint32_t K = cluster_nctarank(), r = cluster_ctarank();
    const uint32_t cid = blockIdx.x / K;       // cluster
    const uint32_t vr = cid / a.qv;            // virtual rank of this cluster (0 unless emulated)
    const uint32_t q = cid - vr * a.qv, Q = a.qv;
    const int64_t voff = (int64_t)vr * a.vr_elems;  // this rank's shard
    const uint32_t nbuf = a.nbuf;
    const uint32_t C = (uint32_t)a.C;
    const uint32_t nT = q < C ? (C - q + Q - 1) / Q : 0;  // channels of this cluster
    uint32_t vlo, vhi;
    if constexpr (MIS)  // whole planes of W slots each (the host ensures N >= K)
        cta_slice(a.m / (uint32_t)a.HW * a.mis_w, a.mis_w, r, K, vlo, vhi);
    else
        cta_slice(a.m / V, (uint32_t)a.HW / V, r, K, vlo, vhi);
    const uint32_t nv = vhi - vlo;
    const int nch = (int)((nv + a.chunk_vecs - 1) / a.chunk_vecs);
    const size_t bufv = (size_t)NIN * a.cap;  // vectors per slab buffer
    const uint32_t smem_u32 = smem_addr(smem);
    const uint32_t pv = (uint32_t)a.HW / V;  // vectors per plane
    // whole-plane slices and chunks (the usual case): plane-structured output addressing
    const bool plane_chunks = vlo % pv == 0 && a.chunk_vecs % pv == 0;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t apply_warps = kApplyWarps;

    if (threadIdx.x == 0) {
        for (uint32_t b = 0; b < nbuf; ++b) {
            for (int k = 0; k < nch; ++k) {
                mbar_init(&full[b][k], 1);
                mbar_init(&empty[b][k], apply_warps);
            }
        }
        for (int i = 0; i < kSlots; ++i) {
            mbar_init(&gathered[i], 1);  // own expect_tx; the K records arrive as transactions
            mbar_init(&slotfree[i], K);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&ready[i], 1);
            mbar_init(&freed[i], apply_warps);
        }
        for (int i = 0; i < kChanRing; ++i) mbar_init(&chanbar[i], 1);
        fence_mbar_init();
    }
    // every CTA's barriers are initialised before any peer may arrive on them
    cluster_arrive_release();
    cluster_wait_acquire();
    pdl_wait();  // the prologue above overlaps the previous kernel's tail

    // Channel of slot t.  Static: q + t Q.  Dynamic (a.dyn, one rank): cluster q starts
    // with channel q, then takes tickets Q + atomicAdd(dyn[0]) -- clusters that finish
    // early take more channels, so the grid's tail shrinks to about one channel (static
    // striding left CTAs idle for up to 8 % of the forward, profiles/r01_trace_phases_k8).
    // CTA 0's producer draws the ticket and stores it into every CTA's chan_ring with
    // st.async (complete_tx on chanbar); every role waits on chanbar before reading it.
    // C = no more channels.
    const bool dynamic = MINB == 2 && a.dyn != nullptr;  // compiled out of the small-slab variant
    auto chan_of = [&](uint32_t t) -> uint32_t {
        if (!dynamic) return t < nT ? q + t * Q : C;
        mbar_wait(&chanbar[t % kChanRing], (t / kChanRing) & 1u);
        return *(volatile uint32_t*)&chan_ring[t % kChanRing];
    };

    if (warp == kProducerWarp) {
        // ================================================ producer: slab t into buffer t % nbuf,
        // chunk by chunk: chunk k is refilled as soon as the apply warps released it.  The
        // bulk copies of a chunk (one per plane) are spread over the warp's lanes: small
        // layers have 16-64 planes per slice, issued serially they delay the first arrival
        // (r50s3 backward 35.1 -> 34.0 us).  Chunks of 1-3 planes stay on lane 0 (cfg4
        // backward 0.835 -> 0.839 ms with the whole warp in the loop).
        const uint64_t chunk_bytes = (uint64_t)a.chunk_vecs * 16u;
        const bool wide = !(a.debug & 8u) &&  // experiments: lane 0 issues all
                          (MIS ? a.chunk_vecs >= 4u * a.mis_w
                               : chunk_bytes >= 4u * (uint64_t)a.HW * sizeof(T));
        if (wide || lane == 0) {
            constexpr bool kL2Hints = MINB == 2;
            const uint32_t nl = wide ? 32u : 1u;  // lanes issuing copies
            const T* src[2] = {(const T*)a.in0 + voff, (const T*)a.in1 + voff};
            const uint32_t hw = (uint32_t)a.HW;
            uint32_t published = 0;  // dynamic: slots whose channel CTA 0 has stored
            bool exhausted = false;
            auto publish = [&](uint32_t u) {  // CTA 0, lane 0
                uint32_t c = C;
                if (!exhausted) {
                    c = u == 0 ? q : Q + atomicAdd(&a.dyn[2 * vr], 1u);
                    if (c >= C) {
                        c = C;
                        exhausted = true;
                    }
                }
                const uint32_t i = u % kChanRing;
                for (uint32_t j = 0; j < K; ++j)
                    asm volatile(
                        "st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                            mapa(&chan_ring[i], j)),
                        "r"(c), "r"(mapa(&chanbar[i], j))
                        : "memory");
            };
            for (uint32_t t = 0;; ++t) {
                uint32_t cu;
                if (dynamic) {
                    if (lane == 0) {
                        if (r == 0)  // one slot ahead: the peers' producers need not wait
                            while (published <= t + 1) publish(published++);
                        mbar_arrive_expect_tx(&chanbar[t % kChanRing], 4u);
                    }
                    cu = chan_of(t);
                } else {
                    cu = t < nT ? q + t * Q : C;
                }
                if (cu >= C) break;
                const uint32_t b = t % nbuf;
                const int64_t c = cu;
                uint4* buf = smem + b * bufv;
                // one decision per slice (not per copy: the producer lane issues one bulk
                // copy per plane, ~100 per slice on 14x14 layers)
                // (L2 hints only in the 2-CTA/SM variant, where single-buffered slices use
                // them: compiled out of the 4-CTA/SM one, measured ~3 % slower on r50s3 with)
                const bool hint_first =
                    kL2Hints && (((a.prefetch & 4u) && t >= nbuf) || (a.prefetch & 8u));
                if (lane == 0 && (a.prefetch & 1u) && t >= nbuf) {
                    // the slice's buffer is still being applied: pull the slice into L2 now,
                    // so that the bulk copies issued as its chunks free up hit L2 (HBM
                    // latency off the refill path; bytes read from HBM once either way)
                    if constexpr (MIS) {
                        for (uint32_t n = vlo / a.mis_w; n < vhi / a.mis_w; ++n) {
                            const MisPlane mp = mis_plane((uint64_t)n * a.C + c, a.hwb);
                            const uint32_t nb =
                                (uint32_t)(((mp.a0 + mp.h + a.hwb + 15) & ~(uint64_t)15) - mp.a0);
#pragma unroll
                            for (int i = 0; i < NIN; ++i)
                                bulk_prefetch_l2((const char*)src[i] + mp.a0, nb);
                        }
                    } else {
                        uint32_t j = vlo * V;
                        const uint32_t jend = vhi * V;
                        uint32_t n = fdiv(j, a.fd_hw);
                        uint32_t sp = j - n * hw;
                        while (j < jend) {
                            const uint32_t len = min(jend - j, hw - sp);
                            const int64_t goff = ((int64_t)n * a.C + c) * a.HW + sp;
#pragma unroll
                            for (int i = 0; i < NIN; ++i) {
                                if (kL2Hints && (a.prefetch & 2u))
                                    bulk_prefetch_l2_hint(src[i] + goff, len * (uint32_t)sizeof(T),
                                                          l2_policy_evict_last());
                                else
                                    bulk_prefetch_l2(src[i] + goff, len * (uint32_t)sizeof(T));
                            }
                            j += len;
                            ++n;
                            sp = 0;
                        }
                    }
                }
                for (int k = 0; k < nch; ++k) {
                    if (t >= nbuf) {
                        mbar_wait(&empty[b][k], (t / nbuf - 1) & 1u);  // chunk k of t - nbuf applied
                        fence_proxy_async_smem();  // generic-proxy reads before the async refill
                    }
                    const uint32_t c_lo = vlo + k * a.chunk_vecs;
                    const uint32_t c_hi = min(vhi, c_lo + a.chunk_vecs);
                    if (lane == 0 && k == 0) IABN_TRACE(a, t, 0);
                    if (lane == 0 && k == nch - 1) IABN_TRACE(a, t, 1);
                    if constexpr (MIS) {
                        // planes [n_lo, n_hi) of the chunk: copy each one's covering range
                        const uint32_t n_lo = c_lo / a.mis_w, n_hi = c_hi / a.mis_w;
                        uint32_t bytes = 0;
                        for (uint32_t n = n_lo + lane; lane < nl && n < n_hi; n += nl) {
                            const MisPlane mp = mis_plane((uint64_t)n * a.C + c, a.hwb);
                            bytes += (uint32_t)(((mp.a0 + mp.h + a.hwb + 15) & ~(uint64_t)15) - mp.a0);
                        }
                        if (wide) bytes = __reduce_add_sync(0xffffffffu, bytes);
                        if (lane == 0) mbar_arrive_expect_tx(&full[b][k], bytes * NIN);
                        if (wide) __syncwarp();
                        for (uint32_t n = n_lo + lane; lane < nl && n < n_hi; n += nl) {
                            const MisPlane mp = mis_plane((uint64_t)n * a.C + c, a.hwb);
                            const uint32_t nb =
                                (uint32_t)(((mp.a0 + mp.h + a.hwb + 15) & ~(uint64_t)15) - mp.a0);
#pragma unroll
                            for (int i = 0; i < NIN; ++i)
                                bulk_g2s(buf + (size_t)i * a.cap + (n * a.mis_w - vlo),
                                         (const char*)src[i] + mp.a0, nb, &full[b][k]);
                        }
                        continue;
                    }
                    if (lane == 0) mbar_arrive_expect_tx(&full[b][k], (c_hi - c_lo) * 16u * NIN);
                    if (wide) __syncwarp();
                    // one bulk copy per plane piece of the chunk
                    auto copy = [&](uint32_t j, uint32_t len, int64_t goff) {
#pragma unroll
                        for (int i = 0; i < NIN; ++i) {
                            if (hint_first)
                                bulk_g2s_hint(buf + (size_t)i * a.cap + (j / V - vlo), src[i] + goff,
                                              len * (uint32_t)sizeof(T), &full[b][k],
                                              l2_policy_evict_first());
                            else
                                bulk_g2s(buf + (size_t)i * a.cap + (j / V - vlo), src[i] + goff,
                                         len * (uint32_t)sizeof(T), &full[b][k]);
                        }
                    };
                    const uint32_t j0 = c_lo * V, jend = c_hi * V;  // channel-space elements
                    if (wide) {
                        // plane n holds [n * hw, (n + 1) * hw); lane l takes planes l, l + 32, ..
                        for (uint32_t n = fdiv(j0, a.fd_hw) + lane;; n += 32) {
                            const uint64_t ps = (uint64_t)n * hw;
                            if (ps >= jend) break;
                            const uint32_t j = ps > j0 ? (uint32_t)ps : j0;
                            const uint32_t len = (ps + hw < jend ? (uint32_t)(ps + hw) : jend) - j;
                            copy(j, len, ((int64_t)n * a.C + c) * a.HW + (j - (uint32_t)ps));
                        }
                    } else {
                        uint32_t j = j0;
                        uint32_t n = fdiv(j, a.fd_hw);
                        uint32_t sp = j - n * hw;
                        while (j < jend) {
                            const uint32_t len = min(jend - j, hw - sp);
                            copy(j, len, ((int64_t)n * a.C + c) * a.HW + sp);
                            j += len;
                            ++n;
                            sp = 0;
                        }
                    }
                }
            }
        }
        __syncwarp();
    } else if (warp == kExchangeWarp) {
        // ================================================ exchange: fold the K records of each
        // channel in rank order (bit-identical in all K CTAs)
        constexpr uint32_t RB = NR == 3 ? 32u : 16u;  // record bytes per peer
        // per-channel terms that do not depend on the records (lane 0)
        auto terms = [&](int64_t cp) {
            Terms t{0.0, 0.0, 0.0, 0.0};
            if (lane == 0) {
                t.g = gamma_eff(a.gamma[cp], a.eps, a.flags);
                t.inv_g = PASS == 1 ? 1.0 / t.g : 0.0;
                t.bet = (double)a.beta[cp];
                if (PASS == 1) t.rstd_b = rsqrt((double)a.save_var[cp] + (double)a.eps);
            }
            return t;
        };
        // fold: lane j < K takes rank j's record, then a fixed xor tree (the same order in
        // every CTA of the cluster => bit-identical coefficients)
        auto fold_cluster = [&](uint32_t rs, double* v) {
#pragma unroll
            for (int k = 0; k < NR; ++k) v[k] = lane < K ? rec[rs][lane][k] : 0.0;
#pragma unroll
            for (int k = 0; k < NR; ++k)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
        };
        // the slot of every peer that pushed into me may be reused by it: released as soon
        // as it is folded, with a relaxed arrive (a release would first wait for this
        // warp's outstanding global stores; measured: cfg2 69.4 -> 64.3 us fwd+bwd)
        auto release_slot = [&](uint32_t rs) {
            __syncwarp();
            if (lane < K) mbar_arrive_cluster_relaxed(mapa(&slotfree[rs], lane));
        };
        // coefficients of channel s from the totals v (global under sync) and this rank's
        // totals lv (lane 0)
        auto finish = [&](uint32_t s, int64_t cp, const Terms& t, double* v, double* lv) {
            const uint32_t slot = s & 1u;
            if (PASS == 0) {
                // mean, biased var; A = g rstd; y = (x - mu_hi) A + B'
                // (v[0] = the count, global under sync)
                const double inv_m = 1.0 / v[0];
                const double mean = v[1] * inv_m;
                double var = fma(-mean, mean, v[2] * inv_m);
                var = var > 0.0 ? var : 0.0;
                const double A = t.g * rsqrt(var + (double)a.eps);
                const float mu_hi = (float)mean;
                const double mu_lo = mean - (double)mu_hi;
                const float Af = (float)A, Bp = (float)(t.bet - mu_lo * A);
                cs[slot].P = make_float2(Af, Af);
                cs[slot].Q = make_float2(Bp, Bp);
                cs[slot].mu = mu_hi;
                mbar_arrive(&ready[slot]);  // release: cs[slot] visible to the apply warps
                IABN_TRACE(a, s, 11);
                if (r == 0 && vr == 0) {
                    a.save_mean[cp] = (float)mean;
                    a.save_var[cp] = (float)var;
                    update_running(a.running_mean, a.running_var, cp, mean, var, v[0],
                                   a.momentum, a.flags);
                }
            } else {
                // dx = alpha dy + kappa y + cc (PAPER.md:168 refolded in y):
                //   alpha = g rstd, kappa = -rstd S2/m, cc = rstd (S2 beta - g S1)/m
                // with dy, y on the branch of sign(z):
                //   z >= 0: alpha dz + kappa z + cc;  z < 0: (alpha a) dz + (kappa / a) z + cc
                // variant II pushed (S1, Q = sum dy y): S2 = (Q - beta S1) / g
                if (!(a.flags & kVariantI)) {
                    v[1] = (v[1] - t.bet * v[0]) * t.inv_g;
                    lv[1] = (lv[1] - t.bet * lv[0]) * t.inv_g;
                }
                const double rm = t.rstd_b * (a.nranks > 1 ? a.inv_mg : 1.0 / (double)a.m);
                const float alpha = (float)(t.g * t.rstd_b);
                const float kappa = (float)(-rm * v[1]);
                const float cc = (float)(rm * fma(v[1], t.bet, -t.g * v[0]));
                cs[slot].P = make_float2(alpha, kappa);
                cs[slot].Q = make_float2(alpha * a.slope, kappa * a.inv_slope);
                cs[slot].mu = cc;
                mbar_arrive(&ready[slot]);  // release: cs[slot] visible to the apply warps
                IABN_TRACE(a, s, 11);
                if (r == 0) {
                    // sync: this rank's sums unless the caller asked for the global ones (R7)
                    const double* pg = (a.flags & kSyncGlobalGrads) ? v : lv;
                    a.dbeta[vr * a.C + cp] = (float)pg[0];
                    a.dgamma[vr * a.C + cp] = (float)(gamma_sign(a.gamma[cp], a.flags) * pg[1]);
                }
            }
        };
        if (a.nranks <= 1) {
            for (uint32_t s = 0;; ++s) {
                const uint32_t cs_ = chan_of(s);
                if (cs_ >= C) break;
                const int64_t cp = cs_;
                const uint32_t rs = s % kSlots;
                if (s >= 2) mbar_wait(&freed[s & 1u], (s / 2 - 1) & 1u);
                const Terms t = terms(cp);
                if (lane == 0) mbar_arrive_expect_tx(&gathered[rs], K * RB);
                // the records are st.async transactions on my own barrier: completing the phase
                // makes them visible, as for a TMA load (CTA-scope acquire, no L1 invalidation)
                mbar_wait(&gathered[rs], (s / kSlots) & 1u);
                if (lane == 0) IABN_TRACE(a, s, 5);
                double v[NR], lv[NR];
                fold_cluster(rs, v);
                release_slot(rs);
#pragma unroll
                for (int k = 0; k < NR; ++k) lv[k] = v[k];
                if (lane == 0) finish(s, cp, t, v, lv);
                __syncwarp();
            }
        } else {
            // synchronized variant: the cluster's total of channel t is stored into every
            // rank's buffer (CTA 0 of the cluster, lane g -> rank g) as soon as the K CTA
            // records are in ("publish"); every CTA then folds the nranks records of the
            // channel from its own rank's buffer.  Publishing runs up to kSlots - 1 channels
            // ahead of the fold, also while the warp waits for other ranks' records, so the
            // cross-rank latency overlaps the pipeline instead of adding to it.
            const uint32_t myrank = a.rank0 + vr;
            // the call's tag; records go to the parity half (tag & 1) of the buffers: a slot
            // is rewritten two calls later, when every rank has finished reading it
            const unsigned long long tag = *(volatile unsigned long long*)a.sync_ctr;
            const size_t half = (size_t)(tag & 1ull) * a.sync_cap * a.nranks;
            const uint32_t flag = rec_flag(tag);
            const PeerRec* own = a.peer[myrank] + half;
            uint32_t pub = 0, armed = 0;
            auto arm = [&](uint32_t t) {  // expect channel t's K records
                if (lane == 0) mbar_arrive_expect_tx(&gathered[t % kSlots], K * RB);
                armed = t + 1;
            };
            auto publish = [&](uint32_t t) {  // channel t's K records (all lanes wait)
                const uint32_t rs = t % kSlots;
                const uint32_t ct = chan_of(t);
                mbar_wait(&gathered[rs], (t / kSlots) & 1u);
                double v[NR];
                fold_cluster(rs, v);
                release_slot(rs);
                if (lane == 0) {
#pragma unroll
                    for (int k = 0; k < NR; ++k) lrec[rs][k] = v[k];
                    lterm[rs] = terms(ct);  // loaded ahead of the fold
                }
                if (r == 0 && lane < a.nranks)
                    st_rec<NR>(a.peer[lane] + half + (size_t)ct * a.nranks + myrank, v, flag);
                pub = t + 1;
            };
            // slot t's channel without blocking (dynamic order: CTA 0's producer may not have
            // drawn it yet -- waiting here could hold up the buffer it needs), C = none
            auto chan_peek = [&](uint32_t t, bool* known) -> uint32_t {
                if (!dynamic) {
                    *known = true;
                    return t < nT ? q + t * Q : C;
                }
                *known = mbar_test(&chanbar[t % kChanRing], (t / kChanRing) & 1u);
                return *known ? *(volatile uint32_t*)&chan_ring[t % kChanRing] : C;
            };
            for (uint32_t s = 0;; ++s) {
                const uint32_t cs_ = chan_of(s);
                if (cs_ >= C) break;
                const int64_t cp = cs_;
                if (s >= 2) mbar_wait(&freed[s & 1u], (s / 2 - 1) & 1u);
                while (pub <= s) {
                    if (armed <= pub) arm(pub);
                    publish(pub);
                }
                // the nranks records of channel s (lane g: rank g), publishing channels whose
                // CTA records come in meanwhile
                const PeerRec* src = own + (size_t)cp * a.nranks + lane;
                double v[NR];
                unsigned long long t0 = 0;
                for (uint32_t it = 0;; ++it) {
                    bool ok = true;
                    if (lane < a.nranks) ok = ld_rec<NR>(src, flag, v);
                    if (__all_sync(0xffffffffu, ok)) break;
                    bool known = false;
                    const uint32_t cpub = pub < s + kSlots ? chan_peek(pub, &known) : C;
                    if (known && cpub < C) {
                        if (armed <= pub) arm(pub);
                        const bool in = __shfl_sync(
                            0xffffffffu,
                            lane == 0 ? mbar_test(&gathered[pub % kSlots], (pub / kSlots) & 1u)
                                      : false,
                            0);
                        if (in) {
                            publish(pub);
                            continue;
                        }
                    }
                    if (it >= 64) __nanosleep(32);
                    if ((it & 1023u) == 0) {
                        if (it == 0) t0 = gtimer();
                        else if (gtimer() - t0 > 20000000000ull) __trap();  // a rank never called
                    }
                }
                if (lane >= a.nranks)
#pragma unroll
                    for (int k = 0; k < NR; ++k) v[k] = 0.0;
#pragma unroll
                for (int k = 0; k < NR; ++k)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
                if (lane == 0) IABN_TRACE(a, s, 5);
                if (lane == 0) {
                    double lv[NR];
#pragma unroll
                    for (int k = 0; k < NR; ++k) lv[k] = lrec[s % kSlots][k];
                    const Terms t = lterm[s % kSlots];
                    finish(s, cp, t, v, lv);
                }
                __syncwarp();
            }
        }
    }

    // ==================================================== reduce (slice t): channel sums over
    // the resident slice; the CTA record is pushed into all K peers (DSMEM).  Threads
    // tid < RT of a group with named barrier gb; warp tid / 32 == 0 folds and pushes.
    auto reduce_slice = [&](const uint32_t t, const uint32_t ct, const uint32_t tid,
                            const uint32_t RT, const uint32_t gb) {
        const uint32_t gw = tid >> 5;
        {
            const int64_t c = ct;
            const uint32_t b = t % nbuf, par = (t / nbuf) & 1u;
            const uint32_t xs = smem_u32 + (uint32_t)(b * bufv * 16);  // x (fwd) or z (bwd)
            const uint32_t ds = xs + a.cap * 16u;                      // dz (bwd)
            float2 s1[NP], s2[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) s1[i] = s2[i] = make_float2(0.f, 0.f);
            float K0 = 0.f;
            float2 ig2 = make_float2(0.f, 0.f), nb2 = ig2;
            if (PASS == 0) {
                group_wait(&full[b][0], par, gw == 0, gb, RT);
                if constexpr (MIS) {  // first element of the slice's first plane
                    const MisPlane mp = mis_plane((uint64_t)(vlo / a.mis_w) * a.C + c, a.hwb);
                    K0 = lds_elem<T>(xs + mp.h);
                } else {
                    float2 p0[NP];
                    Pairs<T>::load(lds128(xs), p0);
                    K0 = p0[0].x;  // shift: a sample of this slice (cancellation-free variance)
                }
            } else {
                const InvAffine ia = inv_affine(__ldg(a.gamma + c), __ldg(a.beta + c), a.eps, a.flags);
                ig2 = make_float2(ia.inv_g, ia.inv_g);
                nb2 = make_float2(ia.nb, ia.nb);
            }
            // backward variant II (BN-dagger, Alg. 2 l.7-8): per channel
            // S1 = sum dy and Q = sum dy y = sum dz z (f' f^-1 = id on each branch), then
            // S2 = sum dy x^ = (Q - beta S1) / g on the exchange warp.  For bf16 storage the
            // sums run on the packed halves: S1 = sum dz - (1 - a) sum_{z<0} dz with the
            // z < 0 indicator from HSET2, products exact in FHFMA.BF16 (no unpacking).
            const bool v2 = !(a.flags & kVariantI);
            float2 sn[NP];  // bf16 variant II: sum of dz over z < 0
#pragma unroll
            for (int i = 0; i < NP; ++i) sn[i] = make_float2(0.f, 0.f);
            // the sums of one vector pair (z, dz) -- or of one x vector in the forward
            // vv: the slot's vector index (ACT backward: y = f^-1(z) and dy = f'(z) dz are
            // written back over z and dz, so that the apply warps do not invert again)
            auto reduce_vec = [&](const uint4 zu, const uint4 du, auto v2tag, uint32_t vv) {
                constexpr bool V2 = decltype(v2tag)::value;
                if (PASS == 0) {
                    float2 d[NP];
                    Pairs<T>::load_sub(zu, K0, d);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        s1[i] = add2(s1[i], d[i]);
                        s2[i] = fma2(d[i], d[i], s2[i]);
                    }
                } else if constexpr (ACT != 0) {  // dy = f'(z) dz, y = f^-1(z)
                    float2 zz[NP], dd[NP];
                    Pairs<T>::load(zu, zz);
                    Pairs<T>::load(du, dd);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const float2 dy = make_float2(Act<ACT>::df(zz[i].x) * dd[i].x,
                                                      Act<ACT>::df(zz[i].y) * dd[i].y);
                        const float2 y = make_float2(Act<ACT>::inv(zz[i].x), Act<ACT>::inv(zz[i].y));
                        s1[i] = add2(s1[i], dy);
                        s2[i] = V2 ? fma2(dy, y, s2[i]) : fma2(dy, fma2(y, ig2, nb2), s2[i]);
                        zz[i] = y;
                        dd[i] = dy;
                    }
                    if constexpr (WB) {
                        sts128(xs + vv * 16u, Pairs<T>::store(zz));
                        sts128(ds + vv * 16u, Pairs<T>::store(dd));
                    }
                } else if (V2 && sizeof(T) == 2) {
                    const uint32_t zw[4] = {zu.x, zu.y, zu.z, zu.w};
                    const uint32_t dw[4] = {du.x, du.y, du.z, du.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        bf16x2_acc(s1[i], dw[i]);                             // sum dz
                        bf16x2_acc_mul(sn[i], dw[i], bf16x2_ind_neg(zw[i]));  // sum_{z<0} dz
                        bf16x2_acc_mul(s2[i], dw[i], zw[i]);                  // sum dz z
                    }
                } else {
                    float2 zz[NP], dd[NP];
                    Pairs<T>::load(zu, zz);
                    Pairs<T>::load(du, dd);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const float2 sel = make_float2(zz[i].x >= 0.f ? 1.f : a.slope,
                                                       zz[i].y >= 0.f ? 1.f : a.slope);
                        const float2 dy = mul2(dd[i], sel);
                        s1[i] = add2(s1[i], dy);
                        if (V2) {
                            s2[i] = fma2(dd[i], zz[i], s2[i]);  // sum dz z
                        } else {
                            // variant I: per element dy x^ = (dz z) inv_g + nb dy
                            s2[i] = add2(s2[i], fma2(mul2(dd[i], zz[i]), ig2, mul2(dy, nb2)));
                        }
                    }
                }
            };
            // MIS: a covering slot with elements outside the plane -- those are skipped
            // (selects, not products: the slot's other bytes may hold anything)
            auto reduce_vec_masked = [&](const uint4 zu, const uint4 du, uint32_t i, uint32_t h,
                                         auto v2tag, uint32_t vv) {
                constexpr bool V2 = decltype(v2tag)::value;
                float zz[V], dd[V];
                unpack<T>(zu, zz);
                unpack<T>(du, dd);
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    const bool ok = mis_valid<T>(i, k, h, a.hwb);
                    float* a1 = (k & 1) ? &s1[k >> 1].y : &s1[k >> 1].x;
                    float* a2 = (k & 1) ? &s2[k >> 1].y : &s2[k >> 1].x;
                    if (PASS == 0) {
                        const float d = ok ? zz[k] - K0 : 0.f;
                        *a1 += d;
                        *a2 = fmaf(d, d, *a2);
                    } else if constexpr (ACT != 0) {
                        // selects, not products: a masked element may be anything
                        const float dy = Act<ACT>::df(zz[k]) * dd[k];
                        const float y = Act<ACT>::inv(zz[k]);
                        const float t2 = dy * (V2 ? y : fmaf(y, ig2.x, nb2.x));
                        *a1 += ok ? dy : 0.f;
                        *a2 += ok ? t2 : 0.f;
                        zz[k] = y;  // written back below (masked elements: the apply skips them)
                        dd[k] = dy;
                    } else if (V2 && sizeof(T) == 2) {
                        float* an = (k & 1) ? &sn[k >> 1].y : &sn[k >> 1].x;
                        *a1 += ok ? dd[k] : 0.f;
                        *an += (ok && zz[k] < 0.f) ? dd[k] : 0.f;
                        *a2 += ok ? dd[k] * zz[k] : 0.f;
                    } else {
                        const float dy = zz[k] >= 0.f ? dd[k] : dd[k] * a.slope;
                        *a1 += ok ? dy : 0.f;
                        const float t2 = V2 ? dd[k] * zz[k]
                                            : fmaf(dd[k] * zz[k], ig2.x, dy * nb2.x);
                        *a2 += ok ? t2 : 0.f;
                    }
                }
                if constexpr (WB) {
                    sts128(xs + vv * 16u, pack<T>(zz));
                    sts128(ds + vv * 16u, pack<T>(dd));
                }
            };
            // all chunks of the slice; the 4-vector body issues its 8 shared loads first
            auto sweep = [&](auto v2tag) {
                if constexpr (MIS) {
                    // slot v of the slice = (plane jn, slot i) with v = jn W + i; a cursor
                    // steps it by RT (no division in the loop); the plane's head offset
                    // is h0 + jn dh (mod 16); kMRU slots' shared loads issued first.  The
                    // main loop takes the interior slots only; the (at most two) partial
                    // slots of each plane follow in a loop of their own, one per thread
                    // (in the main loop they would make every warp run the masked path)
                    constexpr int kMRU = MINB == 4 ? 2 : 4;
                    const uint32_t W = a.mis_w, n0 = vlo / W;
                    const uint32_t h0 = mis_plane((uint64_t)n0 * a.C + c, a.hwb).h;
                    const uint32_t dh = (uint32_t)(((uint64_t)a.C * a.hwb) & 15u);
                    const uint32_t qp = RT / W, qr = RT % W;
                    auto one = [&](const uint4 zu, const uint4 du, uint32_t si, uint32_t sj,
                                   uint32_t vv) {
                        const uint32_t h = (h0 + sj * dh) & 15u;
                        if (si * 16u >= h && si * 16u + 16u <= h + a.hwb) reduce_vec(zu, du, v2tag, vv);
                    };
                    // partial slots of planes [p_lo, p_hi): e = 2 (plane - p_lo) + {0 head, 1 tail}
                    auto edges = [&](uint32_t p_lo, uint32_t p_hi) {
                        for (uint32_t e = tid; e < 2u * (p_hi - p_lo); e += RT) {
                            const uint32_t jn = p_lo + (e >> 1);
                            const uint32_t h = (h0 + jn * dh) & 15u;
                            const uint32_t tail = (h + a.hwb - 1u) >> 4;
                            const uint32_t si = (e & 1u) ? tail : 0u;
                            if ((e & 1u) && tail == 0u) continue;  // one slot: the head's
                            if (si * 16u >= h && si * 16u + 16u <= h + a.hwb) continue;  // interior
                            const uint32_t v = jn * W + si;
                            const uint4 zu = lds128(xs + v * 16u);
                            reduce_vec_masked(zu, PASS == 1 ? lds128(ds + v * 16u) : zu, si, h, v2tag, v);
                        }
                    };
                    for (int k = 0; k < nch; ++k) {
                        if (PASS == 1 || k > 0) group_wait(&full[b][k], par, gw == 0, gb, RT);
                        if (tid == 0 && k == 0) IABN_TRACE(a, t, 2);
                        if (tid == 0 && k == nch - 1) IABN_TRACE(a, t, 3);
                        const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
                        uint32_t v = c_lo + tid;
                        uint32_t jn = fdiv(v, a.fd_w), i = v - jn * W;
                        for (; v + (kMRU - 1) * RT < c_hi;) {
                            uint4 zu[kMRU], du[kMRU];
                            uint32_t iu[kMRU], ju[kMRU], vu[kMRU];
#pragma unroll
                            for (int q = 0; q < kMRU; ++q) {
                                zu[q] = lds128(xs + v * 16u);
                                du[q] = PASS == 1 ? lds128(ds + v * 16u) : zu[q];
                                iu[q] = i;
                                ju[q] = jn;
                                vu[q] = v;
                                v += RT;
                                i += qr;
                                jn += qp;
                                if (i >= W) {
                                    i -= W;
                                    ++jn;
                                }
                            }
#pragma unroll
                            for (int q = 0; q < kMRU; ++q) one(zu[q], du[q], iu[q], ju[q], vu[q]);
                        }
                        for (; v < c_hi;) {
                            const uint4 zu = lds128(xs + v * 16u);
                            one(zu, PASS == 1 ? lds128(ds + v * 16u) : zu, i, jn, v);
                            v += RT;
                            i += qr;
                            jn += qp;
                            if (i >= W) {
                                i -= W;
                                ++jn;
                            }
                        }
                        edges(c_lo / W, c_hi / W);
                    }
                } else {
                    for (int k = 0; k < nch; ++k) {
                        if (PASS == 1 || k > 0) group_wait(&full[b][k], par, gw == 0, gb, RT);
                        if (tid == 0 && k == 0) IABN_TRACE(a, t, 2);
                        if (tid == 0 && k == nch - 1) IABN_TRACE(a, t, 3);
                        const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
                        uint32_t v = c_lo + tid;
                        for (; v + (kRU - 1) * RT < c_hi; v += kRU * RT) {
                            uint4 zu[kRU], du[kRU];
    #pragma unroll
                            for (int j = 0; j < kRU; ++j) {
                                zu[j] = lds128(xs + (v + j * RT) * 16u);
                                du[j] = PASS == 1 ? lds128(ds + (v + j * RT) * 16u) : zu[j];
                            }
    #pragma unroll
                            for (int j = 0; j < kRU; ++j) reduce_vec(zu[j], du[j], v2tag, v + j * RT);
                        }
                        for (; v < c_hi; v += RT) {
                            const uint4 zu = lds128(xs + v * 16u);
                            reduce_vec(zu, PASS == 1 ? lds128(ds + v * 16u) : zu, v2tag, v);
                        }
                    }
                }
            };
            if (PASS == 1 && v2)
                sweep(std::true_type{});
            else
                sweep(std::false_type{});
            // ACT backward: the (y, dy) write-back reaches the apply warps through the record
            // hand-off (release / acquire); the TMA refill of this buffer is ordered after it
            if constexpr (WB) fence_proxy_async_smem();
            if (tid == 0) IABN_TRACE(a, t, 8);
            // fold the thread's fp32 chains and the warp in fp32 (a few rounding steps on
            // partial sums of at most a few thousand terms), the warps and CTAs in fp64
#pragma unroll
            for (int h = NP / 2; h > 0; h >>= 1)
#pragma unroll
                for (int i = 0; i < h; ++i) {
                    s1[i] = add2(s1[i], s1[i + h]);
                    s2[i] = add2(s2[i], s2[i + h]);
                    sn[i] = add2(sn[i], sn[i + h]);
                }
            float f1 = s1[0].x + s1[0].y, f2 = s2[0].x + s2[0].y;
            if (PASS == 1 && v2 && sizeof(T) == 2) f1 -= (1.f - a.slope) * (sn[0].x + sn[0].y);  // S1
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                f1 += __shfl_xor_sync(0xffffffffu, f1, o);
                f2 += __shfl_xor_sync(0xffffffffu, f2, o);
            }
            const double d1 = f1, d2 = f2;
            if (lane == 0) {
                red[t & 1][0][gw] = d1;
                red[t & 1][1][gw] = d2;
            }
            group_sync(gb, RT);
            if (gw == 0) {
                if (tid == 0) IABN_TRACE(a, t, 9);
                double S1 = 0.0, S2 = 0.0;
                for (uint32_t w = 0; w < RT / 32; ++w) {
                    S1 += red[t & 1][0][w];
                    S2 += red[t & 1][1][w];
                }
                double out[NR];
                if (PASS == 0) {
                    const double cnt = MIS ? (double)(nv / a.mis_w) * (double)a.HW : (double)nv * V;
                    write_raw_moments(out, cnt, (double)K0, S1, S2);
                } else {
                    out[0] = S1;
                    out[1] = S2;
                }
                const uint32_t rs = t % kSlots;
                // my record slot rs in every peer must have been folded (channel t - kSlots)
                // (write-after-read only: the peers' release-arrivals follow their reads)
                if (t >= (uint32_t)kSlots) mbar_wait(&slotfree[rs], (t / kSlots - 1) & 1u);
                if (lane == 0) IABN_TRACE(a, t, 10);
                if (lane < K) {  // lane j pushes this CTA's record into peer j (st.async)
                    const uint32_t mb = mapa(&gathered[rs], lane);
                    st_async_f64x2(mapa(&rec[rs][r][0], lane), out[0], out[1], mb);
                    if (NR == 3) st_async_f64x2(mapa(&rec[rs][r][2], lane), out[NR - 1], 0.0, mb);
                }
                if (lane == 0) IABN_TRACE(a, t, 4);
            }
        }
    };

    // ==================================================== apply (slice s): outputs from the
    // resident slice once the channel's coefficients are in (the reduce has read it by then).
    // Threads at < AT of a group with named barrier gb; warp 0 of the group polls.
    auto apply_slice = [&](const uint32_t s, const uint32_t cs_, const uint32_t at,
                           const uint32_t AT, const uint32_t gb) {
        const uint32_t hw = (uint32_t)a.HW;
        const float2 sl2 = make_float2(a.slope, a.slope);
        T* out = (T*)a.out + voff;
        const int64_t chw = a.C * a.HW;
        const int64_t cp = cs_;
        const uint32_t b = s % nbuf, slot = s & 1u;
        group_wait(&ready[slot], (s / 2) & 1u, at < 32, gb, AT);
        if (at == 0) IABN_TRACE(a, s, 6);
        const uint32_t xs = smem_u32 + (uint32_t)(b * bufv * 16);  // shared address of x / z
        const uint32_t ds = xs + a.cap * 16u;                      // dz (bwd)
        const float2 P = cs[slot].P, Q2 = cs[slot].Q;
        const float mu = cs[slot].mu;
        T* const outc = out + cp * a.HW;
        // whole-plane chunks with planes of at least AT vectors: per-plane addressing
        const bool plane_loop = plane_chunks && pv >= AT;
        // outputs of one vector (x, or z and dz) into dst (global)
        auto apply_vals = [&](const uint4 xu, const uint4 du, T* const dst) {
            float2 w[NP];
            if (PASS == 0) {
                Pairs<T>::load_sub(xu, mu, w);
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const float2 y = fma2(w[i], P, Q2);
                    if constexpr (ACT != 0) {
                        w[i] = make_float2(Act<ACT>::f(y.x), Act<ACT>::f(y.y));
                    } else {
                        const float2 ay = mul2(y, sl2);  // f(y) = max(y, a y) for 0 < a <= 1
                        w[i] = make_float2(fmaxf(y.x, ay.x), fmaxf(y.y, ay.y));
                    }
                }
            } else if constexpr (ACT != 0) {  // dx = alpha dy + kappa y + cc
                float2 dd[NP];
                Pairs<T>::load(xu, w);
                Pairs<T>::load(du, dd);
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    if constexpr (!WB) {  // else (y, dy) were written back by the reduce warps
                        dd[i] = make_float2(Act<ACT>::df(w[i].x) * dd[i].x, Act<ACT>::df(w[i].y) * dd[i].y);
                        w[i] = make_float2(Act<ACT>::inv(w[i].x), Act<ACT>::inv(w[i].y));
                    }
                    w[i] = fma2(make_float2(P.x, P.x), dd[i], fma2(make_float2(P.y, P.y), w[i], make_float2(mu, mu)));
                }
            } else {
                float2 dd[NP];
                Pairs<T>::load(xu, w);
                Pairs<T>::load(du, dd);
                const float2 cc2 = make_float2(mu, mu);
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const bool px = w[i].x >= 0.f, py = w[i].y >= 0.f;
                    const float2 al = make_float2(px ? P.x : Q2.x, py ? P.x : Q2.x);
                    const float2 ka = make_float2(px ? P.y : Q2.y, py ? P.y : Q2.y);
                    w[i] = fma2(al, dd[i], fma2(ka, w[i], cc2));
                }
            }
            st_vec(dst, Pairs<T>::store(w));
        };
        auto apply_vec = [&](const uint32_t v, T* const dst) {
            const uint4 xu = lds128(xs + v * 16u);
            apply_vals(xu, PASS == 1 ? lds128(ds + v * 16u) : xu, dst);
        };
        if constexpr (MIS) {
            // slots of the slice by a stride cursor (as in the reduce); interior slots are
            // whole 16-byte stores; the (at most two) edge slots of a plane store only its
            // own elements (the rest of those 16 bytes belong to neighbouring channels),
            // in a loop of their own after the interior ones (as in the reduce)
            constexpr int kMAU = MINB == 4 ? 2 : 4;
            const uint32_t W = a.mis_w, n0 = vlo / W;
            const uint64_t B0 = ((uint64_t)n0 * a.C + cp) * a.hwb;  // plane 0's first byte
            const uint64_t dB = (uint64_t)a.C * a.hwb;               // bytes between planes
            const uint32_t h0 = (uint32_t)(B0 & 15u), dh = (uint32_t)(dB & 15u);
            const uint32_t qp = AT / W, qr = AT % W;
            auto one = [&](const uint4 xu, const uint4 du, uint32_t si, uint32_t sj, bool edge) {
                const uint32_t h = (h0 + sj * dh) & 15u;
                const bool interior = si * 16u >= h && si * 16u + 16u <= h + a.hwb;
                if (interior == edge) return;  // main loop: interior slots; edge loop: the rest
                float2 w[NP];
                if (PASS == 0) {
                    Pairs<T>::load_sub(xu, mu, w);
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        const float2 y = fma2(w[j], P, Q2);
                        if constexpr (ACT != 0) {
                            w[j] = make_float2(Act<ACT>::f(y.x), Act<ACT>::f(y.y));
                        } else {
                            const float2 ay = mul2(y, sl2);
                            w[j] = make_float2(fmaxf(y.x, ay.x), fmaxf(y.y, ay.y));
                        }
                    }
                } else if constexpr (ACT != 0) {
                    float2 dd[NP];
                    Pairs<T>::load(xu, w);
                    Pairs<T>::load(du, dd);
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        if constexpr (!WB) {
                            dd[j] = make_float2(Act<ACT>::df(w[j].x) * dd[j].x, Act<ACT>::df(w[j].y) * dd[j].y);
                            w[j] = make_float2(Act<ACT>::inv(w[j].x), Act<ACT>::inv(w[j].y));
                        }
                        w[j] = fma2(make_float2(P.x, P.x), dd[j], fma2(make_float2(P.y, P.y), w[j], make_float2(mu, mu)));
                    }
                } else {
                    float2 dd[NP];
                    Pairs<T>::load(xu, w);
                    Pairs<T>::load(du, dd);
                    const float2 cc2 = make_float2(mu, mu);
#pragma unroll
                    for (int j = 0; j < NP; ++j) {
                        const bool px = w[j].x >= 0.f, py = w[j].y >= 0.f;
                        const float2 al = make_float2(px ? P.x : Q2.x, py ? P.x : Q2.x);
                        const float2 ka = make_float2(px ? P.y : Q2.y, py ? P.y : Q2.y);
                        w[j] = fma2(al, dd[j], fma2(ka, w[j], cc2));
                    }
                }
                T* const dst = (T*)((char*)out + (B0 + sj * dB - h) + si * 16u);
                if (!edge) {
                    st_vec(dst, Pairs<T>::store(w));
                } else {
#pragma unroll
                    for (int e = 0; e < V; ++e)
                        if (mis_valid<T>(si, e, h, a.hwb))
                            st_scalar<T>(dst + e, (e & 1) ? w[e >> 1].y : w[e >> 1].x);
                }
            };
            for (int k = 0; k < nch; ++k) {
                const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
                uint32_t v = c_lo + at;
                uint32_t jn = fdiv(v, a.fd_w), i = v - jn * W;
                for (; v + (kMAU - 1) * AT < c_hi;) {
                    uint4 xu[kMAU], du[kMAU];
                    uint32_t iu[kMAU], ju[kMAU];
#pragma unroll
                    for (int q = 0; q < kMAU; ++q) {
                        xu[q] = lds128(xs + v * 16u);
                        du[q] = PASS == 1 ? lds128(ds + v * 16u) : xu[q];
                        iu[q] = i;
                        ju[q] = jn;
                        v += AT;
                        i += qr;
                        jn += qp;
                        if (i >= W) {
                            i -= W;
                            ++jn;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < kMAU; ++q) one(xu[q], du[q], iu[q], ju[q], false);
                }
                for (; v < c_hi;) {
                    const uint4 xu = lds128(xs + v * 16u);
                    one(xu, PASS == 1 ? lds128(ds + v * 16u) : xu, i, jn, false);
                    v += AT;
                    i += qr;
                    jn += qp;
                    if (i >= W) {
                        i -= W;
                        ++jn;
                    }
                }
                // edge slots: e = 2 (plane - p_lo) + {0 head, 1 tail}
                const uint32_t p_lo = c_lo / W;
                for (uint32_t e = at; e < 2u * (c_hi / W - p_lo); e += AT) {
                    const uint32_t pj = p_lo + (e >> 1);
                    const uint32_t h = (h0 + pj * dh) & 15u;
                    const uint32_t tail = (h + a.hwb - 1u) >> 4;
                    if ((e & 1u) && tail == 0u) continue;  // one slot: the head's
                    const uint32_t si = (e & 1u) ? tail : 0u;
                    const uint32_t vv = pj * W + si;
                    const uint4 xu = lds128(xs + vv * 16u);
                    one(xu, PASS == 1 ? lds128(ds + vv * 16u) : xu, si, pj, true);
                }
                __syncwarp();
                if ((at & 31) == 0) mbar_arrive(&empty[b][k]);
            }
        } else {
            for (int k = 0; k < nch; ++k) {
                const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
                if (plane_loop) {
                    // the chunk is whole planes: plane n of the channel is vectors [pb, pb + pv).
                    // Thread `at` takes the chunk's vectors u = at, at + AT, ... (u = pb - c_lo + v),
                    // i.e. in each plane the v with v = at - off (mod AT), off = (pb - c_lo) % AT
                    uint32_t n = (vlo + c_lo) / pv, off = 0;
                    const uint32_t pv_mod = pv % AT;
                    for (uint32_t pb = c_lo; pb < c_hi; pb += pv, ++n) {
                        T* const dp = outc + (int64_t)n * chw;
                        uint32_t v = at >= off ? at - off : at + AT - off;
                        for (; v + (kAU - 1) * AT < pv; v += kAU * AT) {  // shared loads first
                            uint4 xu[kAU], du[kAU];
    #pragma unroll
                            for (int j = 0; j < kAU; ++j) {
                                xu[j] = lds128(xs + (pb + v + j * AT) * 16u);
                                du[j] = PASS == 1 ? lds128(ds + (pb + v + j * AT) * 16u) : xu[j];
                            }
    #pragma unroll
                            for (int j = 0; j < kAU; ++j) apply_vals(xu[j], du[j], dp + (v + j * AT) * V);
                        }
                        for (; v < pv; v += AT) apply_vec(pb + v, dp + v * V);
                        off += pv_mod;
                        off = off >= AT ? off - AT : off;
                    }
                } else {
                    // output cursor: the thread visits v = c_lo + at, + AT, ... i.e. channel-space
                    // steps of AT*V elements: one plane wrap at most when the step <= HW, else
                    // the plane by division
                    const uint32_t step = AT * V;
                    const int64_t jump = (int64_t)step + chw - hw;  // step across a plane boundary
                    uint32_t v = c_lo + at;
                    const uint32_t j0 = (vlo + v) * V;
                    const uint32_t n0 = fdiv(j0, a.fd_hw);
                    uint32_t jsp = j0 - n0 * hw;
                    T* dst = outc + (int64_t)n0 * chw + jsp;
                    if (hw >= step) {
                        for (; v < c_hi; v += AT) {
                            apply_vec(v, dst);
                            jsp += step;
                            const bool wrap = jsp >= hw;
                            jsp = wrap ? jsp - hw : jsp;
                            dst += wrap ? jump : (int64_t)step;
                        }
                    } else {
                        for (; v < c_hi; v += AT) {
                            const uint32_t j = (vlo + v) * V;
                            const uint32_t n = fdiv(j, a.fd_hw);
                            apply_vec(v, outc + (int64_t)n * chw + (j - n * hw));
                        }
                    }
                }
                __syncwarp();
                if ((at & 31) == 0) mbar_arrive(&empty[b][k]);  // chunk k of buffer b may be refilled
            }
        }
        if (at == 0) IABN_TRACE(a, s, 7);
        if ((at & 31) == 0) mbar_arrive(&freed[slot]);  // coefficient slot may be rewritten
    };

    if (warp == kProducerWarp || warp == kExchangeWarp) {
        // above
    } else if (warp >= (uint32_t)kReduceWarp0 && warp < (uint32_t)(kReduceWarp0 + kReduceWarps)) {
        for (uint32_t t = 0;; ++t) {
            const uint32_t ct = chan_of(t);
            if (ct >= C) break;
            reduce_slice(t, ct, threadIdx.x - kReduceWarp0 * 32, kReduceWarps * 32, 1);
        }
    } else {
        for (uint32_t s = 0;; ++s) {
            const uint32_t cs_ = chan_of(s);
            if (cs_ >= C) break;
            apply_slice(s, cs_, threadIdx.x - kApplyWarp0 * 32, kApplyWarps * 32, 2);
        }
    }
    // peers may still push records / arrive on this CTA's barriers until they finish
    cluster_arrive_release();
    cluster_wait_acquire();
    if (dynamic && r == 0 && threadIdx.x == 0) {
        // the last cluster (every ticket is drawn by then) re-arms the counters
        __threadfence();
        if (atomicAdd(&a.dyn[2 * vr + 1], 1u) == Q - 1) {  // this rank's clusters
            atomicExch(&a.dyn[2 * vr], 0u);
            atomicExch(&a.dyn[2 * vr + 1], 0u);
        }
    }
    if (a.nranks > 1 && threadIdx.x == 0) {
        // the grid's last CTA advances the call number for the next call on this stream
        __threadfence();
        if (atomicAdd(&a.sync_ctr[1], 1ull) == gridDim.x - 1) {
            atomicExch(&a.sync_ctr[1], 0ull);
            atomicAdd(&a.sync_ctr[0], 1ull);
        }
    }
}

}  // namespace iabn
