// kernels_nhwc_bulk.cuh -- NHWC streaming reductions fed by TMA bulk copies (round 2).
//
// The streaming schedule is what large NHWC layers run (their channel groups do not fit
// on chip).  Its reductions (F1 statistics, B1 gradient sums) were LDG loops whose CTAs
// each covered ~256 rows with 2-4 rows in flight per thread; ncu on DenseNet's
// 128x56^2 bf16 layer: 1.4 TB/s (statistics) and 1.7 TB/s (gradient sums).  Here CTA s
// of a grid of G <= 256 (32 clusters of 8 at 2 CTAs per SM: all resident at once) takes
// the chunks s, s + G, ... of rps whole rows (at any moment the grid reads one contiguous
// front of the tensor) and streams them through a 4-stage shared-memory ring with
// cp.async.bulk (one elected thread, mbarrier complete_tx), 64 KB in flight per CTA
// whatever the register budget.  Consumers read 16-byte vectors from the ring:
//   cv = C*b/16 <= 256 vectors per row; blockDim = rt * cv (rt = 256 / cv row lanes):
//   thread t takes vector j = t % cv (channels j*V .. j*V + V-1) of rows t / cv, + rt, ...
// Packed fp32x2 (FADD2 / FFMA2) and bf16x2 (FHADD / FHFMA.BF16) arithmetic, fp32 per
// thread in runs of <= 64 rows, fp64 across runs; then the rt row lanes in a fixed order
// in shared memory, and the 8 CTAs of a cluster in rank order over DSMEM -> one record
// per (cluster, channel): F1 raw moments (count, sum, sum of squares, shifted by the
// channel's first value as everywhere, R8) or B1 -- (sum dz, sum_{z<0} dz,
// sum dz z) folded to (S1, S2) by BN-dagger, or (sum dy, sum dy x^) with IABN_VARIANT_I --
// the record layout the coefficient kernels combine (<= 32 records instead of 296).
// Requires C*b % 16 == 0 (bulk copies of whole rows) and C*b <= 4 KB.
#pragma once

#include "common.cuh"
#include "kernels_act.cuh"
#include "kernels_stream.cuh"

namespace iabn {

#ifndef IABN_NB_EVICT_LAST
#define IABN_NB_EVICT_LAST 0
#endif
constexpr int kNbStages = 4;
constexpr uint32_t kNbStageBytes = 16384;  // per stage, all inputs together

struct NbArgs {
    const void* in0;  // x (F1) / z (B1)
    const void* in1;  // dz (B1)
    const float* gamma;
    const float* beta;
    int64_t C, rows;
    uint32_t cv;    // 16-byte vectors per row (<= 256)
    uint32_t rt;    // row lanes: blockDim.x = rt * cv
    uint32_t rps;   // rows per stage
    float eps, slope;
    uint32_t flags;
    double* part;   // [G / K][C][3] (F1) / [G / K][C][2] (B1), one record per cluster
    unsigned long long* trace;  // experiments: [G][kNbTrace] %globaltimer of CTA phases
};
// phases: 0 start, 1 PDL wait done, 2 first chunk landed, 3 last chunk landed, 4 loop
// done, 5 row lanes summed, 6 cluster met, 7 records written
constexpr int kNbTrace = 8;

// dynamic shared memory: barriers (128 B) + ring (kNbStages * kNbStageBytes); the fp64
// epilogue reuses the ring
constexpr size_t kNbSmem = 128 + (size_t)kNbStages * kNbStageBytes;
#ifndef IABN_NB_CLUSTER
#define IABN_NB_CLUSTER 8
#endif
constexpr int kNbCluster = IABN_NB_CLUSTER;  // CTAs per cluster: records summed over DSMEM

// PASS 0: F1 shifted sums (sum d, sum d^2), d = x - K.  PASS 1, V2 (default, InPlace-ABN II
// as in the channel-resident kernels, R6): (sum dz, sum_{z<0} dz, sum dz z);
// PASS 1, !V2 (IABN_VARIANT_I): (sum dy, sum dy x^) per element.
// ACT (fp32, PASS 1): 1 sigmoid / 2 tanh -- (sum dy, 0, sum dy y) with dy = f'(z) dz,
// y = f^-1(z) (V2), or (sum dy, sum dy x^) (!V2)
template <typename T, int PASS, bool V2, int ACT = 0>
__global__ void __launch_bounds__(kThreads, 2) nhwc_bulk_reduce_kernel(const NbArgs a) {
    constexpr int V = Elem<T>::kVec;
    constexpr int NP = Pairs<T>::kN;
    constexpr int NI = PASS == 0 ? 1 : 2;
    constexpr int NA = (PASS == 1 && V2) ? 3 : 2;  // accumulators per element
    constexpr int NV = PASS == 0 ? 3 : 2;          // doubles per output record
    extern __shared__ __align__(128) unsigned char nb_smem[];
    auto trace = [&](int k) {
        if (a.trace && threadIdx.x == 0) {
            unsigned long long tm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
            a.trace[(size_t)blockIdx.x * kNbTrace + k] = tm;
        }
    };
    trace(0);
    uint64_t* full = reinterpret_cast<uint64_t*>(nb_smem);
    uint64_t* empty = full + kNbStages;
    unsigned char* ring = nb_smem + 128;
    const uint32_t t = threadIdx.x, lane = t & 31, nwarp = (blockDim.x + 31) / 32;
    const uint32_t G = gridDim.x, s = blockIdx.x;
    const uint32_t cv = a.cv, rt = a.rt, rl = t / cv, j = t - rl * cv;
    const uint32_t rowb = cv * 16u;
    constexpr uint32_t SB = kNbStageBytes / NI;  // bytes per input per stage
    // chunks of rps rows, dealt round-robin: CTA s takes chunks s, s + G, ... (at any
    // moment the grid reads one contiguous front of the tensor)
    const int64_t nall = (a.rows + a.rps - 1) / a.rps;
    const int64_t nchunk = s < nall ? (nall - s + G - 1) / G : 0;
    long long* cnt = reinterpret_cast<long long*>(nb_smem + 64);  // rows taken (F1 count)
    const char* src0 = static_cast<const char*>(a.in0);
    const char* src1 = static_cast<const char*>(a.in1);

    if (t == 0) {
        for (int i = 0; i < kNbStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], nwarp);
        }
        fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();
    trace(1);
    auto rows_of = [&](int64_t k) -> uint32_t {
        const int64_t left = a.rows - (s + k * G) * (int64_t)a.rps;
        return (uint32_t)(left < (int64_t)a.rps ? left : (int64_t)a.rps);
    };
    auto issue = [&](int64_t k) {
        const int st = (int)(k % kNbStages);
        const int64_t r0 = (s + k * G) * (int64_t)a.rps;
        const uint32_t bytes = rows_of(k) * rowb;
        mbar_arrive_expect_tx(&full[st], bytes * NI);
#if IABN_NB_EVICT_LAST  // experiments: keep x in L2 for the apply's re-read
        if (PASS == 0)
            bulk_g2s_hint(ring + (size_t)st * kNbStageBytes, src0 + r0 * rowb, bytes, &full[st],
                          l2_policy_evict_last());
        else
#endif
        bulk_g2s(ring + (size_t)st * kNbStageBytes, src0 + r0 * rowb, bytes, &full[st]);
        if (NI == 2)
            bulk_g2s(ring + (size_t)st * kNbStageBytes + SB, src1 + r0 * rowb, bytes, &full[st]);
    };
    if (t == 0) {
        for (int64_t k = 0; k < (nchunk < kNbStages ? nchunk : (int64_t)kNbStages); ++k) issue(k);
        long long n = 0;
        for (int64_t k = 0; k < nchunk; ++k) n += rows_of(k);
        *cnt = n;
    }

    // per-channel constants of this thread's vector j (channels j*V .. j*V + V-1)
    const int64_t c0 = (int64_t)j * V;
    float2 nK[NP];              // F1: -K (shift = the channel's first value)
    InvAffine ia[PASS == 1 && !V2 ? V : 1];  // (inv_g, -beta/g) per channel
#pragma unroll
    for (int i = 0; i < NP; ++i) nK[i] = make_float2(0.f, 0.f);
    if (PASS == 0) {
        const T* x0 = static_cast<const T*>(a.in0) + c0;
#pragma unroll
        for (int i = 0; i < NP; ++i) nK[i] = make_float2(-ld_scalar<T>(x0 + 2 * i), -ld_scalar<T>(x0 + 2 * i + 1));
    } else if (!V2) {
#pragma unroll
        for (int e = 0; e < (PASS == 1 && !V2 ? V : 1); ++e)
            ia[e] = inv_affine(a.gamma[c0 + e], a.beta[c0 + e], a.eps, a.flags);
    }
    float2 acc[NA][NP];
    double dacc[NA][V];
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            acc[q][i] = make_float2(0.f, 0.f);
            dacc[q][2 * i] = dacc[q][2 * i + 1] = 0.0;
        }
    auto flush = [&]() {
#pragma unroll
        for (int q = 0; q < NA; ++q)
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                dacc[q][2 * i] += acc[q][i].x;
                dacc[q][2 * i + 1] += acc[q][i].y;
                acc[q][i] = make_float2(0.f, 0.f);
            }
    };
    uint32_t run = 0;

    for (int64_t k = 0; k < nchunk; ++k) {
        const int st = (int)(k % kNbStages);
        const uint32_t nr = rows_of(k);
        mbar_wait(&full[st], (uint32_t)((k / kNbStages) & 1));
        if (k == 0) trace(2);
        if (k == nchunk - 1) trace(3);
        const uint32_t base = smem_addr(ring + (size_t)st * kNbStageBytes) + j * 16u;
        for (uint32_t r = rl; r < nr; r += rt) {
            const uint4 u = lds128(base + r * rowb);
            if (PASS == 0) {
                float2 p[NP];
                Pairs<T>::load(u, p);
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const float2 d = add2(p[i], nK[i]);
                    acc[0][i] = add2(acc[0][i], d);
                    acc[1][i] = fma2(d, d, acc[1][i]);
                }
            } else {
                const uint4 w = lds128(base + SB + r * rowb);
                if constexpr (ACT != 0) {
                    float2 zp[NP], dp[NP];
                    Pairs<T>::load(u, zp);
                    Pairs<T>::load(w, dp);
#pragma unroll
                    for (int i = 0; i < NP; ++i) {
                        const float2 dy = make_float2(Act<ACT>::df(zp[i].x) * dp[i].x,
                                                      Act<ACT>::df(zp[i].y) * dp[i].y);
                        float2 y = make_float2(Act<ACT>::inv(zp[i].x), Act<ACT>::inv(zp[i].y));
                        if constexpr (!V2)  // x^ = y inv_g + nb
                            y = make_float2(fmaf(y.x, ia[2 * i].inv_g, ia[2 * i].nb),
                                            fmaf(y.y, ia[2 * i + 1].inv_g, ia[2 * i + 1].nb));
                        acc[0][i] = add2(acc[0][i], dy);
                        acc[NA - 1][i] = fma2(dy, y, acc[NA - 1][i]);
                    }
                } else if constexpr (V2) {
                    if constexpr (sizeof(T) == 2) {  // packed bf16 ops (no unpacking)
                        const uint32_t zw[4] = {u.x, u.y, u.z, u.w}, dw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                        for (int i = 0; i < NP; ++i) {
                            bf16x2_acc(acc[0][i], dw[i]);
                            bf16x2_acc_mul(acc[1][i], dw[i], bf16x2_ind_neg(zw[i]));
                            bf16x2_acc_mul(acc[2][i], dw[i], zw[i]);
                        }
                    } else {
                        float2 zp[NP], dp[NP];
                        Pairs<T>::load(u, zp);
                        Pairs<T>::load(w, dp);
#pragma unroll
                        for (int i = 0; i < NP; ++i) {
                            acc[0][i] = add2(acc[0][i], dp[i]);
                            acc[1][i] = add2(acc[1][i], make_float2(zp[i].x < 0.f ? dp[i].x : 0.f,
                                                                    zp[i].y < 0.f ? dp[i].y : 0.f));
                            acc[2][i] = fma2(dp[i], zp[i], acc[2][i]);
                        }
                    }
                } else {
                    float fz[V], fd[V];
                    unpack<T>(u, fz);
                    unpack<T>(w, fd);
                    const float inv_slope = 1.0f / a.slope;
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        float dy, xh;
                        grad_terms(fz[e], fd[e], a.slope, inv_slope, ia[e], dy, xh);
                        float2& s1 = acc[0][e >> 1];
                        float2& s2 = acc[1][e >> 1];
                        if (e & 1) {
                            s1.y += dy;
                            s2.y = fmaf(dy, xh, s2.y);
                        } else {
                            s1.x += dy;
                            s2.x = fmaf(dy, xh, s2.x);
                        }
                    }
                }
            }
            if (++run == 64) {
                run = 0;
                flush();
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        if (t == 0 && k + kNbStages < nchunk) {
            mbar_wait(&empty[st], (uint32_t)((k / kNbStages) & 1));  // every warp is done
            issue(k + kNbStages);
        }
    }
    flush();
    trace(4);
    // (1) the rt row lanes of this CTA, fixed order, in shared memory (the ring is free:
    // every stage consumed); layout [q][e][rl][j] (consecutive threads, consecutive words)
    __syncthreads();
    double* red = reinterpret_cast<double*>(ring);
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
        for (int e = 0; e < V; ++e) red[(((size_t)q * V + e) * rt + rl) * cv + j] = dacc[q][e];
    __syncthreads();
    // this CTA's per-channel totals, summed over the row lanes into lane 0's slots: one
    // thread per column (q, e, j) -- consecutive threads, consecutive words -- reading its
    // rt values first, then adding them in lane order
    auto fin = [&](uint32_t c, int q) -> size_t {
        const uint32_t jj = c / V, e = c - jj * V;
        return (((size_t)q * V + e) * rt) * cv + jj;
    };
    if (rt > 1) {
        const uint32_t ncol = NA * V * cv;
        for (uint32_t col = t; col < ncol; col += blockDim.x) {
            const uint32_t jj = col % cv, qe = col / cv;  // qe = q * V + e
            const double* src = red + (size_t)qe * rt * cv + jj;
            double v = 0.0;
            for (uint32_t r0 = 0; r0 < rt; r0 += 8) {
                double w[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) w[u] = r0 + u < rt ? src[(size_t)(r0 + u) * cv] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u) v += w[u];
            }
            red[(size_t)qe * rt * cv + jj] = v;
        }
    }
    trace(5);
    // (2) the cluster's CTAs in rank order over DSMEM: rank r finalises channels c = r mod K
    cluster_arrive_release();
    cluster_wait_acquire();
    trace(6);
    const uint32_t rank = cluster_ctarank(), K = cluster_nctarank();
    for (uint32_t c = rank + t * K; c < (uint32_t)a.C; c += blockDim.x * K) {
        double w[kNbCluster][NA], v[NA];  // every remote load in flight, then the adds
#pragma unroll
        for (int r = 0; r < kNbCluster; ++r)
#pragma unroll
            for (int q = 0; q < NA; ++q) w[r][q] = (uint32_t)r < K ? ld_dsmem_f64(red + fin(c, q), r) : 0.0;
#pragma unroll
        for (int q = 0; q < NA; ++q) {
            v[q] = 0.0;
#pragma unroll
            for (int r = 0; r < kNbCluster; ++r) v[q] += w[r][q];
        }
        double* o = a.part + ((size_t)(s / K) * a.C + c) * NV;
        if (PASS == 0) {
            int64_t n = 0;
            for (uint32_t r = 0; r < K; ++r) n += ld_dsmem_s64(cnt, r);
            const double Kc = (double)ld_scalar<T>(static_cast<const T*>(a.in0) + c);
            write_raw_moments(o, (double)n, Kc, v[0], v[1]);
        } else if (V2) {  // BN-dagger: S1 = sum dz - (1 - a) sum_{z<0} dz, S2 = (Q - beta S1)/g
            const double S1 = v[0] - (1.0 - (double)a.slope) * v[1];
            o[0] = S1;
            o[1] = (v[2] - (double)a.beta[c] * S1) / gamma_eff(a.gamma[c], a.eps, a.flags);
        } else {
            o[0] = v[0];
            o[1] = v[1];
        }
    }
    trace(7);
    cluster_arrive_release();  // peers keep their totals until every rank has read them
    cluster_wait_acquire();
}

}  // namespace iabn
