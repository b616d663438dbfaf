// kernels_nhwc.cuh -- channel-group-resident schedule for NHWC ([rows][C], rows = N*HW).
//
// In NHWC a channel's m values are spread over every row of the tensor (stride C), so
// no contiguous per-channel slab exists.  Instead a CLUSTER of K CTAs owns a GROUP of g
// adjacent channels (g*b = 16..256 bytes of every row): CTA r of the cluster holds rows
// [r R_cta, (r+1) R_cta) of the group's columns, loaded with 2-D TMA tensor copies
// (cp.async.bulk.tensor.2d, box = [g channels] x [R rows], SASS UTMALDG) into a dense
// [rows][g] shared-memory slab.  Then, all threads:
//
//   reduce  : per-thread fp32 partials of the thread's fixed column (g*b/16 16-byte
//             columns per row; a thread walks rows with stride 256/cols), folded over the
//             lanes of the same column by xor shuffles and over the 8 warps in fp64;
//             box i is reduced as soon as its TMA transaction lands (one mbarrier per box);
//   exchange: the CTA's fp64 record per channel -- (count, sum x, sum x^2) forward,
//             (sum dy, sum dz z) backward -- stored into every peer's shared memory
//             (DSMEM st.shared::cluster), one cluster barrier, then each CTA folds the K
//             records in rank order (identical totals in every CTA);
//   apply   : z (or dx) computed in place in the slab from the per-channel coefficients,
//             written back with 2-D TMA tensor stores (UTMASTG; in place: z over x, dx
//             over dz allowed).
//
// HBM traffic is the method's minimum: 2*E*b forward, 3*E*b backward (the NHWC
// streaming schedule moves 3*E*b and 5*E*b).  Persistent: cluster q handles groups
// q, q + Q, ...; the next group's boxes are prefetched into L2 while the current one is
// processed.  Arithmetic follows the other schedules: shifted fp32 sums (shift = the
// channel's first value), fp64 records and combine, the fp32-pair mean of the apply
// (fwd_coef_from_moments), and the backward's BN-dagger sums (R6):
// Q = sum dz z, S1 = sum dy = sum dz - (1 - a) sum_{z<0} dz, S2 = (Q - beta S1) / g,
// or per-element dy x^ (IABN_VARIANT_I).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "kernels_act.cuh"
#include "kernels_stream.cuh"

namespace iabn {

constexpr int kNhwcThreads = 256;
constexpr int kNhwcMaxK = 8;        // CTAs per cluster (portable)
constexpr int kNhwcMaxBoxes = 64;   // TMA boxes (mbarriers) per CTA slab

struct NhwcArgs {
    const void* in0;  // forward: x; backward: z  (row 0 gives the forward's shifts)
    const float* gamma;
    const float* beta;
    float* running_mean;
    float* running_var;
    float* save_mean;
    float* save_var;  // forward: out; backward: in
    float* dgamma;
    float* dbeta;
    int64_t C;
    uint32_t m;         // rows (N*HW)
    double inv_m;       // 1 / m
    uint32_t g;         // channels per group
    uint32_t cols;      // 16-byte columns per group row (g*b/16; a power of 2 <= 32)
    uint32_t ngroups;   // ceil(C / g)
    uint32_t K;         // CTAs per cluster
    uint32_t rows_cta;  // rows per CTA slab (multiple of box_rows)
    uint32_t box_rows;  // TMA box height (multiple of 256 / cols, <= 256)
    uint32_t slab_bytes;  // bytes of one input's slab
    uint32_t red_off, rec_off, coef_off, bar_off;  // shared-memory layout (bytes)
    float momentum, eps, slope, inv_slope;
    uint32_t flags;
    uint32_t prefetch;  // L2 prefetch of the next group's boxes
    unsigned long long* trace;  // experiments: [grid][kNhwcTrace] %globaltimer of CTA phases
};
// phase timestamps of the first group (trace != nullptr): 0 start, 1 after the PDL wait,
// 2 loads issued, 3 last box landed (thread 0), 4 reduce folded, 5 records exchanged,
// 6 coefficients ready, 7 applied, 8 stores issued, 9 exit
constexpr int kNhwcTrace = 10;

// ------------------------------------------------------------------ TMA tensor copies
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int32_t c0,
                                            int32_t r0, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(r0), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, int32_t c0, int32_t r0,
                                             const void* src) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
            reinterpret_cast<uint64_t>(tm)),
        "r"(c0), "r"(r0), "r"(smem_addr(src))
        : "memory");
}
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* tm, int32_t c0, int32_t r0) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(
                     reinterpret_cast<uint64_t>(tm)),
                 "r"(c0), "r"(r0)
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* tm) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read0() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// all committed bulk stores have completed (their writes are performed)
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer_nhwc() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mbar_wait_nhwc(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity), "n"(0x100000)
        : "memory");
}

// ------------------------------------------------------------------ kernel
// PASS 0 forward (in0 = x, out = z), PASS 1 backward (in0 = z, in1 = dz, out = dx).
// ACT: 0 leaky ReLU, 1 sigmoid, 2 tanh (fp32 only; kernels_act.cuh)
template <typename T, int PASS, int ACT = 0>
__global__ void __launch_bounds__(kNhwcThreads, 1)
    nhwc_fused_kernel(const __grid_constant__ CUtensorMap tm_in0,
                      const __grid_constant__ CUtensorMap tm_in1,
                      const __grid_constant__ CUtensorMap tm_out, const NhwcArgs a) {
    constexpr int V = Elem<T>::kVec;   // channels per 16-byte column
    constexpr int NP = Pairs<T>::kN;   // fp32 pairs per column
    constexpr int NR = PASS == 0 ? 3 : 2;  // record doubles per channel
    constexpr int NIN = PASS == 0 ? 1 : 2;
    extern __shared__ __align__(128) unsigned char nsm[];
    unsigned char* slab0 = nsm;
    unsigned char* slab1 = nsm + a.slab_bytes;  // backward: dz
    double* red = reinterpret_cast<double*>(nsm + a.red_off);    // [8 warps][g][NR]
    double* rec = reinterpret_cast<double*>(nsm + a.rec_off);    // [2][K][g][NR]
    float* coef = reinterpret_cast<float*>(nsm + a.coef_off);    // [g][8]
    uint64_t* bars = reinterpret_cast<uint64_t*>(nsm + a.bar_off);  // [nbox]

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t K = a.K;
    const uint32_t rank = K > 1 ? cluster_ctarank() : 0;
    const uint32_t q = blockIdx.x / K, Q = gridDim.x / K;
    const uint32_t cols = a.cols, g = a.g;
    const uint32_t rs = kNhwcThreads / cols;  // rows per sweep of the block
    const uint32_t col = tid % cols, trow = tid / cols;
    const uint32_t nbox = a.rows_cta / a.box_rows;
    const uint32_t row0 = rank * a.rows_cta;
    const uint32_t rows_valid = row0 >= a.m ? 0u : min(a.rows_cta, a.m - row0);
    const uint32_t nbox_valid = (rows_valid + a.box_rows - 1) / a.box_rows;
    const uint32_t row_bytes = g * (uint32_t)sizeof(T);
    const uint32_t box_bytes = a.box_rows * row_bytes;
    float* pshift = coef + g * 8;  // [g] forward shifts
    float* pgam = pshift + g;      // [g] gamma, beta, save_var of the group (prefetched)
    float* pbet = pgam + g;
    float* pvar = pbet + g;
    float* prm = pvar + g;  // running mean / var of the group (forward, rank 0)
    float* prv = prm + g;
    auto trace = [&](int k) {
        if (a.trace && tid == 0) a.trace[(size_t)blockIdx.x * kNhwcTrace + k] = gtimer_nhwc();
    };
    trace(0);

    if (tid == 0) {
        tma_prefetch_desc(&tm_in0);
        if (PASS == 1) tma_prefetch_desc(&tm_in1);
        tma_prefetch_desc(&tm_out);
        for (uint32_t i = 0; i < nbox; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    if (K > 1) {
        cluster_arrive_release();
        cluster_wait_acquire();
    } else {
        __syncthreads();
    }
    pdl_wait();
    trace(1);

    const float slope = a.slope, inv_slope = a.inv_slope;
    uint32_t iter = 0;
    for (uint32_t grp = q; grp < a.ngroups; grp += Q, ++iter) {
        const int32_t c0 = (int32_t)(grp * g);
        // ---- per-channel parameters of the group: loaded now, their latency hidden
        // behind the slab's TMA load (read after the reduction)
        if (iter > 0) __syncthreads();  // the previous group's readers of pshift..pvar
        if (tid >= 32 && tid < 32 + g) {
            const uint32_t j = tid - 32;
            const int64_t c = (int64_t)c0 + j;
            const bool ok = c < a.C;
            pgam[j] = ok ? a.gamma[c] : 1.f;
            pbet[j] = ok ? a.beta[c] : 0.f;
            if (PASS == 0) {
                pshift[j] = ok ? ld_scalar<T>(static_cast<const T*>(a.in0) + c) : 0.f;
                if (rank == 0) {  // running statistics, read-modify-written after the fold
                    prm[j] = ok && a.running_mean ? a.running_mean[c] : 0.f;
                    prv[j] = ok && a.running_var ? a.running_var[c] : 0.f;
                }
            } else {
                pvar[j] = ok ? a.save_var[c] : 1.f;
            }
        }
        // ---- load this CTA's rows of the group (one mbarrier per box)
        if (tid == 0) {
            if (iter > 0) bulk_wait_read0();  // the previous group's stores read the slab
            for (uint32_t i = 0; i < nbox_valid; ++i) {
                mbar_arrive_expect_tx(&bars[i], box_bytes * NIN);
                tma_load_2d(slab0 + i * box_bytes, &tm_in0, c0, (int32_t)(row0 + i * a.box_rows),
                            &bars[i]);
                if (PASS == 1)
                    tma_load_2d(slab1 + i * box_bytes, &tm_in1, c0,
                                (int32_t)(row0 + i * a.box_rows), &bars[i]);
            }
            if (iter == 0) trace(2);
            if (a.prefetch && grp + Q < a.ngroups) {
                const int32_t cn = (int32_t)((grp + Q) * g);
                for (uint32_t i = 0; i < nbox_valid; ++i) {
                    tma_prefetch_2d(&tm_in0, cn, (int32_t)(row0 + i * a.box_rows));
                    if (PASS == 1) tma_prefetch_2d(&tm_in1, cn, (int32_t)(row0 + i * a.box_rows));
                }
            }
        }
        const uint32_t cbase = col * V;  // first channel of this thread's column (in group)
        // forward shift: the channel's first value (row 0), identical in every CTA
        float shift[V];
        if (PASS == 0) {
            const T* x0 = static_cast<const T*>(a.in0);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int64_t c = (int64_t)c0 + cbase + k;
                shift[k] = c < a.C ? ld_scalar<T>(x0 + c) : 0.f;
            }
        }
        float betav[V], ginv[V];
        if (PASS == 1 && (ACT != 0 || (a.flags & kVariantI))) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int64_t c = (int64_t)c0 + cbase + k;
                betav[k] = c < a.C ? a.beta[c] : 0.f;
                ginv[k] = c < a.C ? (float)(1.0 / gamma_eff(a.gamma[c], a.eps, a.flags)) : 0.f;
            }
        }
        // ---- reduce (fp32 pairs, per thread)
        float2 s1[NP], s2[NP], s3[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) s1[i] = s2[i] = s3[i] = make_float2(0.f, 0.f);
        const uint32_t sbase0 = smem_addr(slab0), sbase1 = smem_addr(slab1);
        auto red_fwd = [&](const uint4 u) {
            float2 d[NP];
            Pairs<T>::load(u, d);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float2 dd = add2(d[p], make_float2(-shift[2 * p], -shift[2 * p + 1]));
                s1[p] = add2(s1[p], dd);
                s2[p] = fma2(dd, dd, s2[p]);
            }
        };
        auto red_bwd = [&](const uint4 uz, const uint4 ud) {
            float2 zz[NP], dd[NP];
            Pairs<T>::load(uz, zz);
            Pairs<T>::load(ud, dd);
            if constexpr (ACT != 0) {  // s1 = sum dy, s3 = sum dy y (II) / dy x^ (I), s2 = 0
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const float2 dy = make_float2(Act<ACT>::df(zz[p].x) * dd[p].x,
                                                  Act<ACT>::df(zz[p].y) * dd[p].y);
                    float2 y = make_float2(Act<ACT>::inv(zz[p].x), Act<ACT>::inv(zz[p].y));
                    if (a.flags & kVariantI)
                        y = make_float2((y.x - betav[2 * p]) * ginv[2 * p],
                                        (y.y - betav[2 * p + 1]) * ginv[2 * p + 1]);
                    s1[p] = add2(s1[p], dy);
                    s3[p] = fma2(dy, y, s3[p]);
                }
            } else {
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const float2 neg = make_float2(zz[p].x < 0.f ? dd[p].x : 0.f,
                                                   zz[p].y < 0.f ? dd[p].y : 0.f);
                    s1[p] = add2(s1[p], dd[p]);   // sum dz
                    s2[p] = add2(s2[p], neg);     // sum_{z<0} dz
                    if (a.flags & kVariantI) {
                        // dy x^ with dy, y on the branch of sign(z)
                        const float y0 = zz[p].x >= 0.f ? zz[p].x : zz[p].x * inv_slope;
                        const float y1 = zz[p].y >= 0.f ? zz[p].y : zz[p].y * inv_slope;
                        const float dy0 = zz[p].x >= 0.f ? dd[p].x : dd[p].x * slope;
                        const float dy1 = zz[p].y >= 0.f ? dd[p].y : dd[p].y * slope;
                        s3[p].x = fmaf(dy0, (y0 - betav[2 * p]) * ginv[2 * p], s3[p].x);
                        s3[p].y = fmaf(dy1, (y1 - betav[2 * p + 1]) * ginv[2 * p + 1], s3[p].y);
                    } else {
                        s3[p] = fma2(dd[p], zz[p], s3[p]);  // sum dz z = sum dy y
                    }
                }
            }
        };
        for (uint32_t i = 0; i < nbox_valid; ++i) {
            mbar_wait_nhwc(&bars[i], iter & 1u);
            const uint32_t rend = min((i + 1) * a.box_rows, rows_valid);
            uint32_t r = i * a.box_rows + trow;
            // two rows per step: both shared loads issued before the math
            for (; r + rs < rend; r += 2 * rs) {
                const uint32_t o0 = r * row_bytes + col * 16u, o1 = o0 + rs * row_bytes;
                if (PASS == 0) {
                    const uint4 u0 = lds128(sbase0 + o0), u1 = lds128(sbase0 + o1);
                    red_fwd(u0);
                    red_fwd(u1);
                } else {
                    const uint4 z0 = lds128(sbase0 + o0), d0 = lds128(sbase1 + o0);
                    const uint4 z1 = lds128(sbase0 + o1), d1 = lds128(sbase1 + o1);
                    red_bwd(z0, d0);
                    red_bwd(z1, d1);
                }
            }
            if (r < rend) {
                const uint32_t o0 = r * row_bytes + col * 16u;
                if (PASS == 0) red_fwd(lds128(sbase0 + o0));
                else red_bwd(lds128(sbase0 + o0), lds128(sbase1 + o0));
            }
        }
        if (iter == 0) trace(3);
        // ---- fold lanes of the same column (xor over offsets >= cols) in fp32 (a few
        // partials of short per-thread chains), then the 8 warps in fp64
        float v[V][2];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            if (PASS == 0) {
                v[2 * p][0] = s1[p].x; v[2 * p + 1][0] = s1[p].y;
                v[2 * p][1] = s2[p].x; v[2 * p + 1][1] = s2[p].y;
            } else {
                // S1 = sum dz - (1 - a) sum_{z<0} dz
                v[2 * p][0] = fmaf(-(1.f - slope), s2[p].x, s1[p].x);
                v[2 * p + 1][0] = fmaf(-(1.f - slope), s2[p].y, s1[p].y);
                v[2 * p][1] = s3[p].x; v[2 * p + 1][1] = s3[p].y;
            }
        }
        for (uint32_t off = 16; off >= cols; off >>= 1) {
#pragma unroll
            for (int k = 0; k < V; ++k)
#pragma unroll
                for (int j = 0; j < 2; ++j)
                    v[k][j] += __shfl_xor_sync(0xffffffffu, v[k][j], (int)off);
            if (off == 1) break;
        }
        if (lane < cols) {
#pragma unroll
            for (int k = 0; k < V; ++k)
#pragma unroll
                for (int j = 0; j < 2; ++j) red[(warp * g + cbase + k) * NR + j] = (double)v[k][j];
        }
        __syncthreads();
        // ---- CTA record per channel, pushed into every peer's record slots
        const uint32_t par = iter & 1u;
        if (tid < g) {
            double t0 = 0.0, t1 = 0.0;
            for (uint32_t w = 0; w < kNhwcThreads / 32; ++w) {
                t0 += red[(w * g + tid) * NR + 0];
                t1 += red[(w * g + tid) * NR + 1];
            }
            double r_[NR];
            if (PASS == 0) {
                const double Kc = (double)pshift[tid];
                const double n = (double)rows_valid;
                r_[0] = n;
                r_[1] = n * Kc + t0;
                r_[2] = t1 + 2.0 * Kc * t0 + n * Kc * Kc;
            } else {
                r_[0] = t0;
                r_[1] = t1;
            }
            double* dst = rec + ((par * K + rank) * g + tid) * NR;
            if (K > 1) {
                for (uint32_t pr = 0; pr < K; ++pr) {
                    uint32_t ra;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                                 : "=r"(ra)
                                 : "r"(smem_addr(dst)), "r"(pr));
#pragma unroll
                    for (int j = 0; j < NR; ++j)
                        asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra + 8u * j), "d"(r_[j])
                                     : "memory");
                }
            } else {
#pragma unroll
                for (int j = 0; j < NR; ++j) dst[j] = r_[j];
            }
        }
        if (iter == 0) trace(4);
        if (K > 1) {
            cluster_arrive_release();
            cluster_wait_acquire();
        } else {
            __syncthreads();
        }
        if (iter == 0) trace(5);
        // ---- fold the K records (rank order) and derive the coefficients
        if (tid < g) {
            double tot[NR];
#pragma unroll
            for (int j = 0; j < NR; ++j) tot[j] = 0.0;
#pragma unroll
            for (uint32_t pr = 0; pr < (uint32_t)kNhwcMaxK; ++pr)
                if (pr < K)
#pragma unroll
                    for (int j = 0; j < NR; ++j) tot[j] += rec[((par * K + pr) * g + tid) * NR + j];
            const int64_t c = (int64_t)c0 + tid;
            float* cf = coef + tid * 8;
            if (c < a.C) {
                if (PASS == 0) {
                    // fwd_coef_from_moments without its three divisions: the count is the
                    // layer's m (no sync here), 1/m from the host, rstd by rsqrt
                    const double mean = tot[1] * a.inv_m;
                    double var = fma(-mean, mean, tot[2] * a.inv_m);
                    var = var > 0.0 ? var : 0.0;
                    const double Ad = gamma_eff(pgam[tid], a.eps, a.flags) * rsqrt(var + (double)a.eps);
                    const float mu_hi = (float)mean;
                    const float4 f = make_float4((float)Ad, mu_hi, (float)(mean - (double)mu_hi), pbet[tid]);
                    // y = (x - mu_hi) A + (beta - mu_lo A)
                    cf[0] = f.x;
                    cf[1] = f.y;
                    cf[2] = fmaf(-f.z, f.x, f.w);
                    if (rank == 0) {
                        a.save_mean[c] = (float)mean;
                        a.save_var[c] = (float)var;
                        // update_running (kernels_stream.cuh) on the prefetched values
                        const double mo = (double)a.momentum;
                        if (a.running_mean)
                            a.running_mean[c] = (float)((1.0 - mo) * (double)prm[tid] + mo * mean);
                        if (a.running_var) {
                            const double cnt = (double)a.m;
                            const double vv = (a.flags & kRunVarBiased) ? var : var * cnt / (cnt - 1.0);
                            a.running_var[c] = (float)((1.0 - mo) * (double)prv[tid] + mo * vv);
                        }
                    }
                } else {
                    const double gg = gamma_eff(pgam[tid], a.eps, a.flags);
                    const double bet = (double)pbet[tid];
                    double S1 = tot[0], S2 = tot[1];
                    if (!(a.flags & kVariantI)) S2 = (S2 - bet * S1) / gg;  // BN-dagger
                    const double rstd = rsqrt((double)pvar[tid] + (double)a.eps);
                    const double rm = rstd * a.inv_m;
                    const float alpha = (float)(gg * rstd);
                    const float kappa = (float)(-rm * S2);
                    const float cc = (float)(rm * fma(S2, bet, -gg * S1));
                    cf[0] = alpha;
                    cf[1] = kappa;
                    cf[2] = alpha * slope;
                    cf[3] = kappa * inv_slope;
                    cf[4] = cc;
                    if (rank == 0) {
                        a.dbeta[c] = (float)S1;
                        a.dgamma[c] = (float)(gamma_sign(pgam[tid], a.flags) * S2);
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) cf[j] = 0.f;
            }
        }
        __syncthreads();
        if (iter == 0) trace(6);
        // ---- apply in place in the slab, then TMA stores
        if (PASS == 0) {
            float A[V], M[V], B[V];
#pragma unroll
            for (int k = 0; k < V; ++k) {
                A[k] = coef[(cbase + k) * 8 + 0];
                M[k] = coef[(cbase + k) * 8 + 1];
                B[k] = coef[(cbase + k) * 8 + 2];
            }
            auto app = [&](const uint32_t addr, const uint4 u) {
                float2 f[NP];
                Pairs<T>::load(u, f);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    float y0 = fmaf(f[p].x - M[2 * p], A[2 * p], B[2 * p]);
                    float y1 = fmaf(f[p].y - M[2 * p + 1], A[2 * p + 1], B[2 * p + 1]);
                    if constexpr (ACT != 0) {
                        f[p].x = Act<ACT>::f(y0);
                        f[p].y = Act<ACT>::f(y1);
                    } else {
                        f[p].x = y0 >= 0.f ? y0 : y0 * slope;
                        f[p].y = y1 >= 0.f ? y1 : y1 * slope;
                    }
                }
                const uint4 o = Pairs<T>::store(f);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(o.x),
                             "r"(o.y), "r"(o.z), "r"(o.w)
                             : "memory");
            };
            uint32_t r = trow;
            for (; r + rs < rows_valid; r += 2 * rs) {
                const uint32_t a0 = sbase0 + r * row_bytes + col * 16u, a1 = a0 + rs * row_bytes;
                const uint4 u0 = lds128(a0), u1 = lds128(a1);
                app(a0, u0);
                app(a1, u1);
            }
            if (r < rows_valid) {
                const uint32_t a0 = sbase0 + r * row_bytes + col * 16u;
                app(a0, lds128(a0));
            }
        } else {
            float al[V], ka[V], aln[V], kan[V], cc[V];
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const float* cf = coef + (cbase + k) * 8;
                al[k] = cf[0];
                ka[k] = cf[1];
                aln[k] = cf[2];
                kan[k] = cf[3];
                cc[k] = cf[4];
            }
            auto app = [&](const uint32_t off, const uint4 uz, const uint4 ud) {
                float2 zz[NP], dd[NP];
                Pairs<T>::load(uz, zz);
                Pairs<T>::load(ud, dd);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const int k0 = 2 * p, k1 = 2 * p + 1;
                    if constexpr (ACT != 0) {  // dx = alpha dy + kappa y + cc
                        dd[p].x = fmaf(al[k0], Act<ACT>::df(zz[p].x) * dd[p].x,
                                       fmaf(ka[k0], Act<ACT>::inv(zz[p].x), cc[k0]));
                        dd[p].y = fmaf(al[k1], Act<ACT>::df(zz[p].y) * dd[p].y,
                                       fmaf(ka[k1], Act<ACT>::inv(zz[p].y), cc[k1]));
                        continue;
                    }
                    dd[p].x = zz[p].x >= 0.f ? fmaf(al[k0], dd[p].x, fmaf(ka[k0], zz[p].x, cc[k0]))
                                             : fmaf(aln[k0], dd[p].x, fmaf(kan[k0], zz[p].x, cc[k0]));
                    dd[p].y = zz[p].y >= 0.f ? fmaf(al[k1], dd[p].y, fmaf(ka[k1], zz[p].y, cc[k1]))
                                             : fmaf(aln[k1], dd[p].y, fmaf(kan[k1], zz[p].y, cc[k1]));
                }
                const uint4 o = Pairs<T>::store(dd);
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(sbase1 + off),
                             "r"(o.x), "r"(o.y), "r"(o.z), "r"(o.w)
                             : "memory");
            };
            uint32_t r = trow;
            for (; r + rs < rows_valid; r += 2 * rs) {
                const uint32_t o0 = r * row_bytes + col * 16u, o1 = o0 + rs * row_bytes;
                const uint4 z0 = lds128(sbase0 + o0), d0 = lds128(sbase1 + o0);
                const uint4 z1 = lds128(sbase0 + o1), d1 = lds128(sbase1 + o1);
                app(o0, z0, d0);
                app(o1, z1, d1);
            }
            if (r < rows_valid) {
                const uint32_t o0 = r * row_bytes + col * 16u;
                app(o0, lds128(sbase0 + o0), lds128(sbase1 + o0));
            }
        }
        fence_proxy_async_smem();  // generic-proxy writes of the slab -> visible to TMA
        __syncthreads();
        if (iter == 0) trace(7);
        if (tid == 0) {
            unsigned char* src = PASS == 0 ? slab0 : slab1;
            for (uint32_t i = 0; i < nbox_valid; ++i)
                tma_store_2d(&tm_out, c0, (int32_t)(row0 + i * a.box_rows), src + i * box_bytes);
            bulk_commit();
        }
        if (iter == 0) trace(8);
    }
    // the slab must outlive the bulk stores' reads of it (their global writes complete
    // with the grid).  No exit barrier for the records: every peer stored its last
    // records before the last group's cluster barrier, which this CTA has passed.
    if (tid == 0) bulk_wait_read0();
    trace(9);
}

}  // namespace iabn
