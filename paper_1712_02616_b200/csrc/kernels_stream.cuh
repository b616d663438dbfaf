// kernels_stream.cuh -- streaming schedule of the InPlace-ABN hot path.
//
// Any layout / dtype / alignment.  Data are re-read after each global
// dependency (per-channel statistics before normalising, gradient sums before
// dx), so a pass over E elements of b bytes moves:
//   forward : stats (read E*b) + apply (read E*b, write E*b)           = 3*E*b
//   backward: reduce (read 2*E*b) + apply (read 2*E*b, write E*b)      = 5*E*b
// The channel-resident schedule (kernels_fused.cuh) does 2*E*b and 3*E*b.
//
// Numerics (R8): per-thread fp32 partial sums in several independent
// chains, shifted by a per-channel sample K (cancellation-free variance), flushed
// into fp64 every few vectors; fp64 block/cross-block/cross-GPU combines as raw
// moments (count, sum, sum of squares) -- deterministic trees, no atomics.
#pragma once

#include "common.cuh"

namespace iabn {

// Block coordinates of a kernel body: the hardware ones, or a virtual block of a
// persistent (cooperative) kernel that runs several phases in one launch.
struct Blk {
    uint32_t x, y, nx, ny;
};
__device__ __forceinline__ Blk hw_blk() { return {blockIdx.x, blockIdx.y, gridDim.x, gridDim.y}; }

// Coefficient loads: read-only path (NC) when the coefficients come from an earlier
// launch; a plain (coherent) load when a cooperative kernel wrote them in this launch
// (ordered after the writers by the grid barrier's acquire + bar.sync).
template <bool NC>
__device__ __forceinline__ float4 ld_coef(const float4* p) {
    if constexpr (NC) return __ldg(p);
    else return *p;
}

#ifndef IABN_STREAM_UNROLL
#define IABN_STREAM_UNROLL 4
#endif
constexpr int kUnroll = IABN_STREAM_UNROLL;  // independent 16-byte loads in flight per thread
#ifndef IABN_STAT_UNROLL
#define IABN_STAT_UNROLL 8
#endif
constexpr int kStatUnroll = IABN_STAT_UNROLL;  // statistics kernel (one input)
#ifndef IABN_NHWC_UNROLL
#define IABN_NHWC_UNROLL 4
#endif
constexpr int kNhwcUnroll = IABN_NHWC_UNROLL;  // NHWC reductions: rows in flight per thread
#ifndef IABN_NHWC_APPLY_UNROLL
#define IABN_NHWC_APPLY_UNROLL 8
#endif
// NHWC apply kernels: vectors in flight per thread (their register count caps the CTAs
// per SM at 3-4, so the bytes in flight come from the depth per thread)
constexpr int kNhwcApplyUnroll = IABN_NHWC_APPLY_UNROLL;

// Gamma reparametrisation (R4).
enum : uint32_t {
    kGammaPlain = 1u << 0,
    kGammaFixedOne = 1u << 1,
    kRunVarBiased = 1u << 2,
    kSyncGlobalGrads = 1u << 3,  // sync backward: dgamma/dbeta = the all-rank sums
    kVariantI = 1u << 5  // fused backward: per-element x^ products (Alg. 2 I) instead of BN-dagger sums
};

__device__ __forceinline__ double gamma_eff(float gamma, float eps, uint32_t flags) {
    if (flags & kGammaFixedOne) return 1.0;
    if (flags & kGammaPlain) return (double)gamma;
    return fabs((double)gamma) + (double)eps;
}
__device__ __forceinline__ double gamma_sign(float gamma, uint32_t flags) {
    if (flags & (kGammaFixedOne | kGammaPlain)) return 1.0;
    return gamma < 0.f ? -1.0 : 1.0;
}

// ====================================================================== F1: statistics
// Raw fp64 moments of a block's values v_i, accumulated as shifted sums about K:
//   count = n, sum = n K + S1, sumsq = S2 + 2 K S1 + n K^2,  S1 = sum (v-K), S2 = sum (v-K)^2
__device__ __forceinline__ void write_raw_moments(double* out, double n, double K, double S1,
                                                  double S2) {
    out[0] = n;
    out[1] = n * K + S1;
    out[2] = S2 + 2.0 * K * S1 + n * K * K;
}

// Offset (from the channel's first element) of channel-space element j = v*V of an
// NCHW channel, stepped by `step` elements at a time: at most one plane boundary per
// step when step <= HW (pointer arithmetic only), else by division.
struct PlaneCursor {
    int64_t off;
    uint32_t sp;  // offset within the plane
    __device__ __forceinline__ void seek(uint32_t j, const FastDiv& fd_hw, uint32_t HW,
                                         int64_t CHW) {
        const uint32_t n = fdiv(j, fd_hw);
        sp = j - n * HW;
        off = (int64_t)n * CHW + sp;
    }
    // advance by `step` elements to channel-space element j_next
    __device__ __forceinline__ void next(uint32_t step, uint32_t j_next, const FastDiv& fd_hw,
                                         uint32_t HW, int64_t CHW) {
        if (step <= HW) {
            sp += step;
            const bool wrap = sp >= HW;
            sp = wrap ? sp - HW : sp;
            off += wrap ? (int64_t)step + CHW - HW : (int64_t)step;
        } else {
            seek(j_next, fd_hw, HW, CHW);
        }
    }
};

// NCHW: grid (C, S); CTA (c, s) reduces channel-space [lo, hi) of m = N*HW values;
// channel-space index j lives at x[((j / HW) * C + c) * HW + j % HW].
template <typename T, bool VEC>
__device__ __forceinline__ void stats_nchw_body(const T* __restrict__ x, int64_t C, int64_t HW, uint32_t m, FastDiv fd_hw,
                      double* __restrict__ part,
        const Blk bk) {
    constexpr int V = VEC ? Elem<T>::kVec : 1;
    __shared__ double red[2 * kThreads / 32];
    const int64_t c = bk.x;
    const int S = bk.ny, s = bk.y;
    const uint32_t mv = m / V;
    const uint32_t vlo = (uint32_t)((uint64_t)mv * s / S), vhi = (uint32_t)((uint64_t)mv * (s + 1) / S);
    const float K = ld_scalar<T>(x + c * HW);
    const T* xc = x + c * HW;
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1 = 0.0, d2 = 0.0;
    int iter = 0;
    if constexpr (VEC) {
        // raw 16-byte loads first (kStatUnroll in flight per thread), unpacked and
        // shifted by K in the math loop (bf16: FHADD.BF16), fp32x2 chains
        constexpr int NP = Pairs<T>::kN;
        float2 s1[NP], s2[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) s1[i] = s2[i] = make_float2(0.f, 0.f);
        auto accumulate = [&](const uint4 rv) {
            float2 d[NP];
            Pairs<T>::load_sub(rv, K, d);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                s1[i] = add2(s1[i], d[i]);
                s2[i] = fma2(d[i], d[i], s2[i]);
            }
        };
        auto flush = [&]() {
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                d1 += (double)s1[i].x + (double)s1[i].y;
                d2 += (double)s2[i].x + (double)s2[i].y;
                s1[i] = s2[i] = make_float2(0.f, 0.f);
            }
        };
        const int64_t CHW = C * HW;
        const uint32_t step = kThreads * V;
        uint32_t v = vlo + threadIdx.x;
        PlaneCursor cur;
        cur.seek(v * V, fd_hw, (uint32_t)HW, CHW);
        for (; v + (kStatUnroll - 1) * kThreads < vhi;) {
            uint4 r[kStatUnroll];  // all in range: unpredicated loads, issued together
#pragma unroll
            for (int u = 0; u < kStatUnroll; ++u) {
                r[u] = ld_vec_ro(xc + cur.off);
                v += kThreads;
                cur.next(step, v * V, fd_hw, (uint32_t)HW, CHW);
            }
#pragma unroll
            for (int u = 0; u < kStatUnroll; ++u) accumulate(r[u]);
            if (++iter == 8) {
                iter = 0;
                flush();
            }
        }
        for (; v < vhi;) {
            accumulate(ld_vec_ro(xc + cur.off));
            v += kThreads;
            cur.next(step, v * V, fd_hw, (uint32_t)HW, CHW);
        }
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            d1 += (double)s1[i].x + (double)s1[i].y;
            d2 += (double)s2[i].x + (double)s2[i].y;
        }
    } else {
        for (uint32_t base = vlo + threadIdx.x; base < vhi; base += kThreads * kUnroll) {
            float f[kUnroll][V];
    #pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint32_t v = base + u * kThreads;
                if (v < vhi) {
                    const uint32_t j = v * V;
                    const uint32_t n = fdiv(j, fd_hw);
                    const T* p = xc + ((int64_t)n * C) * HW + (j - n * (uint32_t)HW);
                    if constexpr (VEC) {
                        unpack<T>(ld_vec(p), f[u]);
                    } else {
                        f[u][0] = ld_scalar<T>(p);
                    }
                } else {
    #pragma unroll
                    for (int k = 0; k < V; ++k) f[u][k] = K;
                }
            }
    #pragma unroll
            for (int u = 0; u < kUnroll; ++u)
    #pragma unroll
                for (int k = 0; k < V; ++k) {
                    const float dv = f[u][k] - K;
                    a1[k] += dv;
                    a2[k] = fmaf(dv, dv, a2[k]);
                }
            if (++iter == 16) {
                iter = 0;
    #pragma unroll
                for (int k = 0; k < V; ++k) {
                    d1 += a1[k];
                    d2 += a2[k];
                    a1[k] = a2[k] = 0.f;
                }
            }
        }
    #pragma unroll
        for (int k = 0; k < V; ++k) {
            d1 += a1[k];
            d2 += a2[k];
        }
    }
    double v2[2] = {d1, d2};
    block_sum<2>(v2, red);
    if (threadIdx.x == 0)
        write_raw_moments(part + ((int64_t)s * C + c) * 3, (double)(vhi - vlo) * V, K, v2[0],
                          v2[1]);
}
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads)
    stats_nchw_kernel(const T* __restrict__ x, int64_t C, int64_t HW, uint32_t m, FastDiv fd_hw,
                      double* __restrict__ part) {
    pdl_wait();
    stats_nchw_body<T, VEC>(x, C, HW, m, fd_hw, part, hw_blk());
}


// NHWC ([rows][C], rows = N*HW): block = 16 (channel groups of V) x 16 (rows);
// grid (ceil(C / (16 V)), S); CTA reduces rows [rlo, rhi) for 16*V channels.
template <typename T, bool VEC>
__device__ __forceinline__ void stats_nhwc_body(const T* __restrict__ x, int64_t C, int64_t rows, double* __restrict__ part,
        const Blk bk) {
    constexpr int V = VEC ? Elem<T>::kVec : 1;
    constexpr int CT = 16 * V;
    __shared__ double red[16][CT][2];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int S = bk.ny, s = bk.y;
    const int64_t c0 = (int64_t)bk.x * CT + tx * V;
    const int64_t rlo = rows * s / S, rhi = rows * (s + 1) / S;
    const bool active = c0 < C;
    float K[V];
#pragma unroll
    for (int k = 0; k < V; ++k) K[k] = (active && c0 + k < C) ? ld_scalar<T>(x + c0 + k) : 0.f;
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    // fp64 accumulators of this thread in its own slots of red (not registers: the
    // registers go to loads in flight)
    double* const d1 = &red[ty][tx * V][0];
#pragma unroll
    for (int k = 0; k < V; ++k) d1[2 * k] = d1[2 * k + 1] = 0.0;
    if (active) {
        int iter = 0;
        auto acc = [&](const float (&f)[V]) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const float dv = f[k] - K[k];
                a1[k] += dv;
                a2[k] = fmaf(dv, dv, a2[k]);
            }
        };
        auto flush = [&]() {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                d1[2 * k] += a1[k];
                d1[2 * k + 1] += a2[k];
                a1[k] = a2[k] = 0.f;
            }
        };
        int64_t r0 = rlo + ty;
        if constexpr (VEC) {
            // raw loads of kNhwcUnroll rows first (all in range), then the math
            for (; r0 + 16 * (kNhwcUnroll - 1) < rhi; r0 += 16 * kNhwcUnroll) {
                uint4 raw[kNhwcUnroll];
#pragma unroll
                for (int u = 0; u < kNhwcUnroll; ++u) raw[u] = ld_vec_ro(x + (r0 + 16 * u) * C + c0);
#pragma unroll
                for (int u = 0; u < kNhwcUnroll; ++u) {
                    float f[V];
                    unpack<T>(raw[u], f);
                    acc(f);
                }
                if (++iter == 4) {
                    iter = 0;
                    flush();
                }
            }
        }
        for (; r0 < rhi; r0 += 16) {
            float f[V];
            if constexpr (VEC) {
                unpack<T>(ld_vec_ro(x + r0 * C + c0), f);
            } else {
                f[0] = ld_scalar<T>(x + r0 * C + c0);
            }
            acc(f);
            if (++iter == 64) {
                iter = 0;
                flush();
            }
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        d1[2 * k] += a1[k];
        d1[2 * k + 1] += a2[k];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < CT) {
        const int64_t c = (int64_t)bk.x * CT + t;
        if (c < C) {
            double S1 = 0.0, S2 = 0.0;
            for (int y = 0; y < 16; ++y) {
                S1 += red[y][t][0];
                S2 += red[y][t][1];
            }
            const double Kc = (double)ld_scalar<T>(x + c);
            write_raw_moments(part + ((int64_t)s * C + c) * 3, (double)(rhi - rlo), Kc, S1, S2);
        }
    }
}
// NHWC reductions: minimum CTAs per SM for the register allocation (experiments; a
// cap of 3 or 4 spills in the bf16 kernels and measured slower than none)
#ifndef IABN_NHWC_MINB
#define IABN_NHWC_MINB 1
#endif
constexpr int kNhwcMinBlocks = IABN_NHWC_MINB;
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads, kNhwcMinBlocks)
    stats_nhwc_kernel(const T* __restrict__ x, int64_t C, int64_t rows, double* __restrict__ part) {
    pdl_wait();
    stats_nhwc_body<T, VEC>(x, C, rows, part, hw_blk());
}


// Sum S partial records of NV doubles per channel in fixed order: out[c][k].
// extra >= 0: out[NV*C] = extra (the count slot of the backward sums).
// Sum over the S split records of channel c: lane l of the channel's warp takes
// splits l, l+32, ... in order, then a fixed xor tree -- parallel and still the
// same order every run (bitwise reproducible).
template <int NV>
__device__ __forceinline__ void warp_split_sum(const double* __restrict__ part, int S, int64_t C,
                                               int64_t c, double (&acc)[NV]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 0; k < NV; ++k) acc[k] = 0.0;
    // 8 records per lane in flight (loads first, then the adds in the same order)
    for (int s0 = lane; s0 < S; s0 += 32 * 8) {
        double v[8][NV];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int s = s0 + 32 * u;
#pragma unroll
            for (int k = 0; k < NV; ++k)
                v[u][k] = s < S ? __ldcg(part + ((int64_t)s * C + c) * NV + k) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int k = 0; k < NV; ++k) acc[k] += v[u][k];
    }
#pragma unroll
    for (int k = 0; k < NV; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
}
// one warp per channel: blockDim.x = 128 -> 4 channels per block
__device__ __forceinline__ int64_t warp_channel() {
    return (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
}

template <int NV>
__global__ void combine_kernel(const double* __restrict__ part, int S, int64_t C,
                               double* __restrict__ out, double extra) {
    pdl_wait();
    const int64_t c = warp_channel();
    if (c == 0 && threadIdx.x == 0 && extra >= 0.0) out[NV * C] = extra;
    if (c >= C) return;
    double acc[NV];
    warp_split_sum<NV>(part, S, C, c, acc);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) out[c * NV + k] = acc[k];
}

// F1 finalize (+F1' running stats): from S partial raw moments per channel to
//   mean, biased var and the apply coefficients (A, mu_hi, mu_lo, beta) with
//   A = g rstd, so that y = ((x - mu_hi) - mu_lo) A + beta.  The mean is carried
//   as an fp32 pair: x - mu_hi is exact near the mean (Sterbenz), which keeps
//   x^ accurate when |mean| >> std (R8).
struct FwdCoefArgs {
    const double* part;
    int S;
    int64_t C;
    const float* gamma;
    const float* beta;
    float* running_mean;
    float* running_var;
    float* save_mean;
    float* save_var;
    float4* coef;
    float momentum, eps;
    uint32_t flags;
};

__device__ __forceinline__ float4 fwd_coef_from_moments(double cnt, double sum, double sumsq,
                                                        float gamma, float beta, float eps,
                                                        uint32_t flags, double* mean_out,
                                                        double* var_out) {
    const double mean = sum / cnt;
    double var = sumsq / cnt - mean * mean;
    var = var > 0.0 ? var : 0.0;
    const double rstd = 1.0 / sqrt(var + (double)eps);
    const double A = gamma_eff(gamma, eps, flags) * rstd;
    const float mu_hi = (float)mean;
    *mean_out = mean;
    *var_out = var;
    return make_float4((float)A, mu_hi, (float)(mean - (double)mu_hi), beta);
}

// y = ((x - mu_hi) - mu_lo) A + beta
// y = (x - mu_hi) A + (beta - mu_lo A): the same operations as the vectorised apply
// kernels (fwd_apply_rows / fwd_apply_nhwc / fused), so every schedule rounds alike
__device__ __forceinline__ float affine(float x, const float4& cf) {
    return fmaf(x - cf.y, cf.x, fmaf(-cf.z, cf.x, cf.w));
}

__device__ __forceinline__ void update_running(float* rm, float* rv, int64_t c, double mean,
                                               double var, double cnt, float momentum,
                                               uint32_t flags) {
    if (rm) rm[c] = (float)((1.0 - momentum) * (double)rm[c] + (double)momentum * mean);
    if (rv) {
        const double v = (flags & kRunVarBiased) ? var : var * cnt / (cnt - 1.0);
        rv[c] = (float)((1.0 - momentum) * (double)rv[c] + (double)momentum * v);
    }
}

// warp-level: all 32 lanes of the warp call it for channel c
__device__ __forceinline__ void fwd_coef_body(const FwdCoefArgs& a, int64_t c) {
    double acc[3];
    warp_split_sum<3>(a.part, a.S, a.C, c, acc);
    if (threadIdx.x & 31) return;
    const double cnt = acc[0], sum = acc[1], sumsq = acc[2];
    double mean, var;
    a.coef[c] = fwd_coef_from_moments(cnt, sum, sumsq, a.gamma[c], a.beta[c], a.eps, a.flags,
                                      &mean, &var);
    if (a.save_mean) a.save_mean[c] = (float)mean;
    if (a.save_var) a.save_var[c] = (float)var;
    update_running(a.running_mean, a.running_var, c, mean, var, cnt, a.momentum, a.flags);
}
__global__ void fwd_coef_kernel(FwdCoefArgs a) {
    pdl_wait();
    const int64_t c = warp_channel();
    if (c < a.C) fwd_coef_body(a, c);
}

// Eval mode: fixed running statistics.
__global__ void eval_coef_kernel(int64_t C, const float* __restrict__ gamma,
                                 const float* __restrict__ beta, const float* __restrict__ rm,
                                 const float* __restrict__ rv, float eps, uint32_t flags,
                                 float4* __restrict__ coef) {
    pdl_wait();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const double A = gamma_eff(gamma[c], eps, flags) / sqrt((double)rv[c] + (double)eps);
    coef[c] = make_float4((float)A, rm[c], 0.f, beta[c]);
}

// Eval forward without a coefficient launch: the apply kernels derive (A, mu, 0, beta)
// per channel from the running statistics themselves (fp32: A = g~ rsqrt(r_var + eps),
// within a few ulp of eval_coef_kernel's fp64 value).  r02: the extra launch cost
// 1-3 us per layer (32x512x14^2 bf16 eval forward 6.9 -> 5.8 us, NHWC 32x128x56^2
// 13.4 -> 10.2 us; a torch copy of the same tensors: 4.1 / 9.8 us).
struct EvalCoef {
    const float* gamma;
    const float* beta;
    const float* rm;
    const float* rv;
    float eps;
    uint32_t flags;
};
template <bool NC, bool EV>
__device__ __forceinline__ float4 get_coef(const float4* coef, const EvalCoef& ev, uint32_t c) {
    if constexpr (EV) {
        const float gm = __ldg(ev.gamma + c);
        const float g = (ev.flags & kGammaFixedOne) ? 1.f : (ev.flags & kGammaPlain) ? gm : fabsf(gm) + ev.eps;
        return make_float4(g * rsqrtf(__ldg(ev.rv + c) + ev.eps), __ldg(ev.rm + c), 0.f, __ldg(ev.beta + c));
    } else {
        return ld_coef<NC>(coef + c);
    }
}

// ====================================================================== elementwise passes
// Channel of flat element e (e < 2^32 within one launch; the host splits the
// tensor into whole-sample chunks).
template <int LAYOUT>
__device__ __forceinline__ uint32_t channel_of(uint32_t e, const FastDiv& fd_hw,
                                               const FastDiv& fd_c) {
    if (LAYOUT == 0) {  // NCHW
        const uint32_t p = fdiv(e, fd_hw);
        return p - fdiv(p, fd_c) * fd_c.d;
    }
    return e - fdiv(e, fd_c) * fd_c.d;  // NHWC
}

__device__ __forceinline__ float leaky(float y, float slope) { return y >= 0.f ? y : y * slope; }

// F2: z = f(y), y = ((x - mu_hi) - mu_lo) A + beta, in place allowed (each
// element is read then written by the same thread).  ALIGNED: NCHW with HW*b a
// multiple of 16 (a 16-byte vector lies in one channel) or NHWC with C*b a
// multiple of 16 (a vector holds channels c0 .. c0+V-1); otherwise the channel
// is resolved per element.
template <typename T, int LAYOUT, bool ALIGNED, bool NC = true, bool EV = false>
__device__ __forceinline__ void fwd_apply_body(const T* x, T* z, const float4* __restrict__ coef, uint32_t E, FastDiv fd_hw,
                     FastDiv fd_c, float slope,
        const Blk bk, const EvalCoef& ev = EvalCoef{}) {
    constexpr int V = Elem<T>::kVec;
    const uint32_t nvec = E / V;
    const uint32_t stride = bk.nx * kThreads;
    for (uint32_t base = bk.x * kThreads + threadIdx.x; base < nvec;
         base += stride * kUnroll) {
        uint4 r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) r[u] = ld_vec(x + (size_t)v * V);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                float f[V];
                unpack<T>(r[u], f);
                const uint32_t e = v * V;
                if (ALIGNED && LAYOUT == 0) {  // NCHW: the vector lies in one channel
                    const float4 cf = get_coef<NC, EV>(coef, ev, channel_of<LAYOUT>(e, fd_hw, fd_c));
#pragma unroll
                    for (int k = 0; k < V; ++k) f[k] = leaky(affine(f[k], cf), slope);
                } else if (ALIGNED) {  // NHWC, C % V == 0: channels c0 .. c0+V-1
                    const uint32_t c0 = channel_of<LAYOUT>(e, fd_hw, fd_c);
#pragma unroll
                    for (int k = 0; k < V; ++k) f[k] = leaky(affine(f[k], get_coef<NC, EV>(coef, ev, c0 + k)), slope);
                } else {
#pragma unroll
                    for (int k = 0; k < V; ++k) {
                        const float4 cf = get_coef<NC, EV>(coef, ev, channel_of<LAYOUT>(e + k, fd_hw, fd_c));
                        f[k] = leaky(affine(f[k], cf), slope);
                    }
                }
                st_vec(z + (size_t)v * V, pack<T>(f));
            }
        }
    }
    // tail (E % V elements) by the first threads of block 0
    if (bk.x == 0 && threadIdx.x < E - nvec * V) {
        const uint32_t e = nvec * V + threadIdx.x;
        const float4 cf = get_coef<false, EV>(coef, ev, channel_of<LAYOUT>(e, fd_hw, fd_c));
        st_scalar<T>(z + e, leaky(affine(ld_scalar<T>(x + e), cf), slope));
    }
}
template <typename T, int LAYOUT, bool ALIGNED, bool EV = false>
__global__ void __launch_bounds__(kThreads)
    fwd_apply_kernel(const T* x, T* z, const float4* __restrict__ coef, uint32_t E, FastDiv fd_hw,
                     FastDiv fd_c, float slope, EvalCoef ev) {
    pdl_wait();
    fwd_apply_body<T, LAYOUT, ALIGNED, true, EV>(x, z, coef, E, fd_hw, fd_c, slope, hw_blk(), ev);
}


// F2 for NCHW with HW >= V (any alignment): a grid-stride walk over 16-byte vectors
// (the whole grid sweeps one contiguous window at a time) with a (plane offset,
// channel) cursor advanced by the fixed stride -- no divisions in the loop -- and
// kUnroll loads issued before the math.  A vector that straddles two planes (HW*b
// not a multiple of 16) takes its tail elements' coefficients from the next channel.
// y = (x - mu_hi) A + (beta - mu_lo A), z = max(y, a y).
template <typename T, bool NC = true, bool EV = false>
__device__ __forceinline__ void fwd_apply_rows_body(const T* x, T* z, const float4* __restrict__ coef,
                                                    uint32_t E, uint32_t HW, uint32_t C,
                                                    FastDiv fd_hw, FastDiv fd_c, float slope,
                                                    const Blk bk, const EvalCoef& ev = EvalCoef{}) {
    constexpr int V = Elem<T>::kVec;
    constexpr int NP = Pairs<T>::kN;
    const uint32_t nvec = E / V;
    const uint32_t stride = bk.nx * kThreads;  // vectors
    uint32_t v = bk.x * kThreads + threadIdx.x;
    if (bk.x == 0 && threadIdx.x < E - nvec * V) {  // tail elements
        const uint32_t e = nvec * V + threadIdx.x;
        const float4 cf = get_coef<NC, EV>(coef, ev, channel_of<0>(e, fd_hw, fd_c));
        st_scalar<T>(z + e, leaky(affine(ld_scalar<T>(x + e), cf), slope));
    }
    if (v >= nvec) return;
    // cursor of element e = v V: plane offset sp, channel c; one stride = q planes + rr
    const uint32_t se = stride * V;
    const uint32_t q = fdiv(se, fd_hw), rr = se - q * HW;
    const uint32_t qc = q - fdiv(q, fd_c) * C;
    uint32_t row = fdiv(v * V, fd_hw);
    uint32_t sp = v * V - row * HW;
    uint32_t c = row - fdiv(row, fd_c) * C;
    const float2 sl2 = make_float2(slope, slope);
    auto apply = [&](const uint4 r, const uint32_t cc, const uint32_t spv, const uint32_t vv) {
        const float4 cf = get_coef<NC, EV>(coef, ev, cc);  // (A, mu_hi, mu_lo, beta)
        const float bp = fmaf(-cf.z, cf.x, cf.w);
        if (spv + V <= HW) {
            const float2 A2 = make_float2(cf.x, cf.x), B2 = make_float2(bp, bp);
            float2 w[NP];
            Pairs<T>::load_sub(r, cf.y, w);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                const float2 y = fma2(w[i], A2, B2);
                const float2 ay = mul2(y, sl2);
                w[i] = make_float2(fmaxf(y.x, ay.x), fmaxf(y.y, ay.y));
            }
            st_vec(z + (size_t)vv * V, Pairs<T>::store(w));
        } else {  // elements k >= HW - spv belong to the next channel
            const float4 cf2 = get_coef<NC, EV>(coef, ev, cc + 1 == C ? 0 : cc + 1);
            const float bp2 = fmaf(-cf2.z, cf2.x, cf2.w);
            const uint32_t kb = HW - spv;
            float f[V];
            unpack<T>(r, f);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const bool first = (uint32_t)k < kb;
                const float y = fmaf(f[k] - (first ? cf.y : cf2.y), first ? cf.x : cf2.x,
                                     first ? bp : bp2);
                f[k] = fmaxf(y, y * slope);
            }
            st_vec(z + (size_t)vv * V, pack<T>(f));
        }
    };
    auto advance = [&]() {
        v += stride;
        sp += rr;
        const bool carry = sp >= HW;
        sp = carry ? sp - HW : sp;
        c += qc + (carry ? 1u : 0u);
        c = c >= C ? c - C : c;
    };
    for (; v + (kUnroll - 1) * stride < nvec;) {
        uint4 r[kUnroll];
        uint32_t cu[kUnroll], su[kUnroll], vu[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            r[u] = ld_vec(x + (size_t)v * V);
            cu[u] = c;
            su[u] = sp;
            vu[u] = v;
            advance();
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) apply(r[u], cu[u], su[u], vu[u]);
    }
    for (; v < nvec;) {
        const uint4 r = ld_vec(x + (size_t)v * V);
        const uint32_t cc = c, ss = sp, vv = v;
        advance();
        apply(r, cc, ss, vv);
    }
}
template <typename T, bool EV = false>
__global__ void __launch_bounds__(kThreads)
    fwd_apply_rows_kernel(const T* x, T* z, const float4* __restrict__ coef, uint32_t E,
                          uint32_t HW, uint32_t C, FastDiv fd_hw, FastDiv fd_c, float slope,
                          EvalCoef ev) {
    pdl_wait();
    fwd_apply_rows_body<T, true, EV>(x, z, coef, E, HW, C, fd_hw, fd_c, slope, hw_blk(), ev);
}

// ====================================================================== B1: gradient sums
// Per element (Alg. 2 l.2-5): dy = f'(z) dz, y = f^-1(z),
// x^ = (y - beta)/g = y * inv_g + nb;  per channel S1 = sum dy, S2 = sum dy x^.
struct InvAffine {
    float inv_g, nb;
};
__device__ __forceinline__ InvAffine inv_affine(float gamma, float beta, float eps, uint32_t flags) {
    const double g = gamma_eff(gamma, eps, flags);
    return {(float)(1.0 / g), (float)(-(double)beta / g)};
}

__device__ __forceinline__ void grad_terms(float z, float dz, float slope, float inv_slope,
                                           InvAffine ia, float& dy, float& xh) {
    const bool pos = z >= 0.f;  // sign(z) = sign(y) for slope > 0; -0.0 counts as >= 0
    const float y = pos ? z : z * inv_slope;
    dy = pos ? dz : dz * slope;
    xh = fmaf(y, ia.inv_g, ia.nb);
}

template <typename T, bool VEC>
__device__ __forceinline__ void bwd_reduce_nchw_body(const T* __restrict__ z, const T* __restrict__ dz,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           int64_t C, int64_t HW, uint32_t m, FastDiv fd_hw, float eps,
                           float slope, float inv_slope, uint32_t flags,
                           double* __restrict__ part,
        const Blk bk) {
    constexpr int V = VEC ? Elem<T>::kVec : 1;
    __shared__ double red[2 * kThreads / 32];
    const int64_t c = bk.x;
    const int S = bk.ny, s = bk.y;
    const uint32_t mv = m / V;
    const uint32_t vlo = (uint32_t)((uint64_t)mv * s / S), vhi = (uint32_t)((uint64_t)mv * (s + 1) / S);
    const InvAffine ia = inv_affine(gamma[c], beta[c], eps, flags);
    const T* zc = z + c * HW;
    const T* dzc = dz + c * HW;
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1 = 0.0, d2 = 0.0;
    int iter = 0;
    if constexpr (VEC) {
        // raw 16-byte loads of z and dz first (2 x kUnroll in flight), plane cursor
        const int64_t CHW = C * HW;
        const uint32_t step = kThreads * V;
        uint32_t v = vlo + threadIdx.x;
        PlaneCursor cur;
        cur.seek(v * V, fd_hw, (uint32_t)HW, CHW);
        auto accumulate = [&](const uint4 rz, const uint4 rd) {
            float fz[V], fd[V];
            unpack<T>(rz, fz);
            unpack<T>(rd, fd);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                float dy, xh;
                grad_terms(fz[k], fd[k], slope, inv_slope, ia, dy, xh);
                a1[k] += dy;
                a2[k] = fmaf(dy, xh, a2[k]);
            }
        };
        for (; v + (kUnroll - 1) * kThreads < vhi;) {
            uint4 rz[kUnroll], rd[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                rz[u] = ld_vec_ro(zc + cur.off);
                rd[u] = ld_vec_ro(dzc + cur.off);
                v += kThreads;
                cur.next(step, v * V, fd_hw, (uint32_t)HW, CHW);
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) accumulate(rz[u], rd[u]);
            if (++iter == 16) {
                iter = 0;
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    d1 += a1[k];
                    d2 += a2[k];
                    a1[k] = a2[k] = 0.f;
                }
            }
        }
        for (; v < vhi;) {
            accumulate(ld_vec_ro(zc + cur.off), ld_vec_ro(dzc + cur.off));
            v += kThreads;
            cur.next(step, v * V, fd_hw, (uint32_t)HW, CHW);
        }
    } else {
        for (uint32_t base = vlo + threadIdx.x; base < vhi; base += kThreads * kUnroll) {
            float fz[kUnroll][V], fd[kUnroll][V];
    #pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint32_t v = base + u * kThreads;
                if (v < vhi) {
                    const uint32_t j = v * V;
                    const uint32_t n = fdiv(j, fd_hw);
                    const int64_t off = ((int64_t)n * C) * HW + (j - n * (uint32_t)HW);
                    if constexpr (VEC) {
                        unpack<T>(ld_vec(zc + off), fz[u]);
                        unpack<T>(ld_vec(dzc + off), fd[u]);
                    } else {
                        fz[u][0] = ld_scalar<T>(zc + off);
                        fd[u][0] = ld_scalar<T>(dzc + off);
                    }
                } else {
    #pragma unroll
                    for (int k = 0; k < V; ++k) fz[u][k] = fd[u][k] = 0.f;
                }
            }
    #pragma unroll
            for (int u = 0; u < kUnroll; ++u)
    #pragma unroll
                for (int k = 0; k < V; ++k) {
                    float dy, xh;
                    grad_terms(fz[u][k], fd[u][k], slope, inv_slope, ia, dy, xh);
                    a1[k] += dy;
                    a2[k] = fmaf(dy, xh, a2[k]);
                }
            if (++iter == 16) {
                iter = 0;
    #pragma unroll
                for (int k = 0; k < V; ++k) {
                    d1 += a1[k];
                    d2 += a2[k];
                    a1[k] = a2[k] = 0.f;
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        d1 += a1[k];
        d2 += a2[k];
    }
    double v2[2] = {d1, d2};
    block_sum<2>(v2, red);
    if (threadIdx.x == 0) {
        double* o = part + ((int64_t)s * C + c) * 2;
        o[0] = v2[0];
        o[1] = v2[1];
    }
}
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads)
    bwd_reduce_nchw_kernel(const T* __restrict__ z, const T* __restrict__ dz,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           int64_t C, int64_t HW, uint32_t m, FastDiv fd_hw, float eps,
                           float slope, float inv_slope, uint32_t flags,
                           double* __restrict__ part) {
    pdl_wait();
    bwd_reduce_nchw_body<T, VEC>(z, dz, gamma, beta, C, HW, m, fd_hw, eps, slope, inv_slope, flags, part, hw_blk());
}


template <typename T, bool VEC>
__device__ __forceinline__ void bwd_reduce_nhwc_body(const T* __restrict__ z, const T* __restrict__ dz,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           int64_t C, int64_t rows, float eps, float slope, float inv_slope,
                           uint32_t flags, double* __restrict__ part,
        const Blk bk) {
    constexpr int V = VEC ? Elem<T>::kVec : 1;
    constexpr int CT = 16 * V;
    __shared__ double red[16][CT][2];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int S = bk.ny, s = bk.y;
    const int64_t c0 = (int64_t)bk.x * CT + tx * V;
    const int64_t rlo = rows * s / S, rhi = rows * (s + 1) / S;
    const bool active = c0 < C;
    constexpr int kBU = kNhwcUnroll / 2 > 0 ? kNhwcUnroll / 2 : 1;  // two inputs per row
    InvAffine ia[V];
#pragma unroll
    for (int k = 0; k < V; ++k)
        ia[k] = (active && c0 + k < C) ? inv_affine(gamma[c0 + k], beta[c0 + k], eps, flags)
                                       : InvAffine{0.f, 0.f};
    float a1[V], a2[V];
    // fp64 accumulators of this thread in its own slots of red (registers go to loads)
    double* const d1 = &red[ty][tx * V][0];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        a1[k] = a2[k] = 0.f;
        d1[2 * k] = d1[2 * k + 1] = 0.0;
    }
    if (active) {
        int iter = 0;
        auto acc = [&](const float (&fz)[V], const float (&fd)[V]) {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                float dy, xh;
                grad_terms(fz[k], fd[k], slope, inv_slope, ia[k], dy, xh);
                a1[k] += dy;
                a2[k] = fmaf(dy, xh, a2[k]);
            }
        };
        auto flush = [&]() {
#pragma unroll
            for (int k = 0; k < V; ++k) {
                d1[2 * k] += a1[k];
                d1[2 * k + 1] += a2[k];
                a1[k] = a2[k] = 0.f;
            }
        };
        int64_t r0 = rlo + ty;
        if constexpr (VEC) {
            // raw loads of z and dz for kBU rows first (all in range), then the math
            for (; r0 + 16 * (kBU - 1) < rhi; r0 += 16 * kBU) {
                uint4 rz[kBU], rd[kBU];
#pragma unroll
                for (int u = 0; u < kBU; ++u) {
                    rz[u] = ld_vec_ro(z + (r0 + 16 * u) * C + c0);
                    rd[u] = ld_vec_ro(dz + (r0 + 16 * u) * C + c0);
                }
#pragma unroll
                for (int u = 0; u < kBU; ++u) {
                    float fz[V], fd[V];
                    unpack<T>(rz[u], fz);
                    unpack<T>(rd[u], fd);
                    acc(fz, fd);
                }
                if (++iter == 4) {
                    iter = 0;
                    flush();
                }
            }
        }
        for (; r0 < rhi; r0 += 16) {
            float fz[V], fd[V];
            const int64_t off = r0 * C + c0;
            if constexpr (VEC) {
                unpack<T>(ld_vec_ro(z + off), fz);
                unpack<T>(ld_vec_ro(dz + off), fd);
            } else {
                fz[0] = ld_scalar<T>(z + off);
                fd[0] = ld_scalar<T>(dz + off);
            }
            acc(fz, fd);
            if (++iter == 16) {
                iter = 0;
                flush();
            }
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        d1[2 * k] += a1[k];
        d1[2 * k + 1] += a2[k];
    }
    __syncthreads();
    const int t = threadIdx.x;
    if (t < CT) {
        const int64_t c = (int64_t)bk.x * CT + t;
        if (c < C) {
            double S1 = 0.0, S2 = 0.0;
            for (int y = 0; y < 16; ++y) {
                S1 += red[y][t][0];
                S2 += red[y][t][1];
            }
            double* o = part + ((int64_t)s * C + c) * 2;
            o[0] = S1;
            o[1] = S2;
        }
    }
}
template <typename T, bool VEC>
__global__ void __launch_bounds__(kThreads, kNhwcMinBlocks)
    bwd_reduce_nhwc_kernel(const T* __restrict__ z, const T* __restrict__ dz,
                           const float* __restrict__ gamma, const float* __restrict__ beta,
                           int64_t C, int64_t rows, float eps, float slope, float inv_slope,
                           uint32_t flags, double* __restrict__ part) {
    pdl_wait();
    bwd_reduce_nhwc_body<T, VEC>(z, dz, gamma, beta, C, rows, eps, slope, inv_slope, flags, part, hw_blk());
}


// B2 coefficients (refolded in y):
//   dx = g rstd (dy - x^ S2/m - S1/m),  x^ = (y - beta)/g
//      = alpha dy + kappa y + cc,  alpha = g rstd, kappa = -rstd S2/m,
//        cc = rstd (S2/m) beta - g rstd S1/m
// S1, S2, m: global (all ranks) sums; dgamma/dbeta from the local or global sums.
struct BwdCoefArgs {
    const double* glob;  // [S_glob][C][2]
    int S_glob;
    const double* loc;  // [S_loc][C][2]
    int S_loc;
    const double* count_ptr;  // device count (sync) or nullptr
    double count;             // used when count_ptr == nullptr
    int64_t C;
    const float* gamma;
    const float* beta;
    const float* save_var;
    float* dgamma;
    float* dbeta;
    float4* coef;
    float eps;
    uint32_t flags;
};

__device__ __forceinline__ float4 bwd_coef_from_sums(double S1, double S2, double m, float gamma,
                                                     float beta, float var, float eps,
                                                     uint32_t flags) {
    const double g = gamma_eff(gamma, eps, flags);
    const double rstd = 1.0 / sqrt((double)var + (double)eps);
    const double alpha = g * rstd;
    const double kappa = -rstd * S2 / m;
    const double cc = rstd * (S2 / m) * (double)beta - g * rstd * S1 / m;
    return make_float4((float)alpha, (float)kappa, (float)cc, 0.f);
}

// warp-level: all 32 lanes of the warp call it for channel c
__device__ __forceinline__ void bwd_coef_body(const BwdCoefArgs& a, int64_t c) {
    double gs[2], ls[2];
    warp_split_sum<2>(a.glob, a.S_glob, a.C, c, gs);
    if (a.loc == a.glob) {
        ls[0] = gs[0];
        ls[1] = gs[1];
    } else {
        warp_split_sum<2>(a.loc, a.S_loc, a.C, c, ls);
    }
    if (threadIdx.x & 31) return;
    const double g1 = gs[0], g2 = gs[1], l1 = ls[0], l2 = ls[1];
    const double m = a.count_ptr ? *a.count_ptr : a.count;
    a.coef[c] = bwd_coef_from_sums(g1, g2, m, a.gamma[c], a.beta[c], a.save_var[c], a.eps, a.flags);
    a.dbeta[c] = (float)l1;
    a.dgamma[c] = (float)(gamma_sign(a.gamma[c], a.flags) * l2);
}
__global__ void bwd_coef_kernel(BwdCoefArgs a) {
    pdl_wait();
    const int64_t c = warp_channel();
    if (c < a.C) bwd_coef_body(a, c);
}

// B2: dx = alpha dy + kappa y + cc, dx may alias dz.
template <typename T, int LAYOUT, bool ALIGNED, bool NC = true>
__device__ __forceinline__ void bwd_apply_body(const T* __restrict__ z, const T* dz, T* dx, const float4* __restrict__ coef,
                     uint32_t E, FastDiv fd_hw, FastDiv fd_c, float slope, float inv_slope,
        const Blk bk) {
    constexpr int V = Elem<T>::kVec;
    const uint32_t nvec = E / V;
    const uint32_t stride = bk.nx * kThreads;
    for (uint32_t base = bk.x * kThreads + threadIdx.x; base < nvec;
         base += stride * kUnroll) {
        uint4 rz[kUnroll], rd[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                rz[u] = ld_vec(z + (size_t)v * V);
                rd[u] = ld_vec(dz + (size_t)v * V);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                float fz[V], fd[V];
                unpack<T>(rz[u], fz);
                unpack<T>(rd[u], fd);
                const uint32_t e = v * V;
                float4 cf;
                uint32_t c0 = 0;
                if (ALIGNED) c0 = channel_of<LAYOUT>(e, fd_hw, fd_c);
                if (ALIGNED && LAYOUT == 0) cf = ld_coef<NC>(coef + c0);  // NCHW: one channel
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    if (ALIGNED && LAYOUT == 1) cf = ld_coef<NC>(coef + c0 + k);  // NHWC: c0 + k
                    if (!ALIGNED) cf = ld_coef<NC>(coef + channel_of<LAYOUT>(e + k, fd_hw, fd_c));
                    const bool pos = fz[k] >= 0.f;
                    const float y = pos ? fz[k] : fz[k] * inv_slope;
                    const float dy = pos ? fd[k] : fd[k] * slope;
                    fz[k] = fmaf(cf.x, dy, fmaf(cf.y, y, cf.z));
                }
                st_vec(dx + (size_t)v * V, pack<T>(fz));
            }
        }
    }
    if (bk.x == 0 && threadIdx.x < E - nvec * V) {
        const uint32_t e = nvec * V + threadIdx.x;
        const float4 cf = coef[channel_of<LAYOUT>(e, fd_hw, fd_c)];
        const float zz = ld_scalar<T>(z + e), dd = ld_scalar<T>(dz + e);
        const bool pos = zz >= 0.f;
        const float y = pos ? zz : zz * inv_slope;
        const float dy = pos ? dd : dd * slope;
        st_scalar<T>(dx + e, fmaf(cf.x, dy, fmaf(cf.y, y, cf.z)));
    }
}
template <typename T, int LAYOUT, bool ALIGNED>
__global__ void __launch_bounds__(kThreads)
    bwd_apply_kernel(const T* __restrict__ z, const T* dz, T* dx, const float4* __restrict__ coef,
                     uint32_t E, FastDiv fd_hw, FastDiv fd_c, float slope, float inv_slope) {
    pdl_wait();
    bwd_apply_body<T, LAYOUT, ALIGNED>(z, dz, dx, coef, E, fd_hw, fd_c, slope, inv_slope, hw_blk());
}


// B2 for NCHW with HW >= V (any alignment): the stride cursor of fwd_apply_rows_body;
// dx = al dy + ka y + cc with (al, ka, cc) of the element's channel.
template <typename T, bool NC = true>
__device__ __forceinline__ void bwd_apply_rows_body(const T* __restrict__ z, const T* dz, T* dx,
                                                    const float4* __restrict__ coef, uint32_t E,
                                                    uint32_t HW, uint32_t C, FastDiv fd_hw,
                                                    FastDiv fd_c, float slope, float inv_slope,
                                                    const Blk bk) {
    constexpr int V = Elem<T>::kVec;
    const uint32_t nvec = E / V;
    const uint32_t stride = bk.nx * kThreads;
    uint32_t v = bk.x * kThreads + threadIdx.x;
    auto grad = [&](float zz, float dd, const float4& cf) {
        const bool pos = zz >= 0.f;  // -0.0 counts as >= 0
        const float y = pos ? zz : zz * inv_slope;
        const float dy = pos ? dd : dd * slope;
        return fmaf(cf.x, dy, fmaf(cf.y, y, cf.z));
    };
    if (bk.x == 0 && threadIdx.x < E - nvec * V) {  // tail elements
        const uint32_t e = nvec * V + threadIdx.x;
        const float4 cf = ld_coef<NC>(coef + channel_of<0>(e, fd_hw, fd_c));
        st_scalar<T>(dx + e, grad(ld_scalar<T>(z + e), ld_scalar<T>(dz + e), cf));
    }
    if (v >= nvec) return;
    const uint32_t se = stride * V;
    const uint32_t q = fdiv(se, fd_hw), rr = se - q * HW;
    const uint32_t qc = q - fdiv(q, fd_c) * C;
    uint32_t row = fdiv(v * V, fd_hw);
    uint32_t sp = v * V - row * HW;
    uint32_t c = row - fdiv(row, fd_c) * C;
    auto apply = [&](const uint4 rz, const uint4 rd, const uint32_t cc, const uint32_t spv,
                     const uint32_t vv) {
        const float4 cf = ld_coef<NC>(coef + cc);
        const float4 cf2 = spv + V <= HW ? cf : ld_coef<NC>(coef + (cc + 1 == C ? 0 : cc + 1));
        const uint32_t kb = HW - spv;  // elements k >= kb belong to the next channel
        float fz[V], fd[V];
        unpack<T>(rz, fz);
        unpack<T>(rd, fd);
#pragma unroll
        for (int k = 0; k < V; ++k) fz[k] = grad(fz[k], fd[k], (uint32_t)k < kb ? cf : cf2);
        st_vec(dx + (size_t)vv * V, pack<T>(fz));
    };
    auto advance = [&]() {
        v += stride;
        sp += rr;
        const bool carry = sp >= HW;
        sp = carry ? sp - HW : sp;
        c += qc + (carry ? 1u : 0u);
        c = c >= C ? c - C : c;
    };
    for (; v + (kUnroll - 1) * stride < nvec;) {
        uint4 rz[kUnroll], rd[kUnroll];
        uint32_t cu[kUnroll], su[kUnroll], vu[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            rz[u] = ld_vec(z + (size_t)v * V);
            rd[u] = ld_vec(dz + (size_t)v * V);
            cu[u] = c;
            su[u] = sp;
            vu[u] = v;
            advance();
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) apply(rz[u], rd[u], cu[u], su[u], vu[u]);
    }
    for (; v < nvec;) {
        const uint4 rz = ld_vec(z + (size_t)v * V), rd = ld_vec(dz + (size_t)v * V);
        const uint32_t cc = c, ss = sp, vv = v;
        advance();
        apply(rz, rd, cc, ss, vv);
    }
}
template <typename T>
__global__ void __launch_bounds__(kThreads)
    bwd_apply_rows_kernel(const T* __restrict__ z, const T* dz, T* dx,
                          const float4* __restrict__ coef, uint32_t E, uint32_t HW, uint32_t C,
                          FastDiv fd_hw, FastDiv fd_c, float slope, float inv_slope) {
    pdl_wait();
    bwd_apply_rows_body<T>(z, dz, dx, coef, E, HW, C, fd_hw, fd_c, slope, inv_slope, hw_blk());
}

// ====================================================================== misaligned NCHW reductions
// NCHW with HW*b not a multiple of 16 (e.g. bf16 14x14: 392-byte planes): plane n of
// channel c starts at element P = (n C + c) HW, not on a 16-byte boundary.  Each plane
// is read as the aligned 16-byte vectors that cover it (at most W = HW/V + 2), the
// elements outside [P, P + HW) masked out -- full-width loads, a few neighbour bytes
// per plane (served by L2).  Work item u = n W + i: vector i of plane n; split s of S
// takes items [N W s / S, N W (s+1) / S).  PASS 0: raw moments (count, sum, sum of
// squares) shifted by K; PASS 1: (sum dy, sum dy x^) as bwd_reduce_nchw_body.
template <typename T, int PASS>
__device__ __forceinline__ void nchw_cover_body(const T* __restrict__ in0, const T* __restrict__ in1,
                                                const float* __restrict__ gamma,
                                                const float* __restrict__ beta, int64_t C,
                                                int64_t HW, int64_t N, int64_t E, float eps,
                                                float slope, float inv_slope, uint32_t flags,
                                                FastDiv fdw, double* __restrict__ part,
                                                const Blk bk) {
    constexpr int V = Elem<T>::kVec;
    __shared__ double red[3 * kThreads / 32];
    const int64_t c = bk.x;
    const int S = bk.ny, s = bk.y;
    const uint32_t W = fdw.d;  // HW / V + 2 covering vectors per plane
    const uint64_t items = (uint64_t)N * W;
    const uint32_t ulo = (uint32_t)(items * s / S), uhi = (uint32_t)(items * (s + 1) / S);
    const float K = PASS == 0 ? ld_scalar<T>(in0 + c * HW) : 0.f;
    InvAffine ia{0.f, 0.f};
    if (PASS == 1) ia = inv_affine(gamma[c], beta[c], eps, flags);
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1 = 0.0, d2 = 0.0;
    uint32_t cnt = 0;
    int iter = 0;
    for (uint32_t u0 = ulo + threadIdx.x; u0 < uhi; u0 += kThreads * kUnroll) {
        uint4 r0[kUnroll], r1[kUnroll];
        int64_t e0[kUnroll], p0[kUnroll];
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            const uint32_t u = u0 + q * kThreads;
            const uint32_t n = fdiv(u, fdw), i = u - n * W;
            const int64_t P = ((int64_t)n * C + c) * HW;
            const int64_t ev = (P / V + i) * V;  // first element of the covering vector
            p0[q] = P;
            e0[q] = (u < uhi && ev < P + HW) ? ev : -1;
            if (e0[q] >= 0 && ev + V <= E) {
                r0[q] = ld_vec_ro(in0 + ev);
                if (PASS == 1) r1[q] = ld_vec_ro(in1 + ev);
            } else if (e0[q] >= 0) {  // the tensor's last, partial vector
                float f0[V], f1[V];
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    f0[k] = ev + k < E ? ld_scalar<T>(in0 + ev + k) : 0.f;
                    f1[k] = (PASS == 1 && ev + k < E) ? ld_scalar<T>(in1 + ev + k) : 0.f;
                }
                r0[q] = pack<T>(f0);
                r1[q] = pack<T>(f1);
            }
        }
#pragma unroll
        for (int q = 0; q < kUnroll; ++q) {
            if (e0[q] < 0) continue;
            float f0[V], f1[V];
            unpack<T>(r0[q], f0);
            if (PASS == 1) unpack<T>(r1[q], f1);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const int64_t e = e0[q] + k;
                const bool in = e >= p0[q] && e < p0[q] + HW;
                if (PASS == 0) {
                    const float d = in ? f0[k] - K : 0.f;
                    a1[k] += d;
                    a2[k] = fmaf(d, d, a2[k]);
                    cnt += in ? 1u : 0u;
                } else {
                    float dy, xh;
                    grad_terms(f0[k], in ? f1[k] : 0.f, slope, inv_slope, ia, dy, xh);
                    a1[k] += dy;
                    a2[k] = fmaf(dy, xh, a2[k]);
                }
            }
        }
        if (++iter == 16) {
            iter = 0;
#pragma unroll
            for (int k = 0; k < V; ++k) {
                d1 += a1[k];
                d2 += a2[k];
                a1[k] = a2[k] = 0.f;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < V; ++k) {
        d1 += a1[k];
        d2 += a2[k];
    }
    double v3[3] = {d1, d2, (double)cnt};
    block_sum<3>(v3, red);
    if (threadIdx.x == 0) {
        if (PASS == 0) {
            write_raw_moments(part + ((int64_t)s * C + c) * 3, v3[2], K, v3[0], v3[1]);
        } else {
            double* o = part + ((int64_t)s * C + c) * 2;
            o[0] = v3[0];
            o[1] = v3[1];
        }
    }
}
template <typename T, int PASS>
__global__ void __launch_bounds__(kThreads)
    nchw_cover_kernel(const T* __restrict__ in0, const T* __restrict__ in1,
                      const float* __restrict__ gamma, const float* __restrict__ beta, int64_t C,
                      int64_t HW, int64_t N, int64_t E, float eps, float slope, float inv_slope,
                      uint32_t flags, FastDiv fdw, double* __restrict__ part) {
    pdl_wait();
    nchw_cover_body<T, PASS>(in0, in1, gamma, beta, C, HW, N, E, eps, slope, inv_slope, flags,
                             fdw, part, hw_blk());
}

// ====================================================================== NHWC elementwise passes
// NHWC with C*b a multiple of 16: vector v holds channels (v mod C/V)*V .. +V-1.  The
// host sizes the grid so that the grid stride (gridDim.x*kThreads vectors) is a
// multiple of C/V: every thread then keeps ONE channel group for the whole walk,
// its V channels' coefficients live in registers, and the loop is pure streaming.
// Per thread: batches of kNhwcApplyUnroll vectors (stride apart), every load of a batch predicated
// and in flight before its math; the first batch is issued before the coefficient loads
// so that the two latencies overlap, and the host sizes the grid so that most threads
// run one batch (r02: a tail of single dependent loads cost 1-2 extra latencies).
template <typename T, bool EV = false>
__global__ void __launch_bounds__(kThreads)
    fwd_apply_nhwc_kernel(const T* x, T* z, const float4* __restrict__ coef, uint32_t nvec,
                          uint32_t cv, float slope, EvalCoef ev) {
    pdl_wait();
    constexpr int V = Elem<T>::kVec;
    constexpr int NP = V / 2;
    const uint32_t stride = gridDim.x * kThreads;
    uint32_t v = blockIdx.x * kThreads + threadIdx.x;
    if (v >= nvec) return;
    uint4 r[kNhwcApplyUnroll];
    auto load = [&](uint32_t vb) {
#pragma unroll
        for (int u = 0; u < kNhwcApplyUnroll; ++u)
            if (vb + u * stride < nvec) r[u] = ld_vec(x + (size_t)(vb + u * stride) * V);
    };
    load(v);
    const uint32_t c0 = (v % cv) * V;
    float2 A[NP], B[NP], M[NP];  // per channel pair: A, beta - mu_lo A, mu_hi
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        const float4 c_a = get_coef<true, EV>(coef, ev, c0 + 2 * i),
                     c_b = get_coef<true, EV>(coef, ev, c0 + 2 * i + 1);
        A[i] = make_float2(c_a.x, c_b.x);
        B[i] = make_float2(fmaf(-c_a.z, c_a.x, c_a.w), fmaf(-c_b.z, c_b.x, c_b.w));
        M[i] = make_float2(c_a.y, c_b.y);
    }
    const float2 sl2 = make_float2(slope, slope);
    auto apply = [&](const uint4 rr, const uint32_t vv) {
        float2 w[NP];
        Pairs<T>::load(rr, w);
#pragma unroll
        for (int i = 0; i < NP; ++i) {
            const float2 y = fma2(add2(w[i], make_float2(-M[i].x, -M[i].y)), A[i], B[i]);
            const float2 ay = mul2(y, sl2);
            w[i] = make_float2(fmaxf(y.x, ay.x), fmaxf(y.y, ay.y));
        }
        st_vec(z + (size_t)vv * V, Pairs<T>::store(w));
    };
    while (true) {
#pragma unroll
        for (int u = 0; u < kNhwcApplyUnroll; ++u)
            if (v + u * stride < nvec) apply(r[u], v + u * stride);
        v += kNhwcApplyUnroll * stride;
        if (v >= nvec) break;
        load(v);
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    bwd_apply_nhwc_kernel(const T* __restrict__ z, const T* dz, T* dx,
                          const float4* __restrict__ coef, uint32_t nvec, uint32_t cv,
                          float slope, float inv_slope) {
    pdl_wait();
    constexpr int V = Elem<T>::kVec;
    const uint32_t stride = gridDim.x * kThreads;
    uint32_t v = blockIdx.x * kThreads + threadIdx.x;
    if (v >= nvec) return;
    uint4 rz[kNhwcApplyUnroll], rd[kNhwcApplyUnroll];
    auto load = [&](uint32_t vb) {
#pragma unroll
        for (int u = 0; u < kNhwcApplyUnroll; ++u)
            if (vb + u * stride < nvec) {
                rz[u] = ld_vec(z + (size_t)(vb + u * stride) * V);
                rd[u] = ld_vec(dz + (size_t)(vb + u * stride) * V);
            }
    };
    load(v);
    const uint32_t c0 = (v % cv) * V;
    float al[V], ka[V], cc[V];  // dx = al dy + ka y + cc
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const float4 cf = __ldg(coef + c0 + k);
        al[k] = cf.x;
        ka[k] = cf.y;
        cc[k] = cf.z;
    }
    auto apply = [&](const uint4 qz, const uint4 qd, const uint32_t vv) {
        float fz[V], fd[V];
        unpack<T>(qz, fz);
        unpack<T>(qd, fd);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const bool pos = fz[k] >= 0.f;  // -0.0 counts as >= 0
            const float y = pos ? fz[k] : fz[k] * inv_slope;
            const float dy = pos ? fd[k] : fd[k] * slope;
            fz[k] = fmaf(al[k], dy, fmaf(ka[k], y, cc[k]));
        }
        st_vec(dx + (size_t)vv * V, pack<T>(fz));
    };
    while (true) {
#pragma unroll
        for (int u = 0; u < kNhwcApplyUnroll; ++u)
            if (v + u * stride < nvec) apply(rz[u], rd[u], v + u * stride);
        v += kNhwcApplyUnroll * stride;
        if (v >= nvec) break;
        load(v);
    }
}

// ====================================================================== test-time folding
// BN at test time is linear and is absorbed into the preceding Conv.
// Block k scales row k of w (k_per_out values) by s_k = g_k / sqrt(rv_k + eps) and
// writes bias'_k = s_k (bias_k - rm_k) + beta_k.
__global__ void __launch_bounds__(kThreads)
    fold_conv_kernel(const float* w, const float* bias, const float* __restrict__ rm,
                     const float* __restrict__ rv, const float* __restrict__ gamma,
                     const float* __restrict__ beta, float eps, uint32_t flags, int64_t kper,
                     float* w_out, float* bias_out) {
    pdl_wait();
    const int64_t k = blockIdx.x;
    const double sd = gamma_eff(gamma[k], eps, flags) / sqrt((double)rv[k] + (double)eps);
    const float s = (float)sd;
    const float* src = w + k * kper;
    float* dst = w_out + k * kper;
    for (int64_t j = threadIdx.x; j < kper; j += kThreads) dst[j] = src[j] * s;
    if (threadIdx.x == 0) {
        const double b = bias ? (double)bias[k] : 0.0;
        bias_out[k] = (float)(sd * (b - (double)rm[k]) + (double)beta[k]);
    }
}

}  // namespace iabn
