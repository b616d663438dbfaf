// kernels_small.cuh -- register-resident schedule for small NCHW layers (round 2).
//
// On 14x14 and 7x7 layers (N = 32: 3-25 KB per channel) the channel-resident kernels
// (kernels_fused.cuh) spend most of a pass on per-channel latency: bulk copies of
// 400-byte planes serialise in the copy engine, then reduce, exchange and apply run one
// after another on a short slice.  Here a channel's whole slab lives in REGISTERS: a team
// of 32 tw threads (tw = 1, 2, 4 or 8 warps) loads the 16-byte slots covering each of the
// channel's N planes with coherent LDG.128 -- up to kSmallR = 8 slots per thread and input,
// all in flight at once -- reduces them (fp32 per thread, warp shuffles, the team's warps
// in fp64 through shared memory), the team leader derives the coefficients, and the team
// writes the outputs from the same registers: interior slots as 16-byte stores, the edge
// slots of a plane element by element (their other bytes belong to the neighbouring
// channels).  One launch per pass, 2*E*b / 3*E*b of HBM traffic, no cluster, no copy
// engine.  In place is allowed: a thread reads every slot before writing any, and the
// bytes of a neighbour's edge slot that another CTA may be rewriting are read (coherent
// loads) but never used.
//
// Arithmetic as in the other schedules: shifted fp32 sums (shift = the channel's first
// value), fp64 team combine as raw moments, fwd_coef_from_moments; backward BN-dagger sums
// Q = sum dz z and S1 = sum dz - (1 - a) sum_{z<0} dz, S2 = (Q - beta S1) / g (IABN_VARIANT_I:
// per-element dy x^).
#pragma once

#include "common.cuh"
#include "kernels_act.cuh"
#include "kernels_stream.cuh"

namespace iabn {

constexpr int kSmallThreads = 256;
#ifndef IABN_SMALL_MINB_F4
#define IABN_SMALL_MINB_F4 4  // forward, R = 4: CTAs per SM the register cap is sized for
#endif
#ifndef IABN_SMALL_EARLY_TRIGGER
#define IABN_SMALL_EARLY_TRIGGER 0
#endif
#ifndef IABN_SMALL_L2HINT
#define IABN_SMALL_L2HINT ""  // experiments: ".L2::128B" / ".L2::256B" prefetch-size hint
#endif
#ifndef IABN_SMALL_MINB_B4
#define IABN_SMALL_MINB_B4 4  // backward, R = 4 (64 registers: spills ~70 bytes of stack)
#endif
constexpr int kSmallR = 8;  // most 16-byte slots per thread and input (R = 4 or 8)

struct SmallArgs {
    const void* in0;  // forward: x; backward: z
    const void* in1;  // backward: dz
    void* out;        // forward: z; backward: dx
    const float* gamma;
    const float* beta;
    float* running_mean;
    float* running_var;
    float* save_mean;
    float* save_var;
    float* dgamma;
    float* dbeta;
    int64_t C, HW;
    uint32_t N;
    uint32_t W;       // 16-byte slots reserved per plane (covering range <= W)
    FastDiv fd_w;
    uint32_t tw;      // warps per channel team
    float momentum, eps, slope, inv_slope;
    uint32_t flags;
    double inv_n;  // 1 / (N HW)
    unsigned long long* trace;  // experiments: [grid][kSmallTrace] %globaltimer of CTA phases
};
// phases: 0 start, 1 PDL wait done, 2 thread 0's sums done (its loads landed), 3 team
// partials in shared memory, 4 coefficients ready, 5 stores issued
constexpr int kSmallTrace = 6;

// element k of 16-byte slot i lies in the plane's bytes [h, h + hwb)
template <typename T>
__device__ __forceinline__ bool mis_valid_small(uint32_t i, int k, uint32_t h, uint32_t hwb) {
    const uint32_t byte = i * 16u + (uint32_t)k * (uint32_t)sizeof(T);
    return byte >= h && byte < h + hwb;
}

__device__ __forceinline__ uint4 ldg_coherent(const void* p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate" IABN_SMALL_L2HINT ".v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// ACT: 0 leaky ReLU, 1 sigmoid, 2 tanh (fp32 only; kernels_act.cuh)
template <typename T, int PASS, int R, int ACT = 0>
__global__ void __launch_bounds__(kSmallThreads, R <= 4 ? (PASS == 0 ? IABN_SMALL_MINB_F4 : IABN_SMALL_MINB_B4) : (PASS == 0 ? 3 : 2))
    small_kernel(const SmallArgs a) {
    constexpr int V = Elem<T>::kVec;
    constexpr int NP = Pairs<T>::kN;
    constexpr uint32_t B = sizeof(T);
    __shared__ double red[kSmallThreads / 32][2];
    __shared__ float cf[kSmallThreads / 32][8];
    __shared__ double stash[kSmallThreads / 32][2];
    __shared__ float pre[kSmallThreads / 32][2];  // forward: old running mean / var

    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t tw = a.tw, TT = 32 * tw, team = warp / tw, tt = tid - team * TT;
    const uint32_t nteam = (kSmallThreads / 32) / tw;
    const int64_t c = (int64_t)blockIdx.x * nteam + team;
    const bool active = c < a.C;
    const uint32_t hwb = (uint32_t)a.HW * B;
    const uint32_t nslots = a.N * a.W;
    const char* in0 = static_cast<const char*>(a.in0);
    const char* in1 = static_cast<const char*>(a.in1);
    auto trace = [&](int k) {
#ifdef IABN_PHASE_TRACE  // experiments build only: the pointer costs registers (spills)
        if (a.trace && tid == 0) {
            unsigned long long tm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
            a.trace[(size_t)blockIdx.x * kSmallTrace + k] = tm;
        }
#else
        (void)k;
#endif
    };
    trace(0);
    pdl_wait();
#if IABN_SMALL_EARLY_TRIGGER  // experiments: let the next kernel's CTAs launch as ours exit
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    trace(1);
    // slot k of this thread: plane n = i / W, slot si = i % W of the plane's covering
    // range (recomputed where needed: registers go to the data)
    struct Slot {
        bool ok;
        uint32_t h, si;
        uint64_t off;
    };
    auto slot = [&](int k) -> Slot {
        Slot sl{false, 0, 0, 0};
        const uint32_t i = tt + (uint32_t)k * TT;
        if (active && i < nslots) {
            const uint32_t n = fdiv(i, a.fd_w), si = i - n * a.W;
            const uint64_t Bp = ((uint64_t)n * a.C + c) * hwb;  // plane's first byte
            const uint32_t h = (uint32_t)(Bp & 15u);
            if (si * 16u < h + hwb) sl = Slot{true, h, si, (Bp & ~(uint64_t)15) + si * 16u};
        }
        return sl;
    };
    // ---- load the channel's covering slots into registers (all loads in flight)
    uint4 xr[R], dr[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const Slot sl = slot(k);
        if (sl.ok) {
            xr[k] = ldg_coherent(in0 + sl.off);
            if (PASS == 1) dr[k] = ldg_coherent(in1 + sl.off);
        }
    }
    // the leader's old running statistics, fetched while the slab's loads are in flight (its
    // read-modify-write after the coefficient barrier would otherwise delay its warp's
    // stores by a global round trip; r02 phase trace: 7x7 layers' slowest CTAs)
    if (PASS == 0 && tt == 0 && active) {
        pre[team][0] = a.running_mean ? a.running_mean[c] : 0.f;
        pre[team][1] = a.running_var ? a.running_var[c] : 0.f;
    }
    float K0 = 0.f, gam = 1.f, bet = 0.f, var_s = 1.f;
    if (active) {
        if (PASS == 0) K0 = ld_scalar<T>(static_cast<const T*>(a.in0) + c * a.HW);
        gam = a.gamma[c];
        bet = a.beta[c];
        if (PASS == 1) var_s = a.save_var[c];
    }
    float ig = 0.f;
    if (PASS == 1 && (a.flags & kVariantI)) ig = (float)(1.0 / gamma_eff(gam, a.eps, a.flags));
    // ---- per-thread sums
    float s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const Slot sl = slot(k);
        if (!sl.ok) continue;
        const bool inner = sl.si * 16u >= sl.h && sl.si * 16u + 16u <= sl.h + hwb;
        float2 p[NP], q[NP];
        Pairs<T>::load(xr[k], p);
        if (PASS == 1) Pairs<T>::load(dr[k], q);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            const bool ok = inner || mis_valid_small<T>(sl.si, e, sl.h, hwb);
            const float x = (e & 1) ? p[e >> 1].y : p[e >> 1].x;
            if (PASS == 0) {
                const float d = ok ? x - K0 : 0.f;
                s1 += d;
                s2 = fmaf(d, d, s2);
            } else if constexpr (ACT != 0) {  // dy = f'(z) dz, y = f^-1(z); selects (masked
                                              // slots may hold anything)
                const float dy = Act<ACT>::df(x) * ((e & 1) ? q[e >> 1].y : q[e >> 1].x);
                const float y = Act<ACT>::inv(x);
                const float t3 = (a.flags & kVariantI) ? dy * ((y - bet) * ig) : dy * y;
                s1 += ok ? dy : 0.f;
                s3 += ok ? t3 : 0.f;
            } else {
                const float dz = ok ? ((e & 1) ? q[e >> 1].y : q[e >> 1].x) : 0.f;
                s1 += dz;
                s2 += x < 0.f ? dz : 0.f;
                if (a.flags & kVariantI) {
                    const float y = x >= 0.f ? x : x * a.inv_slope;
                    const float dy = x >= 0.f ? dz : dz * a.slope;
                    s3 = fmaf(dy, (y - bet) * ig, s3);
                } else {
                    s3 = fmaf(dz, x, s3);
                }
            }
        }
    }
    trace(2);
    float r1 = PASS == 0 ? s1 : fmaf(-(1.f - a.slope), s2, s1);
    float r2 = PASS == 0 ? s2 : s3;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        r1 += __shfl_xor_sync(0xffffffffu, r1, o);
        r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    }
    if (lane == 0) {
        red[warp][0] = r1;
        red[warp][1] = r2;
    }
    __syncthreads();
    trace(3);
    // ---- team leader: channel totals and coefficients
    if (tt == 0 && active) {
        double t1 = 0.0, t2 = 0.0;
        for (uint32_t w = team * tw; w < (team + 1) * tw; ++w) {
            t1 += red[w][0];
            t2 += red[w][1];
        }
        float* co = cf[team];
        if (PASS == 0) {
            // shifted moments in fp64 without a division: d = t1/n, var = t2/n - d^2 with the
            // host's 1/n, rstd by rsqrt (the same quantities as fwd_coef_from_moments, which
            // rebuilds raw moments and divides three times: r02 phase trace, 7x7 layers'
            // coefficient step 1.1 -> 0.8 us)
            const double d = (double)t1 * a.inv_n;
            double var = fma(-d, d, (double)t2 * a.inv_n);
            var = var > 0.0 ? var : 0.0;
            const double mean = (double)K0 + d;
            const double A = gamma_eff(gam, a.eps, a.flags) * rsqrt(var + (double)a.eps);
            const float mu_hi = (float)mean;
            const float4 f = make_float4((float)A, mu_hi, (float)(mean - (double)mu_hi), bet);
            co[0] = f.x;
            co[1] = f.y;
            co[2] = fmaf(-f.z, f.x, f.w);
            stash[team][0] = mean;  // the global writes wait until after the barrier
            stash[team][1] = var;
        } else {
            const double gg = gamma_eff(gam, a.eps, a.flags), bb = (double)bet;
            double S1 = t1, S2 = t2;
            if (!(a.flags & kVariantI)) S2 = (S2 - bb * S1) / gg;  // BN-dagger
            const double rstd = rsqrt((double)var_s + (double)a.eps);
            const double rm = rstd * a.inv_n;
            const float alpha = (float)(gg * rstd), kappa = (float)(-rm * S2);
            co[0] = alpha;
            co[1] = kappa;
            co[2] = alpha * a.slope;
            co[3] = kappa * a.inv_slope;
            co[4] = (float)(rm * fma(S2, bb, -gg * S1));
            stash[team][0] = S1;
            stash[team][1] = S2;
        }
    }
    __syncthreads();
    trace(4);
    if (!active) return;
    // the leader's global writes (statistics, running update, parameter gradients) off the
    // critical path: the team's stores below need only the coefficients (r02 phase trace:
    // the running update's read-modify-write cost ~0.5 us before the barrier)
    if (tt == 0) {
        if (PASS == 0) {
            const double mean = stash[team][0], var = stash[team][1];
            a.save_mean[c] = (float)mean;
            a.save_var[c] = (float)var;
            // update_running (kernels_stream.cuh) on the prefetched values, same arithmetic
            const double mo = (double)a.momentum, cnt = (double)a.N * (double)a.HW;
            if (a.running_mean)
                a.running_mean[c] = (float)((1.0 - mo) * (double)pre[team][0] + mo * mean);
            if (a.running_var) {
                const double v = (a.flags & kRunVarBiased) ? var : var * cnt / (cnt - 1.0);
                a.running_var[c] = (float)((1.0 - mo) * (double)pre[team][1] + mo * v);
            }
        } else {
            a.dbeta[c] = (float)stash[team][0];
            a.dgamma[c] = (float)(gamma_sign(gam, a.flags) * stash[team][1]);
        }
    }
    // ---- outputs from the registers
    const float* co = cf[team];
    const float c0 = co[0], c1 = co[1], c2 = co[2], c3 = PASS == 1 ? co[3] : 0.f,
                c4 = PASS == 1 ? co[4] : 0.f;
    char* out = static_cast<char*>(a.out);
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const Slot sl = slot(k);
        if (!sl.ok) continue;
        const bool inner = sl.si * 16u >= sl.h && sl.si * 16u + 16u <= sl.h + hwb;
        float2 p[NP], q[NP], w[NP];
        Pairs<T>::load(xr[k], p);
        if (PASS == 1) Pairs<T>::load(dr[k], q);
#pragma unroll
        for (int e = 0; e < NP; ++e) {
            if (PASS == 0) {
                const float y0 = fmaf(p[e].x - c1, c0, c2), y1 = fmaf(p[e].y - c1, c0, c2);
                if constexpr (ACT != 0)
                    w[e] = make_float2(Act<ACT>::f(y0), Act<ACT>::f(y1));
                else
                    w[e] = make_float2(y0 >= 0.f ? y0 : y0 * a.slope, y1 >= 0.f ? y1 : y1 * a.slope);
            } else if constexpr (ACT != 0) {  // dx = alpha dy + kappa y + cc
                const float z0 = p[e].x, z1 = p[e].y;
                w[e].x = fmaf(c0, Act<ACT>::df(z0) * q[e].x, fmaf(c1, Act<ACT>::inv(z0), c4));
                w[e].y = fmaf(c0, Act<ACT>::df(z1) * q[e].y, fmaf(c1, Act<ACT>::inv(z1), c4));
            } else {
                const float z0 = p[e].x, z1 = p[e].y;
                w[e].x = z0 >= 0.f ? fmaf(c0, q[e].x, fmaf(c1, z0, c4)) : fmaf(c2, q[e].x, fmaf(c3, z0, c4));
                w[e].y = z1 >= 0.f ? fmaf(c0, q[e].y, fmaf(c1, z1, c4)) : fmaf(c2, q[e].y, fmaf(c3, z1, c4));
            }
        }
        T* dst = reinterpret_cast<T*>(out + sl.off);
        if (inner) {
            st_vec(dst, Pairs<T>::store(w));
        } else {
#pragma unroll
            for (int e = 0; e < V; ++e)
                if (mis_valid_small<T>(sl.si, e, sl.h, hwb))
                    st_scalar<T>(dst + e, (e & 1) ? w[e >> 1].y : w[e >> 1].x);
        }
    }
    trace(5);
}

}  // namespace iabn
