// kernels_act.cuh -- BN followed by another invertible activation (round 2).
//
// "Many activation functions are actually invertible and can be computed
// in-place (e.g. sigmoid, hyperbolic tangent, Leaky ReLU, and others)".  The leaky-ReLU
// path (the paper's choice, every other schedule) stays as it is; this file adds the
// streaming schedule for f = sigmoid and f = tanh, fp32 storage only:
//
//   forward   stats (kernels_stream.cuh) -> fwd_coef -> act_fwd_apply: z = f(y)
//   backward  act_bwd_reduce: per channel sum dy and sum dy x^ with dy = f'(z) dz and
//             x^ = (f^-1(z) - beta) / g (Alg. 2 l.2-5, inverting z) -> bwd_coef ->
//             act_bwd_apply: dx = alpha dy + kappa y + cc  (Alg. 2 l.6, y = f^-1(z))
//
// Every element needs f^-1(z) in both backward passes, so the BN-dagger reading of
// variant II (which avoids the inversion for leaky ReLU) has nothing to save here: one
// reduction for both variants.  f' from z:  sigmoid z (1 - z),  tanh 1 - z^2.
// Inversion of saturated outputs (R17): z is clamped into the open range
// before f^-1 -- sigmoid to [FLT_MIN, 1 - 2^-24], tanh to [-(1 - 2^-24), 1 - 2^-24] --
// where f'(z) dz is 0 (or one ulp) anyway; the y of a saturated element is the one
// information InPlace-ABN cannot recover in fp32.
#pragma once

#include "common.cuh"
#include "kernels_stream.cuh"

namespace iabn {

enum : uint32_t { kActSigmoid = 1u << 13, kActTanh = 1u << 14 };

constexpr float kOneBelow1 = 0.99999994f;  // 1 - 2^-24, the largest float below 1

// MUFU forms (ex2 / lg2 / rcp): the backward evaluates f^-1 twice per element and would
// otherwise be ALU-bound.  Absolute errors: f a few ulp of 1, f^-1 ~ 1e-6 |y| + 1e-7,
// well inside the 1e-4 normwise tolerance (the fp64 oracle decides, tests/).
template <int ACT>  // 1 = sigmoid, 2 = tanh
struct Act {
    static __device__ __forceinline__ float f(float y) {
        // __fdividef: MUFU.RCP + one multiply (__frcp_rn is a correctly rounded software
        // sequence: it made the channel-resident forward's apply warps ALU-bound); for a
        // denominator beyond 2^126 (y < -87) the quotient is 0, the limit
        if (ACT == 1) return __fdividef(1.f, 1.f + __expf(-y));
        return 1.f - __fdividef(2.f, __expf(2.f * y) + 1.f);  // +-inf / 0 give +-1
    }
    static __device__ __forceinline__ float df(float z) {  // f'(f^-1(z))
        if (ACT == 1) return z * (1.f - z);
        return fmaf(-z, z, 1.f);
    }
    static __device__ __forceinline__ float inv(float z) {
        if (ACT == 1) {  // log z - log(1 - z); 1 - z exact for z >= 1/2
            z = fminf(fmaxf(z, 1.17549435e-38f), kOneBelow1);
            return __logf(z) - __logf(1.f - z);
        }
        z = fminf(fmaxf(z, -kOneBelow1), kOneBelow1);  // (log(1 + z) - log(1 - z)) / 2
        return 0.5f * (__logf(1.f + z) - __logf(1.f - z));
    }
};

// Elementwise passes over a chunk whose base is 16-byte aligned: kUnroll float4 loads in
// flight per thread, then the math.  ALIGNED: NCHW with HW % 4 == 0 (a vector lies in
// one channel) or NHWC with C % 4 == 0 (a vector holds channels c0 .. c0 + 3); else the
// channel is resolved per element.  PASS 0: out = f(y(in0)) (in place allowed);
// PASS 1: out = alpha f'(z) dz + kappa f^-1(z) + cc with z = in0, dz = in1 (out may alias
// dz).
template <int ACT, int PASS>
__device__ __forceinline__ float act_elem(float v, float d, const float4& cf) {
    if (PASS == 0) return Act<ACT>::f(affine(v, cf));
    return fmaf(cf.x, Act<ACT>::df(v) * d, fmaf(cf.y, Act<ACT>::inv(v), cf.z));
}

template <int ACT, int PASS, int LAYOUT, bool ALIGNED>
__global__ void __launch_bounds__(kThreads)
    act_apply_kernel(const float* in0, const float* in1, float* out,
                     const float4* __restrict__ coef, uint32_t E, FastDiv fd_hw, FastDiv fd_c) {
    pdl_wait();
    const uint32_t nvec = E / 4, stride = gridDim.x * kThreads;
    for (uint32_t base = blockIdx.x * kThreads + threadIdx.x; base < nvec;
         base += stride * kUnroll) {
        float4 r0[kUnroll], r1[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                r0[u] = *reinterpret_cast<const float4*>(in0 + (size_t)v * 4);
                if (PASS == 1) r1[u] = *reinterpret_cast<const float4*>(in1 + (size_t)v * 4);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                float* f0 = reinterpret_cast<float*>(&r0[u]);
                const float* f1 = reinterpret_cast<const float*>(&r1[u]);
                const uint32_t e = v * 4;
                const uint32_t c0 = ALIGNED ? channel_of<LAYOUT>(e, fd_hw, fd_c) : 0;
                float4 cf = ALIGNED && LAYOUT == 0 ? __ldg(coef + c0) : float4{};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (ALIGNED && LAYOUT == 1) cf = __ldg(coef + c0 + k);
                    if (!ALIGNED) cf = __ldg(coef + channel_of<LAYOUT>(e + k, fd_hw, fd_c));
                    f0[k] = act_elem<ACT, PASS>(f0[k], PASS == 1 ? f1[k] : 0.f, cf);
                }
                *reinterpret_cast<float4*>(out + (size_t)v * 4) = r0[u];
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < E - nvec * 4) {
        const uint32_t e = nvec * 4 + threadIdx.x;
        out[e] = act_elem<ACT, PASS>(in0[e], PASS == 1 ? in1[e] : 0.f,
                                     __ldg(coef + channel_of<LAYOUT>(e, fd_hw, fd_c)));
    }
}

// NHWC, C % 4 == 0, grid stride a multiple of the C/4 vectors of a row (nhwc_grid): a
// thread's channel group never changes, so its four coefficient records are loaded once.
template <int ACT, int PASS>
__global__ void __launch_bounds__(kThreads)
    act_apply_fixed_kernel(const float* in0, const float* in1, float* out,
                           const float4* __restrict__ coef, uint32_t E, FastDiv fd_hw,
                           FastDiv fd_c) {
    pdl_wait();
    const uint32_t nvec = E / 4, stride = gridDim.x * kThreads;
    const uint32_t v0 = blockIdx.x * kThreads + threadIdx.x;
    if (v0 >= nvec) return;  // C % 4 == 0: no tail
    const uint32_t c0 = channel_of<1>(v0 * 4, fd_hw, fd_c);
    const float4 cf[4] = {__ldg(coef + c0), __ldg(coef + c0 + 1), __ldg(coef + c0 + 2),
                          __ldg(coef + c0 + 3)};
    for (uint32_t base = v0; base < nvec; base += stride * kUnroll) {
        float4 r0[kUnroll], r1[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                r0[u] = *reinterpret_cast<const float4*>(in0 + (size_t)v * 4);
                if (PASS == 1) r1[u] = *reinterpret_cast<const float4*>(in1 + (size_t)v * 4);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t v = base + u * stride;
            if (v < nvec) {
                float* f0 = reinterpret_cast<float*>(&r0[u]);
                const float* f1 = reinterpret_cast<const float*>(&r1[u]);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    f0[k] = act_elem<ACT, PASS>(f0[k], PASS == 1 ? f1[k] : 0.f, cf[k]);
                *reinterpret_cast<float4*>(out + (size_t)v * 4) = r0[u];
            }
        }
    }
}

// per-element backward terms: dy = f'(z) dz, x^ = (f^-1(z) - beta) / g
template <int ACT>
__device__ __forceinline__ void act_terms(float z, float dz, float bt, float ig, float& a1,
                                          float& a2) {
    const float dy = Act<ACT>::df(z) * dz;
    a1 += dy;
    a2 = fmaf(dy, (Act<ACT>::inv(z) - bt) * ig, a2);
}

// NCHW partial sums: grid (C, S); block (c, s) sums the s-th share of the channel's
// m = N*HW elements; part[s][c] = (sum dy, sum dy x^), fp32 per thread (runs of <= 64
// updates), fp64 across runs and the block.  VEC (HW % 4 == 0): float4 slots q of the
// channel (plane n = q / (HW/4)), kUnroll slots of z and dz in flight; else scalars.
template <int ACT, bool VEC>
__global__ void __launch_bounds__(kThreads)
    act_bwd_reduce_nchw_kernel(const float* __restrict__ z, const float* __restrict__ dz,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               int64_t C, uint32_t HW, uint32_t m, FastDiv fd_hw, float eps,
                               uint32_t flags, double* __restrict__ part) {
    pdl_wait();
    constexpr int V = VEC ? 4 : 1;
    __shared__ double red[2 * kThreads / 32];
    const int64_t c = blockIdx.x;
    const uint32_t S = gridDim.y, s = blockIdx.y, hv = HW / V, mv = m / V;
    const uint32_t lo = (uint32_t)((uint64_t)mv * s / S), hi = (uint32_t)((uint64_t)mv * (s + 1) / S);
    const float bt = beta[c], ig = (float)(1.0 / gamma_eff(gamma[c], eps, flags));
    float a1 = 0.f, a2 = 0.f;
    double d1 = 0.0, d2 = 0.0;
    int run = 0;
    for (uint32_t q0 = lo + threadIdx.x; q0 < hi; q0 += kThreads * kUnroll) {
        float4 rz[kUnroll], rd[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t q = q0 + u * kThreads;
            if (q < hi) {
                const uint32_t n = fdiv(q, fd_hw);  // fd_hw divides by hv
                const size_t off = ((size_t)n * C + c) * HW + (size_t)(q - n * hv) * V;
                if (VEC) {
                    rz[u] = __ldg(reinterpret_cast<const float4*>(z + off));
                    rd[u] = __ldg(reinterpret_cast<const float4*>(dz + off));
                } else {
                    rz[u].x = __ldg(z + off);
                    rd[u].x = __ldg(dz + off);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (q0 + u * kThreads < hi) {
                const float* fz = reinterpret_cast<const float*>(&rz[u]);
                const float* fd = reinterpret_cast<const float*>(&rd[u]);
#pragma unroll
                for (int k = 0; k < V; ++k) act_terms<ACT>(fz[k], fd[k], bt, ig, a1, a2);
            }
        }
        if (++run * kUnroll * V >= 64) {
            d1 += a1;
            d2 += a2;
            a1 = a2 = 0.f;
            run = 0;
        }
    }
    double v[2] = {d1 + a1, d2 + a2};
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        part[((size_t)s * C + c) * 2 + 0] = v[0];
        part[((size_t)s * C + c) * 2 + 1] = v[1];
    }
}

// NHWC ([rows][C]) partial sums, C % 4 == 0: block = 16 lanes of 4 channels x 16 row
// lanes, grid (ceil(C / 64), S); block (cx, s) sums rows [rows s / S, rows (s + 1) / S)
// of its 64 channels (16 lanes read 256 contiguous bytes of a row), kUnroll rows of z
// and dz in flight per thread; fp64 combine of the 16 row lanes in shared memory.
template <int ACT>
__global__ void __launch_bounds__(kThreads)
    act_bwd_reduce_nhwc_kernel(const float* __restrict__ z, const float* __restrict__ dz,
                               const float* __restrict__ gamma, const float* __restrict__ beta,
                               int64_t C, int64_t rows, float eps, uint32_t flags,
                               double* __restrict__ part) {
    pdl_wait();
    __shared__ double red[16][64][2];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const uint32_t S = gridDim.y, s = blockIdx.y;
    const int64_t c0 = (int64_t)blockIdx.x * 64 + tx * 4;
    const int64_t lo = rows * s / S, hi = rows * (s + 1) / S;
    double d1[4] = {0.0, 0.0, 0.0, 0.0}, d2[4] = {0.0, 0.0, 0.0, 0.0};
    if (c0 < C) {
        float bt[4], ig[4], a1[4], a2[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            bt[k] = beta[c0 + k];
            ig[k] = (float)(1.0 / gamma_eff(gamma[c0 + k], eps, flags));
            a1[k] = a2[k] = 0.f;
        }
        int run = 0;
        for (int64_t r0 = lo + ty; r0 < hi; r0 += 16 * kUnroll) {
            float4 rz[kUnroll], rd[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const int64_t r = r0 + u * 16;
                if (r < hi) {
                    rz[u] = __ldg(reinterpret_cast<const float4*>(z + (size_t)r * C + c0));
                    rd[u] = __ldg(reinterpret_cast<const float4*>(dz + (size_t)r * C + c0));
                }
            }
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (r0 + u * 16 < hi) {
                    const float* fz = reinterpret_cast<const float*>(&rz[u]);
                    const float* fd = reinterpret_cast<const float*>(&rd[u]);
#pragma unroll
                    for (int k = 0; k < 4; ++k) act_terms<ACT>(fz[k], fd[k], bt[k], ig[k], a1[k], a2[k]);
                }
            if (++run * kUnroll >= 64) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    d1[k] += a1[k];
                    d2[k] += a2[k];
                    a1[k] = a2[k] = 0.f;
                }
                run = 0;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            d1[k] += a1[k];
            d2[k] += a2[k];
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        red[ty][tx * 4 + k][0] = d1[k];
        red[ty][tx * 4 + k][1] = d2[k];
    }
    __syncthreads();
    // 64 channels x 2 sums: thread t < 128 adds the 16 row lanes of one (channel, sum)
    if (threadIdx.x < 128) {
        const int ch = threadIdx.x >> 1, k = threadIdx.x & 1;
        const int64_t c = (int64_t)blockIdx.x * 64 + ch;
        if (c < C) {
            double t = 0.0;
            for (int r = 0; r < 16; ++r) t += red[r][ch][k];
            part[((size_t)s * C + c) * 2 + k] = t;
        }
    }
}

// NHWC with C % 4 != 0: one channel per lane, 32 channel lanes x 8 row lanes.
template <int ACT>
__global__ void __launch_bounds__(kThreads)
    act_bwd_reduce_nhwc_scalar_kernel(const float* __restrict__ z, const float* __restrict__ dz,
                                      const float* __restrict__ gamma,
                                      const float* __restrict__ beta, int64_t C, int64_t rows,
                                      float eps, uint32_t flags, double* __restrict__ part) {
    pdl_wait();
    constexpr int RL = kThreads / 32;
    __shared__ double red[RL][32][2];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const uint32_t S = gridDim.y, s = blockIdx.y;
    const int64_t c = (int64_t)blockIdx.x * 32 + tx;
    const int64_t lo = rows * s / S, hi = rows * (s + 1) / S;
    double d1 = 0.0, d2 = 0.0;
    if (c < C) {
        const float bt = beta[c], ig = (float)(1.0 / gamma_eff(gamma[c], eps, flags));
        float a1 = 0.f, a2 = 0.f;
        int run = 0;
        for (int64_t r = lo + ty; r < hi; r += RL) {
            act_terms<ACT>(__ldg(z + (size_t)r * C + c), __ldg(dz + (size_t)r * C + c), bt, ig,
                           a1, a2);
            if (++run == 64) {
                d1 += a1;
                d2 += a2;
                a1 = a2 = 0.f;
                run = 0;
            }
        }
        d1 += a1;
        d2 += a2;
    }
    red[ty][tx][0] = d1;
    red[ty][tx][1] = d2;
    __syncthreads();
    if (ty == 0 && c < C) {
        for (int k = 1; k < RL; ++k) {
            d1 += red[k][tx][0];
            d2 += red[k][tx][1];
        }
        part[((size_t)s * C + c) * 2 + 0] = d1;
        part[((size_t)s * C + c) * 2 + 1] = d2;
    }
}

}  // namespace iabn
