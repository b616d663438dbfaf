// kernels_gres.cuh -- grid-resident schedule for NHWC layers that fit on chip.
//
// NHWC ([rows][C], rows = N*HW) keeps every channel spread over all rows, so a
// channel slab cannot be made resident the way the NCHW cluster kernels do.  For
// a layer whose input fits in the GPU's aggregate shared memory (2 CTAs x ~100 KB
// per SM), the whole tensor is made resident instead: CTA i of a cooperative grid
// bulk-copies rows [r_i, r_{i+1}) into shared memory once, publishes its
// per-channel partial moments, the grid meets at a barrier, one warp per channel
// combines the G partials (fixed order) into the coefficients, a second barrier,
// then every CTA writes its outputs from the resident rows.  HBM traffic is the
// channel-resident minimum (2*E*b forward, 3*E*b backward) in one launch; the
// alternative is three streaming kernels moving 3*E*b / 5*E*b.
//
// Thread mapping: a row holds cv = C*b/16 vectors; thread t < rt*cv takes column
// j = t % cv (channels j*V .. j*V+V-1, fixed for the whole kernel) and rows
// t / cv, + rt, ...  (rt = 256 / cv threads per column).
#pragma once

#include "kernels_stream.cuh"

namespace iabn {

// Sense-reversing grid barrier whose state persists across launches (no reset
// between calls): count returns to 0 after every barrier, gen only grows.  The
// state is one of the library's per-stream slots (zeroed once at allocation).
struct GridBar {
    unsigned count, gen;
};
__device__ __forceinline__ void grid_sync(GridBar* b, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&b->gen) : "memory");
        __threadfence();  // this block's writes before its arrival
        if (atomicAdd(&b->count, 1u) == G - 1) {
            atomicExch(&b->count, 0u);  // every block has arrived: re-arm, then release
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&b->gen), "r"(g + 1)
                         : "memory");
        } else {
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(&b->gen)
                             : "memory");
                if (v != g) break;
                __nanosleep(32);
            }
        }
    }
    __syncthreads();
}

struct GresArgs {
    const void* in0;  // x (fwd) / z (bwd)
    const void* in1;  // dz (bwd)
    void* out;        // z (fwd, may be x) / dx (bwd, may be dz)
    int64_t C, rows;
    uint32_t cv;      // 16-byte vectors per row
    float slope, inv_slope, eps;
    uint32_t flags;
    const float* gamma;
    const float* beta;
    double* part;     // [G][C][3] forward raw moments / [G][C][2] backward sums
    float4* coef;     // [C]
    GridBar* bar;     // persistent per-stream barrier state
    FwdCoefArgs fwd;  // phase 2 (S = G)
    BwdCoefArgs bwd;
};

template <typename T, int PASS>
__global__ void __launch_bounds__(kThreads, 2) gres_kernel(const GresArgs a) {
    constexpr int V = Elem<T>::kVec;
    constexpr int NIN = PASS == 0 ? 1 : 2;
    extern __shared__ __align__(128) uint4 slab[];
    __shared__ __align__(8) uint64_t landed;
    __shared__ double red[2][kThreads];
    pdl_wait();
    const uint32_t G = gridDim.x, i = blockIdx.x;
    const int64_t C = a.C;
    const uint32_t cv = a.cv;
    const uint32_t rt = kThreads / cv;       // threads per column
    const uint32_t active = rt * cv;
    const uint32_t t = threadIdx.x, j = t % cv, r0 = t / cv;
    const int64_t r_lo = a.rows * i / G, r_hi = a.rows * (i + 1) / G;
    const uint32_t nr = (uint32_t)(r_hi - r_lo);
    const size_t row_v = cv;                 // vectors per row
    const size_t in_v = (size_t)nr * row_v;  // vectors per input held
    const T* in0 = (const T*)a.in0;
    const T* in1 = (const T*)a.in1;

    // ---- phase 0: bulk-copy this CTA's rows of every input into shared memory
    if (t == 0) {
        mbar_init(&landed, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (t == 0) {
        const uint32_t bytes = (uint32_t)(in_v * 16);
        mbar_arrive_expect_tx(&landed, bytes * NIN);
        const T* src[2] = {in0, in1};
        for (int k = 0; k < NIN; ++k) {
            const char* g = (const char*)(src[k] + r_lo * C);
            char* d = (char*)(slab + k * in_v);
            for (uint32_t off = 0; off < bytes; off += 32768u)
                bulk_g2s(d + off, g + off, min(32768u, bytes - off), &landed);
        }
    }
    // per-thread column constants, overlapping the copy
    const int64_t c0 = (int64_t)j * V;
    float kc[V];  // forward shift: the channel's first element (row 0 of the tensor)
    InvAffine ia[V];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        kc[k] = 0.f;
        ia[k] = InvAffine{0.f, 0.f};
        if (t < active) {
            if (PASS == 0) kc[k] = ld_scalar<T>(in0 + c0 + k);
            else ia[k] = inv_affine(a.gamma[c0 + k], a.beta[c0 + k], a.eps, a.flags);
        }
    }
    mbar_wait(&landed, 0);

    // ---- phase 1: per-channel partial sums of the resident rows
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1[V], d2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) d1[k] = d2[k] = 0.0;
    if (t < active) {
        int iter = 0;
        for (uint32_t r = r0; r < nr; r += rt) {
            float f0[V], f1[V];
            unpack<T>(slab[(size_t)r * row_v + j], f0);
            if (PASS == 1) unpack<T>(slab[in_v + (size_t)r * row_v + j], f1);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                if (PASS == 0) {
                    const float dv = f0[k] - kc[k];
                    a1[k] += dv;
                    a2[k] = fmaf(dv, dv, a2[k]);
                } else {
                    float dy, xh;
                    grad_terms(f0[k], f1[k], a.slope, a.inv_slope, ia[k], dy, xh);
                    a1[k] += dy;
                    a2[k] = fmaf(dy, xh, a2[k]);
                }
            }
            if (++iter == 16) {
                iter = 0;
#pragma unroll
                for (int k = 0; k < V; ++k) {
                    d1[k] += a1[k];
                    d2[k] += a2[k];
                    a1[k] = a2[k] = 0.f;
                }
            }
        }
    }
    // column reduction, one channel offset k at a time (threads of a column in order)
#pragma unroll
    for (int k = 0; k < V; ++k) {
        red[0][t] = d1[k] + a1[k];
        red[1][t] = d2[k] + a2[k];
        __syncthreads();
        if (t < cv) {
            double S1 = 0.0, S2 = 0.0;
            for (uint32_t y = 0; y < rt; ++y) {
                S1 += red[0][y * cv + t];
                S2 += red[1][y * cv + t];
            }
            const int64_t c = (int64_t)t * V + k;
            if (PASS == 0) {
                write_raw_moments(a.part + ((int64_t)i * C + c) * 3, (double)nr,
                                  (double)ld_scalar<T>(in0 + c), S1, S2);
            } else {
                double* o = a.part + ((int64_t)i * C + c) * 2;
                o[0] = S1;
                o[1] = S2;
            }
        }
        __syncthreads();
    }
    grid_sync(a.bar, G);

    // ---- phase 2: one warp per channel combines the G partials, coefficients
    {
        const int64_t nw = (int64_t)G * (kThreads / 32);
        for (int64_t c = (int64_t)i * (kThreads / 32) + (t >> 5); c < C; c += nw) {
            if (PASS == 0)
                fwd_coef_body(a.fwd, c);
            else
                bwd_coef_body(a.bwd, c);
        }
    }
    grid_sync(a.bar, G);

    // ---- phase 3: outputs of the resident rows (coefficients of this column in registers)
    if (t >= active) return;
    float4 cf[V];
#pragma unroll
    for (int k = 0; k < V; ++k) cf[k] = ld_coef<false>(a.coef + c0 + k);
    T* out = (T*)a.out + r_lo * C;
    for (uint32_t r = r0; r < nr; r += rt) {
        float f0[V];
        unpack<T>(slab[(size_t)r * row_v + j], f0);
        if (PASS == 0) {
#pragma unroll
            for (int k = 0; k < V; ++k) f0[k] = leaky(affine(f0[k], cf[k]), a.slope);
        } else {
            float f1[V];
            unpack<T>(slab[in_v + (size_t)r * row_v + j], f1);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                const bool pos = f0[k] >= 0.f;  // -0.0 counts as >= 0
                const float y = pos ? f0[k] : f0[k] * a.inv_slope;
                const float dy = pos ? f1[k] : f1[k] * a.slope;
                f0[k] = fmaf(cf[k].x, dy, fmaf(cf[k].y, y, cf[k].z));
            }
        }
        st_vec(out + (size_t)r * C + c0, pack<T>(f0));
    }
}

}  // namespace iabn
