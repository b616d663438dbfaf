// kernels_coop.cuh -- one-launch schedule for small layers (any layout / alignment).
//
// The streaming schedule's three phases -- per-split partial sums, per-channel
// combine + coefficients, elementwise apply -- run in ONE cooperative launch
// separated by two grid barriers instead of three kernel launches.  The apply
// re-reads its inputs while they are still in the 126 MB L2 (the layer is
// small), so HBM sees ~2*E*b forward and ~3*E*b backward, and the layer pays one
// launch latency instead of three.  Every phase is the streaming kernels' body
// on virtual block ids with the same partitions, so results are bitwise those
// of the streaming schedule (tests/test_parity_gpu.py::test_coop_*).
#pragma once

#include "kernels_stream.cuh"

namespace iabn {

// Monotonic grid barrier: the k-th barrier of a launch waits until k*gridDim.x
// blocks have arrived (the counter is zeroed before the launch; all blocks are
// co-resident: cooperative launch).  Release: fence before the arrival; acquire:
// ld.acquire of the counter, then the block barrier.
__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        unsigned v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= target) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
}

struct CoopArgs {
    const void* in0;  // x (fwd) / z (bwd)
    const void* in1;  // dz (bwd)
    void* out;        // z (fwd) / dx (bwd)
    int64_t C, HW, rows, N;
    uint32_t m, E;
    FastDiv fd_hw, fd_c, fd_cover;
    int S;
    double* part;
    float4* coef;
    unsigned* bar;
    float slope, inv_slope, eps;
    uint32_t flags;
    const float* gamma;
    const float* beta;
    FwdCoefArgs fwd;
    BwdCoefArgs bwd;
};

template <typename T, int LAYOUT, bool VEC, int PASS>
__global__ void __launch_bounds__(kThreads, 2) coop_kernel(const CoopArgs a) {
    const T* in0 = (const T*)a.in0;
    const T* in1 = (const T*)a.in1;
    const uint32_t C = (uint32_t)a.C, S = (uint32_t)a.S;
    // ---- phase 1: partial sums of split s of channel (column block) c
    if (LAYOUT == 0) {
        for (uint32_t vb = blockIdx.x; vb < C * S; vb += gridDim.x) {
            const Blk bk{vb % C, vb / C, C, S};
            if (!VEC)  // planes not 16-byte aligned: masked covering vectors
                nchw_cover_body<T, PASS>(in0, in1, a.gamma, a.beta, a.C, a.HW, a.N, a.E, a.eps,
                                         a.slope, a.inv_slope, a.flags, a.fd_cover, a.part, bk);
            else if (PASS == 0)
                stats_nchw_body<T, VEC>(in0, a.C, a.HW, a.m, a.fd_hw, a.part, bk);
            else
                bwd_reduce_nchw_body<T, VEC>(in0, in1, a.gamma, a.beta, a.C, a.HW, a.m, a.fd_hw,
                                             a.eps, a.slope, a.inv_slope, a.flags, a.part, bk);
            __syncthreads();  // the body's shared scratch is reused by the next virtual block
        }
    } else {
        constexpr uint32_t CT = 16 * (VEC ? Elem<T>::kVec : 1);
        const uint32_t ncol = (C + CT - 1) / CT;
        for (uint32_t vb = blockIdx.x; vb < ncol * S; vb += gridDim.x) {
            const Blk bk{vb % ncol, vb / ncol, ncol, S};
            if (PASS == 0)
                stats_nhwc_body<T, VEC>(in0, a.C, a.rows, a.part, bk);
            else
                bwd_reduce_nhwc_body<T, VEC>(in0, in1, a.gamma, a.beta, a.C, a.rows, a.eps,
                                             a.slope, a.inv_slope, a.flags, a.part, bk);
            __syncthreads();
        }
    }
    grid_barrier(a.bar, gridDim.x);
    // ---- phase 2: one warp per channel: combine the S splits, coefficients
    {
        const int64_t nw = (int64_t)gridDim.x * (kThreads / 32);
        for (int64_t c = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); c < a.C;
             c += nw) {
            if (PASS == 0)
                fwd_coef_body(a.fwd, c);
            else
                bwd_coef_body(a.bwd, c);
        }
    }
    grid_barrier(a.bar, 2 * gridDim.x);
    // ---- phase 3: elementwise apply (inputs re-read from L2)
    const Blk bk{blockIdx.x, 0, gridDim.x, 1};
    if (PASS == 0 && LAYOUT == 0 && VEC)
        fwd_apply_rows_body<T, false>(in0, (T*)a.out, a.coef, a.E, (uint32_t)a.HW, C,
                               a.fd_hw, a.fd_c, a.slope, bk);
    else if (PASS == 0)
        fwd_apply_body<T, LAYOUT, VEC, false>(in0, (T*)a.out, a.coef, a.E, a.fd_hw, a.fd_c,
                                              a.slope, bk);
    else
        bwd_apply_body<T, LAYOUT, VEC, false>(in0, in1, (T*)a.out, a.coef, a.E, a.fd_hw, a.fd_c,
                                              a.slope, a.inv_slope, bk);
}

}  // namespace iabn
