// kernels_fused.cuh -- channel-resident schedule (NCHW, HW*b a multiple of 16 B).
//
// One thread-block CLUSTER of K CTAs owns one channel c.  CTA r of the cluster
// owns the channel-space slice [lo_r, hi_r) of the channel's m = N*HW values
// (planes n of HW contiguous values, stride C*HW), which it pulls into shared
// memory with TMA bulk copies (cp.async.bulk, one mbarrier per ~chunk so the
// reduction starts on the first chunk while later ones are in flight).  The
// per-channel reduction is a CTA tree followed by a DSMEM exchange of the K
// partial records (fixed order => deterministic, identical in every CTA); the
// apply pass then reads the slice from shared memory and writes the result with
// 16-byte stores.  HBM traffic is the minimum the method allows:
//   forward  FF: read x once, write z once                 = 2*E*b
//   backward BF: read z and dz once, write dx once          = 3*E*b
// (vs 3*E*b and 5*E*b for kernels_stream.cuh).
#pragma once

#include "common.cuh"
#include "kernels_stream.cuh"

namespace iabn {

constexpr int kMaxChunks = 48;

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
    uint32_t m;  // values per channel
    FastDiv fd_hw;
    uint32_t chunk_vecs;  // 16-byte vectors per chunk (per input)
    float momentum, eps, slope, inv_slope;
    uint32_t flags;
};

// Slice of the channel owned by cluster rank r of K, in 16-byte vectors.
__device__ __forceinline__ void cta_slice(uint32_t mv, uint32_t r, uint32_t K, uint32_t& vlo,
                                          uint32_t& vhi) {
    vlo = (uint32_t)((uint64_t)mv * r / K);
    vhi = (uint32_t)((uint64_t)mv * (r + 1) / K);
}

// Thread 0: arm chunk barriers and issue the bulk copies of `nin` inputs for
// channel-space vectors [vlo, vhi) into consecutive smem regions of nv vectors.
template <typename T>
__device__ __forceinline__ void issue_loads(const FusedArgs& a, int64_t c, uint32_t vlo,
                                            uint32_t vhi, uint4* smem, uint64_t* bars,
                                            int nchunks, int nin) {
    constexpr int V = Elem<T>::kVec;
    const uint32_t nv = vhi - vlo;
    const uint32_t hw = (uint32_t)a.HW;
    const T* src[2] = {(const T*)a.in0, (const T*)a.in1};
    for (int k = 0; k < nchunks; ++k) {
        const uint32_t c_lo = vlo + k * a.chunk_vecs;
        const uint32_t c_hi = min(vhi, c_lo + a.chunk_vecs);
        mbar_arrive_expect_tx(&bars[k], (c_hi - c_lo) * 16u * nin);
        uint32_t j = c_lo * V;  // channel-space element
        const uint32_t jend = c_hi * V;
        while (j < jend) {
            const uint32_t n = j / hw, s = j - n * hw;
            const uint32_t len = min(jend - j, hw - s);
            const int64_t goff = ((int64_t)n * a.C + c) * a.HW + s;
            for (int i = 0; i < nin; ++i)
                bulk_g2s(smem + (size_t)i * nv + (j / V - vlo), src[i] + goff,
                         len * (uint32_t)sizeof(T), &bars[k]);
            j += len;
        }
    }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fused_fwd_kernel(const FusedArgs a) {
    constexpr int V = Elem<T>::kVec;
    extern __shared__ __align__(128) uint4 smem[];
    __shared__ __align__(8) uint64_t bars[kMaxChunks];
    __shared__ double red[2 * kThreads / 32];
    __shared__ double part[3];
    __shared__ float4 coef_s;

    const uint32_t K = cluster_nctarank(), r = cluster_ctarank();
    const int64_t c = blockIdx.x / K;
    uint32_t vlo, vhi;
    cta_slice(a.m / V, r, K, vlo, vhi);
    const uint32_t nv = vhi - vlo;
    const int nchunks = (int)((nv + a.chunk_vecs - 1) / a.chunk_vecs);

    if (threadIdx.x == 0) {
        for (int k = 0; k < nchunks; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) issue_loads<T>(a, c, vlo, vhi, smem, bars, nchunks, 1);

    // ---- F1: shifted fp32 chains over the resident slice, fp64 combine
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1 = 0.0, d2 = 0.0;
    float K0 = 0.f;
    if (nchunks > 0) {
        mbar_wait(&bars[0], 0);
        float f[V];
        unpack<T>(smem[0], f);
        K0 = f[0];
    }
    for (int k = 0; k < nchunks; ++k) {
        mbar_wait(&bars[k], 0);
        const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
        for (uint32_t v = c_lo + threadIdx.x; v < c_hi; v += kThreads) {
            float f[V];
            unpack<T>(smem[v], f);
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const float dv = f[q] - K0;
                a1[q] += dv;
                a2[q] = fmaf(dv, dv, a2[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < V; ++q) {
            d1 += a1[q];
            d2 += a2[q];
            a1[q] = a2[q] = 0.f;
        }
    }
    double v2[2] = {d1, d2};
    block_sum<2>(v2, red);
    if (threadIdx.x == 0) write_raw_moments(part, (double)nv * V, (double)K0, v2[0], v2[1]);

    // ---- cluster exchange of the K partial records (DSMEM)
    cluster_arrive_release();
    cluster_wait_acquire();
    if (threadIdx.x == 0) {
        double cnt = 0.0, sum = 0.0, sumsq = 0.0;
        for (uint32_t q = 0; q < K; ++q) {
            cnt += ld_dsmem_f64(&part[0], q);
            sum += ld_dsmem_f64(&part[1], q);
            sumsq += ld_dsmem_f64(&part[2], q);
        }
        double mean, var;
        coef_s = fwd_coef_from_moments(cnt, sum, sumsq, a.gamma[c], a.beta[c], a.eps, a.flags,
                                       &mean, &var);
        if (r == 0) {
            a.save_mean[c] = (float)mean;
            a.save_var[c] = (float)var;
            update_running(a.running_mean, a.running_var, c, mean, var, cnt, a.momentum, a.flags);
        }
    }
    __syncthreads();
    cluster_arrive_release();  // this CTA no longer reads remote shared memory

    // ---- F2: z = f(x A + B) from shared memory, 16-byte stores (z may be x)
    const float4 cf = coef_s;
    const float slope = a.slope;
    T* z = (T*)a.out;
    const uint32_t hw = (uint32_t)a.HW;
    for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        float f[V];
        unpack<T>(smem[v], f);
#pragma unroll
        for (int q = 0; q < V; ++q) f[q] = leaky(affine(f[q], cf), slope);
        const uint32_t j = (vlo + v) * V;
        const uint32_t n = fdiv(j, a.fd_hw);
        st_vec(z + ((int64_t)n * a.C + c) * a.HW + (j - n * hw), pack<T>(f));
    }
    cluster_wait_acquire();  // peers are done reading this CTA's part[]
}

template <typename T>
__global__ void __launch_bounds__(kThreads) fused_bwd_kernel(const FusedArgs a) {
    constexpr int V = Elem<T>::kVec;
    extern __shared__ __align__(128) uint4 smem[];
    __shared__ __align__(8) uint64_t bars[kMaxChunks];
    __shared__ double red[2 * kThreads / 32];
    __shared__ double part[2];
    __shared__ float4 coef_s;

    const uint32_t K = cluster_nctarank(), r = cluster_ctarank();
    const int64_t c = blockIdx.x / K;
    uint32_t vlo, vhi;
    cta_slice(a.m / V, r, K, vlo, vhi);
    const uint32_t nv = vhi - vlo;
    const int nchunks = (int)((nv + a.chunk_vecs - 1) / a.chunk_vecs);
    const uint4* zs = smem;
    const uint4* ds = smem + nv;

    if (threadIdx.x == 0) {
        for (int k = 0; k < nchunks; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) issue_loads<T>(a, c, vlo, vhi, smem, bars, nchunks, 2);

    const InvAffine ia = inv_affine(a.gamma[c], a.beta[c], a.eps, a.flags);
    const float slope = a.slope, inv_slope = a.inv_slope;

    // ---- B1: S1 = sum dy, S2 = sum dy x^ over the resident slice
    float a1[V], a2[V];
#pragma unroll
    for (int k = 0; k < V; ++k) a1[k] = a2[k] = 0.f;
    double d1 = 0.0, d2 = 0.0;
    for (int k = 0; k < nchunks; ++k) {
        mbar_wait(&bars[k], 0);
        const uint32_t c_lo = k * a.chunk_vecs, c_hi = min(nv, c_lo + a.chunk_vecs);
        for (uint32_t v = c_lo + threadIdx.x; v < c_hi; v += kThreads) {
            float fz[V], fd[V];
            unpack<T>(zs[v], fz);
            unpack<T>(ds[v], fd);
#pragma unroll
            for (int q = 0; q < V; ++q) {
                float dy, xh;
                grad_terms(fz[q], fd[q], slope, inv_slope, ia, dy, xh);
                a1[q] += dy;
                a2[q] = fmaf(dy, xh, a2[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < V; ++q) {
            d1 += a1[q];
            d2 += a2[q];
            a1[q] = a2[q] = 0.f;
        }
    }
    double v2[2] = {d1, d2};
    block_sum<2>(v2, red);
    if (threadIdx.x == 0) {
        part[0] = v2[0];
        part[1] = v2[1];
    }
    cluster_arrive_release();
    cluster_wait_acquire();
    if (threadIdx.x == 0) {
        double S1 = 0.0, S2 = 0.0;
        for (uint32_t q = 0; q < K; ++q) {
            S1 += ld_dsmem_f64(&part[0], q);
            S2 += ld_dsmem_f64(&part[1], q);
        }
        coef_s = bwd_coef_from_sums(S1, S2, (double)a.m, a.gamma[c], a.beta[c], a.save_var[c],
                                    a.eps, a.flags);
        if (r == 0) {
            a.dbeta[c] = (float)S1;
            a.dgamma[c] = (float)(gamma_sign(a.gamma[c], a.flags) * S2);
        }
    }
    __syncthreads();
    cluster_arrive_release();

    // ---- B2: dx = alpha dy + kappa y + cc (dx may be dz: this CTA's dz slice is resident)
    const float4 cf = coef_s;
    T* dx = (T*)a.out;
    const uint32_t hw = (uint32_t)a.HW;
    for (uint32_t v = threadIdx.x; v < nv; v += kThreads) {
        float fz[V], fd[V];
        unpack<T>(zs[v], fz);
        unpack<T>(ds[v], fd);
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const bool pos = fz[q] >= 0.f;
            const float y = pos ? fz[q] : fz[q] * inv_slope;
            const float dy = pos ? fd[q] : fd[q] * slope;
            fz[q] = fmaf(cf.x, dy, fmaf(cf.y, y, cf.z));
        }
        const uint32_t j = (vlo + v) * V;
        const uint32_t n = fdiv(j, a.fd_hw);
        st_vec(dx + ((int64_t)n * a.C + c) * a.HW + (j - n * hw), pack<T>(fz));
    }
    cluster_wait_acquire();
}

}  // namespace iabn
