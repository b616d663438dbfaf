// common.cuh -- device helpers shared by the InPlace-ABN kernels (sm_100a).
//
// Nothing here is numerics of the method; it is data movement (16-byte vectors,
// bf16 packing, TMA bulk copies + mbarriers, warp reductions, fast division).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace iabn {

constexpr int kThreads = 256;

// ------------------------------------------------------------------ storage types
template <typename T>
struct Elem;
template <>
struct Elem<float> {
    static constexpr int kVec = 4;  // elements per 16-byte vector
    static constexpr int kBytes = 4;
};
template <>
struct Elem<__nv_bfloat16> {
    static constexpr int kVec = 8;
    static constexpr int kBytes = 2;
};

__device__ __forceinline__ float bf16_bits_to_float(uint32_t h) { return __uint_as_float(h << 16); }

__device__ __forceinline__ uint32_t float_to_bf16_bits(float f) {
    // round to nearest even (NaN kept quiet by the intrinsic)
    return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f));
}

template <typename T>
__device__ __forceinline__ void unpack(const uint4& u, float* f);
template <>
__device__ __forceinline__ void unpack<float>(const uint4& u, float* f) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void unpack<__nv_bfloat16>(const uint4& u, float* f) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = bf16_bits_to_float(w[i] & 0xffffu);
        f[2 * i + 1] = bf16_bits_to_float(w[i] >> 16);
    }
}

template <typename T>
__device__ __forceinline__ uint4 pack(const float* f);
template <>
__device__ __forceinline__ uint4 pack<float>(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
}
template <>
__device__ __forceinline__ uint4 pack<__nv_bfloat16>(const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        w[i] = float_to_bf16_bits(f[2 * i]) | (float_to_bf16_bits(f[2 * i + 1]) << 16);
    return make_uint4(w[0], w[1], w[2], w[3]);
}

template <typename T>
__device__ __forceinline__ float ld_scalar(const T* p);
template <>
__device__ __forceinline__ float ld_scalar<float>(const float* p) { return *p; }
template <>
__device__ __forceinline__ float ld_scalar<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}
template <typename T>
__device__ __forceinline__ void st_scalar(T* p, float v);
template <>
__device__ __forceinline__ void st_scalar<float>(float* p, float v) { *p = v; }
template <>
__device__ __forceinline__ void st_scalar<__nv_bfloat16>(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
}

// 16-byte global accesses, no L1 allocation (data touched once per kernel); stores are
// plain (write-back L2).  ld_vec is the coherent load: the apply kernels use it on
// buffers the same kernel overwrites (z over x, dx over dz in place), which the
// read-only .nc path does not allow.
__device__ __forceinline__ uint4 ld_vec(const void* p) {
    uint4 r;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
// Non-coherent read-only load, not volatile (the compiler may batch and hoist it): only
// for inputs that no thread of the kernel writes (the reduction kernels).
__device__ __forceinline__ uint4 ld_vec_ro(const void* p) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p));
    return r;
}
// (no "memory" clobber: output stores need no ordering w.r.t. this kernel's other
// memory accesses -- nothing in the kernel reads them back -- so shared-memory loads
// of the next vectors may be scheduled ahead of them)
__device__ __forceinline__ void st_vec(void* p, const uint4& v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w));
}

// ------------------------------------------------------------------ fast u32 division
// q = floor(n / d) for all 32-bit n, d >= 1 (Granlund-Montgomery round-up method).
struct FastDiv {
    uint32_t d, m, s;
};
inline FastDiv make_fastdiv(uint32_t d) {
    FastDiv f;
    f.d = d;
    uint32_t s = 0;
    while (s < 32 && (1ull << s) < d) ++s;
    f.s = s;
    f.m = (uint32_t)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
    return f;
}
__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv& f) {
    return (uint32_t)(((uint64_t)__umulhi(n, f.m) + n) >> f.s);
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block sum of NV doubles per thread; result valid in thread 0.
// scratch: >= NV * (blockDim.x / 32) doubles of shared memory.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < NV; ++k) scratch[k * nw + warp] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += scratch[k * nw + w];
            v[k] = t;
        }
    }
}

// ------------------------------------------------------------------ TMA bulk copy + mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// Programmatic dependent launch: a kernel launched with programmatic stream
// serialisation may start while the previous kernel of the stream finishes; every
// kernel calls this before its first global-memory access (read or write), which
// waits until the previous grid has completed and its writes are visible.  A no-op
// for kernels launched without the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// 16-byte shared-memory load by 32-bit shared address (volatile: stays after the
// mbarrier wait that makes the data visible)
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}

// 16-byte shared-memory store by 32-bit shared address
__device__ __forceinline__ void sts128(uint32_t addr, const uint4& v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    // try_wait suspends the warp in hardware until the phase completes (or the
    // time hint expires), so waiting warps do not burn issue slots spinning.
    const uint32_t a = smem_addr(bar);
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1, %2;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity), "n"(0x100000)
        : "memory");
}
// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P;\n}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
// global -> shared bulk copy (TMA engine, SASS UBLKCP), completion counted on bar.
// dst, src 16-byte aligned; bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// global -> L2 bulk prefetch (no destination, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
// L2 cache policies (createpolicy): keep prefetched lines until their bulk copy, then
// let them go first
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_prefetch_l2_hint(const void* src, uint32_t bytes,
                                                      uint64_t pol) {
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src),
                 "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

// ------------------------------------------------------------------ cluster barrier
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// Read a double from the shared memory of CTA `rank` of this cluster (DSMEM).
__device__ __forceinline__ long long ld_dsmem_s64(const long long* local_ptr, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(remote)
                 : "r"((uint32_t)__cvta_generic_to_shared(local_ptr)), "r"(rank));
    long long v;
    asm volatile("ld.shared::cluster.s64 %0, [%1];" : "=l"(v) : "r"(remote));
    return v;
}
__device__ __forceinline__ double ld_dsmem_f64(const double* local_ptr, uint32_t rank) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(remote)
                 : "r"(smem_addr(local_ptr)), "r"(rank));
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote));
    return v;
}

}  // namespace iabn

namespace iabn {
// ------------------------------------------------------------------ packed fp32x2 math (sm_100a:
// FADD2 / FMUL2 / FFMA2 -- two fp32 lanes per instruction)
__device__ __forceinline__ unsigned long long f2_bits(float2 a) {
    return ((unsigned long long)__float_as_uint(a.y) << 32) | __float_as_uint(a.x);
}
__device__ __forceinline__ float2 f2_from(unsigned long long b) {
    return make_float2(__uint_as_float((uint32_t)b), __uint_as_float((uint32_t)(b >> 32)));
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(d);
}
__device__ __forceinline__ float2 mul2(float2 a, float2 b) {
    unsigned long long d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)));
    return f2_from(d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2_bits(a)), "l"(f2_bits(b)), "l"(f2_bits(c)));
    return f2_from(d);
}

// bf16 pair (one 32-bit word) -> fp32 pair, exact.
__device__ __forceinline__ float2 bf16x2_to_f2(uint32_t w) {
    return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}
// (lo - k, hi - k) in fp32 straight from a bf16 pair: mixed-precision sub.f32.bf16
// (SASS FHADD.BF16 with half select, no separate unpack).
__device__ __forceinline__ float2 bf16x2_sub_f2(uint32_t w, float k) {
    float a, b;
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
        "sub.f32.bf16 %0, lo, %3;\n\tsub.f32.bf16 %1, hi, %3;\n}"
        : "=f"(a), "=f"(b)
        : "r"(w), "f"(k));
    return make_float2(a, b);
}
// Packed bf16 helpers of the backward reduction (no unpacking):
// 1.0 in each half where the bf16 value is < 0 (-0.0 is not), else 0.0 (HSET2.BF16)
__device__ __forceinline__ uint32_t bf16x2_ind_neg(uint32_t w) {
    uint32_t d;
    asm("set.lt.bf16x2.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(w), "r"(0u));
    return d;
}
// acc.{x,y} += w.{lo,hi}  (FHADD.BF16: fp32 add of a bf16 operand, exact widening)
__device__ __forceinline__ void bf16x2_acc(float2& acc, uint32_t w) {
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
        "add.f32.bf16 %0, lo, %0;\n\tadd.f32.bf16 %1, hi, %1;\n}"
        : "+f"(acc.x), "+f"(acc.y)
        : "r"(w));
}
// acc.{x,y} += a.{lo,hi} * b.{lo,hi}  (FHFMA.BF16: bf16 x bf16 product, fp32 accumulate)
__device__ __forceinline__ void bf16x2_acc_mul(float2& acc, uint32_t a, uint32_t b) {
    asm("{\n\t.reg .b16 a0, a1, b0, b1;\n\tmov.b32 {a0, a1}, %2;\n\tmov.b32 {b0, b1}, %3;\n\t"
        "fma.rn.f32.bf16 %0, a0, b0, %0;\n\tfma.rn.f32.bf16 %1, a1, b1, %1;\n}"
        : "+f"(acc.x), "+f"(acc.y)
        : "r"(a), "r"(b));
}

// fp32 pair -> bf16 pair, round to nearest even (F2FP.BF16.F32.PACK_AB).
__device__ __forceinline__ uint32_t f2_to_bf16x2(float2 v) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v.x, v.y);
    return *reinterpret_cast<uint32_t*>(&h);
}

// A 16-byte vector as fp32 pairs: 4 pairs (bf16) or 2 pairs (fp32).
template <typename T>
struct Pairs;
template <>
struct Pairs<float> {
    static constexpr int kN = 2;
    __device__ __forceinline__ static void load(const uint4& u, float2* p) {
        p[0] = make_float2(__uint_as_float(u.x), __uint_as_float(u.y));
        p[1] = make_float2(__uint_as_float(u.z), __uint_as_float(u.w));
    }
    __device__ __forceinline__ static void load_sub(const uint4& u, float k, float2* p) {
        load(u, p);
        p[0] = add2(p[0], make_float2(-k, -k));
        p[1] = add2(p[1], make_float2(-k, -k));
    }
    __device__ __forceinline__ static uint4 store(const float2* p) {
        return make_uint4(__float_as_uint(p[0].x), __float_as_uint(p[0].y), __float_as_uint(p[1].x),
                          __float_as_uint(p[1].y));
    }
};
template <>
struct Pairs<__nv_bfloat16> {
    static constexpr int kN = 4;
    __device__ __forceinline__ static void load(const uint4& u, float2* p) {
        p[0] = bf16x2_to_f2(u.x);
        p[1] = bf16x2_to_f2(u.y);
        p[2] = bf16x2_to_f2(u.z);
        p[3] = bf16x2_to_f2(u.w);
    }
    __device__ __forceinline__ static void load_sub(const uint4& u, float k, float2* p) {
        p[0] = bf16x2_sub_f2(u.x, k);
        p[1] = bf16x2_sub_f2(u.y, k);
        p[2] = bf16x2_sub_f2(u.z, k);
        p[3] = bf16x2_sub_f2(u.w, k);
    }
    __device__ __forceinline__ static uint4 store(const float2* p) {
        return make_uint4(f2_to_bf16x2(p[0]), f2_to_bf16x2(p[1]), f2_to_bf16x2(p[2]),
                          f2_to_bf16x2(p[3]));
    }
};
}  // namespace iabn
