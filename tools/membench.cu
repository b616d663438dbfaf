// tools/membench.cu -- HBM data-movement microbenchmarks on B200 (sm_100a) used to
// choose the channel-resident kernel design: how fast can TMA bulk copies
// (cp.async.bulk) stream HBM into shared memory, vs. plain 16-byte LDG/STG?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
//   ./membench            (prints one line per variant: GB/s of bytes moved)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sa(s)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }

// mode 0: TMA read only (sum a word per chunk so it is not dead)
// mode 1: TMA read + STG copy out (threads read smem, write global)
// mode 2: TMA read + TMA bulk store out
__global__ void tma_stream(const uint4* __restrict__ in, uint4* __restrict__ out, size_t nvec,
                           int chunk_vecs, int stages, int mode, unsigned* sink) {
    extern __shared__ __align__(128) uint4 sm[];
    __shared__ uint64_t bar[32];
    const size_t nchunks = nvec / chunk_vecs;
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    size_t first = blockIdx.x;
    int issued = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            size_t ch = first + (size_t)s * gridDim.x;
            if (ch >= nchunks) break;
            expect_tx(&bar[s], chunk_vecs * 16);
            g2s(sm + (size_t)s * chunk_vecs, in + ch * chunk_vecs, chunk_vecs * 16, &bar[s]);
        }
    }
    unsigned acc = 0;
    int it = 0;
    for (size_t ch = first; ch < nchunks; ch += gridDim.x, ++it) {
        const int s = it % stages;
        const uint32_t par = (it / stages) & 1;
        mwait(&bar[s], par);
        uint4* buf = sm + (size_t)s * chunk_vecs;
        if (mode == 0) {
            if (threadIdx.x < 32) acc += buf[threadIdx.x].x;
        } else if (mode == 1) {
            for (int v = threadIdx.x; v < chunk_vecs; v += blockDim.x) {
                uint4 u = buf[v];
                asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(out + ch * chunk_vecs + v), "r"(u.x), "r"(u.y), "r"(u.z), "r"(u.w) : "memory");
            }
        } else {
            if (threadIdx.x == 0) {
                s2g(out + ch * chunk_vecs, buf, chunk_vecs * 16);
                bulk_commit();
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (mode == 2) bulk_wait_read<0>();
            size_t nx = ch + (size_t)stages * gridDim.x;
            if (nx < nchunks) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                expect_tx(&bar[s], chunk_vecs * 16);
                g2s(buf, in + nx * chunk_vecs, chunk_vecs * 16, &bar[s]);
            }
        }
    }
    if (mode == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (acc == 0xdeadbeef) *sink = acc;
}

// plain LDG/STG, 2 reads : 1 write (the fused backward's mix: z, dz in, dx out)
template <int UNROLL>
__global__ void ldg_2r1w(const uint4* __restrict__ in, const uint4* __restrict__ in2,
                         uint4* __restrict__ out, size_t nvec) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += stride * UNROLL) {
        uint4 r[UNROLL], q[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            size_t i = base + u * stride;
            if (i < nvec) {
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w) : "l"(in + i));
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q[u].x), "=r"(q[u].y), "=r"(q[u].z), "=r"(q[u].w) : "l"(in2 + i));
            }
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            size_t i = base + u * stride;
            if (i < nvec) out[i] = make_uint4(r[u].x ^ q[u].x, r[u].y ^ q[u].y, r[u].z ^ q[u].z, r[u].w ^ q[u].w);
        }
    }
}

// plain LDG/STG: read-only reduce (mode 0) or copy (mode 1), UNROLL vectors in flight
template <int UNROLL>
__global__ void ldg_stream(const uint4* __restrict__ in, uint4* __restrict__ out, size_t nvec,
                           int mode, unsigned* sink) {
    unsigned acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (size_t base = (size_t)blockIdx.x * blockDim.x + threadIdx.x; base < nvec; base += stride * UNROLL) {
        uint4 r[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            size_t i = base + u * stride;
            if (i < nvec) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r[u].x), "=r"(r[u].y), "=r"(r[u].z), "=r"(r[u].w) : "l"(in + i));
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            size_t i = base + u * stride;
            if (i < nvec) {
                if (mode == 0) acc += r[u].x ^ r[u].w;
                else out[i] = r[u];
            }
        }
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main(int argc, char** argv) {
    const bool quick = argc > 1;  // any argument: the LDG variants only
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = (size_t)1644 << 20;  // ~1.64 GB, the cfg4 bf16 tensor
    const size_t nvec = bytes / 16;
    uint4 *in, *out;
    unsigned* sink;
    CK(cudaMalloc(&in, bytes));
    CK(cudaMalloc(&out, bytes));
    CK(cudaMalloc(&sink, 4));
    uint4* in2;
    CK(cudaMalloc(&in2, bytes));
    CK(cudaMemset(in, 1, bytes));
    CK(cudaMemset(in2, 2, bytes));
    CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto launch, double moved, const char* name) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(a);
        const int reps = 10;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaError_t e = cudaGetLastError();
        printf("%-48s %8.1f GB/s  (%.3f ms)%s\n", name, moved / (ms / reps * 1e-3) / 1e9, ms / reps,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    char name[128];
    for (int u : {4, 8, 16}) {
        for (int bps : {4, 8}) {
            int grid = sms * bps;
            snprintf(name, sizeof name, "ldg read  unroll=%d ctas/sm=%d", u, bps);
            if (u == 4) timeit([&] { ldg_stream<4><<<grid, 256>>>(in, out, nvec, 0, sink); }, bytes, name);
            if (u == 8) timeit([&] { ldg_stream<8><<<grid, 256>>>(in, out, nvec, 0, sink); }, bytes, name);
            if (u == 16) timeit([&] { ldg_stream<16><<<grid, 256>>>(in, out, nvec, 0, sink); }, bytes, name);
            snprintf(name, sizeof name, "ldg copy  unroll=%d ctas/sm=%d", u, bps);
            if (u == 4) timeit([&] { ldg_stream<4><<<grid, 256>>>(in, out, nvec, 1, sink); }, 2.0 * bytes, name);
            if (u == 8) timeit([&] { ldg_stream<8><<<grid, 256>>>(in, out, nvec, 1, sink); }, 2.0 * bytes, name);
            if (u == 16) timeit([&] { ldg_stream<16><<<grid, 256>>>(in, out, nvec, 1, sink); }, 2.0 * bytes, name);
        }
    }
    for (int bps : {2, 4, 8}) {
        const int grid = sms * bps;
        snprintf(name, sizeof name, "ldg 2r1w  unroll=4 ctas/sm=%d", bps);
        timeit([&] { ldg_2r1w<4><<<grid, 256>>>(in, in2, out, nvec); }, 3.0 * bytes, name);
        snprintf(name, sizeof name, "ldg 2r1w  unroll=8 ctas/sm=%d", bps);
        timeit([&] { ldg_2r1w<8><<<grid, 256>>>(in, in2, out, nvec); }, 3.0 * bytes, name);
    }
    if (quick) return 0;
    for (int mode : {0, 1, 2}) {
        for (int ckb : {4, 8, 16, 32}) {
            for (int bps : {1, 2, 4}) {
                for (int stages : {2, 4, 8}) {
                    size_t smem = (size_t)stages * ckb * 1024;
                    if (smem * bps > 220 * 1024 || stages > 32) continue;
                    int cv = ckb * 1024 / 16;
                    int grid = sms * bps;
                    snprintf(name, sizeof name, "tma mode=%d chunk=%dKB ctas/sm=%d stages=%d", mode, ckb, bps, stages);
                    timeit([&] { tma_stream<<<grid, 256, smem>>>(in, out, nvec, cv, stages, mode, sink); },
                           mode == 0 ? (double)bytes : 2.0 * bytes, name);
                }
            }
        }
    }
    return 0;
}
