// Probe (experiments): the element mapping of tcgen05.cp.cta_group::1.128x256b from a
// no-swizzle shared-memory matrix descriptor into TMEM, read back per warp quarter with
// tcgen05.ld.32x32b.x8.  Prints, for TMEM lanes 0..127 and columns 0..7, the 32-bit word
// index of shared memory it came from, for (LBO, SBO) given on the command line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tmem_probe tools/tmem_probe.cu
//   tools/tmem_probe 128 256
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out, uint32_t lbo, uint32_t sbo, uint32_t timing_iters,
                      unsigned long long* cycles) {
    __shared__ __align__(1024) uint32_t buf[1024 * 8];  // 32 KB
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t taddr_holder;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (uint32_t i = tid; i < 1024 * 8; i += blockDim.x) buf[i] = i;
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        const uint32_t h = (uint32_t)__cvta_generic_to_shared(&taddr_holder);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(h));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t taddr = taddr_holder;
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(buf);
    auto desc = [&](uint32_t addr) {
        uint64_t d = 0;
        d |= (uint64_t)((addr >> 4) & 0x3fff);
        d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
        d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
        d |= (uint64_t)1 << 46;  // version 1 (sm_100)
        return d;
    };
    if (tid == 0) {
        const uint64_t d = desc(sa);
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(d));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a));
    }
    {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0; selp.u32 %0, 1, 0, P;}"
                         : "=r"(ok) : "r"(bar_a) : "memory");
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr + ((warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 8; ++c) out[(warp * 32 + lane) * 8 + c] = r[c];
    // timing: back-to-back 4 KB copies (one thread) and 32x32b.x8 loads (all warps)
    if (timing_iters) {
        __syncthreads();
        unsigned long long t0 = clock64();
        if (tid == 0) {
            for (uint32_t i = 0; i < timing_iters; ++i) {
                const uint64_t d = desc(sa + (i & 7) * 4096);
                asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr + 8 * (i & 7)), "l"(d));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar_a));
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{.reg .pred P; mbarrier.try_wait.parity.shared::cta.b64 P, [%1], 1; selp.u32 %0, 1, 0, P;}"
                             : "=r"(ok) : "r"(bar_a) : "memory");
            cycles[0] = clock64() - t0;
        }
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        t0 = clock64();
        uint32_t acc = 0;
        for (uint32_t i = 0; i < timing_iters; ++i) {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                           "=r"(r[6]), "=r"(r[7])
                         : "r"(taddr + ((warp * 32) << 16) + 8 * (i & 7)));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            acc += r[0] ^ r[7];
        }
        __syncthreads();
        if (tid == 0) cycles[1] = clock64() - t0;
        if (acc == 0xdeadbeef) out[0] = acc;
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(taddr));
}

int main(int argc, char** argv) {
    const uint32_t lbo = argc > 1 ? atoi(argv[1]) : 128, sbo = argc > 2 ? atoi(argv[2]) : 256;
    uint32_t* d;
    unsigned long long* cyc;
    cudaMalloc(&d, 128 * 8 * 4);
    cudaMalloc(&cyc, 16);
    probe<<<1, 128>>>(d, lbo, sbo, 256, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error: %s\n", cudaGetErrorString(e));
        return 1;
    }
    uint32_t h[128 * 8];
    unsigned long long hc[2];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    printf("LBO=%u SBO=%u: TMEM lane -> smem words of columns 0..7\n", lbo, sbo);
    for (int l = 0; l < 128; ++l) {
        if (l < 20 || l % 16 == 0 || l > 124) {
            printf("lane %3d:", l);
            for (int c = 0; c < 8; ++c) printf(" %5u", h[l * 8 + c]);
            printf("\n");
        }
    }
    printf("256 x 4KB tcgen05.cp (one thread): %llu cycles (%.1f B/cycle)\n", hc[0],
           256.0 * 4096 / hc[0]);
    printf("256 x 32x32b.x8 ld per warp, 4 warps: %llu cycles (%.1f B/cycle)\n", hc[1],
           256.0 * 4 * 32 * 32 / hc[1]);
    return 0;
}
