// tools/gridbar.cu -- cost of a software grid barrier (atomic arrive + acquire poll)
// on B200: a cooperative launch of G blocks doing NB barriers and nothing else.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridbar tools/gridbar.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_barrier(unsigned* cnt, unsigned target, int sleep_ns) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        unsigned v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory");
            if (v >= target) break;
            if (sleep_ns) __nanosleep(sleep_ns);
        }
    }
    __syncthreads();
}

__global__ void bar_kernel(unsigned* cnt, int nb, int sleep_ns) {
    for (int i = 1; i <= nb; ++i) grid_barrier(cnt, i * gridDim.x, sleep_ns);
}

int main() {
    unsigned* cnt;
    cudaMalloc(&cnt, 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int sleep_ns : {0, 64}) {
        for (int G : {16, 64, 148, 296, 592}) {
            for (int nb : {0, 2, 8}) {
                cudaEvent_t a, b;
                cudaEventCreate(&a);
                cudaEventCreate(&b);
                const int reps = 200;
                float best = 1e9f;
                for (int trial = 0; trial < 3; ++trial) {
                    cudaEventRecord(a, st);
                    for (int r = 0; r < reps; ++r) {
                        cudaMemsetAsync(cnt, 0, 4, st);
                        cudaLaunchConfig_t cfg = {};
                        cfg.gridDim = dim3(G);
                        cfg.blockDim = dim3(256);
                        cfg.stream = st;
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeCooperative;
                        at[0].val.cooperative = 1;
                        cfg.attrs = at;
                        cfg.numAttrs = 1;
                        cudaLaunchKernelEx(&cfg, bar_kernel, cnt, nb, sleep_ns);
                    }
                    cudaEventRecord(b, st);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    best = ms < best ? ms : best;
                }
                printf("sleep %2d ns  G %4d  barriers %d: %7.2f us per launch (incl. memset)\n",
                       sleep_ns, G, nb, best * 1e3f / reps);
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
