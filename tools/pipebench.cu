// tools/pipebench.cu -- issue/pipe throughput of the instructions the fused kernels'
// inner loops are made of, on B200 (sm_100a): cycles per warp-instruction per SMSP
// with W warps per SMSP, 8 independent chains per thread.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipebench tools/pipebench.cu
//   tools/pipebench
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kIters = 4096;

template <int OP>
__device__ __forceinline__ void op8(float (&f)[8], uint32_t (&u)[8], uint32_t k, uint32_t saddr) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (OP == 0) {  // FFMA (3 registers)
            asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(__uint_as_float(u[i])), "f"(__uint_as_float(k)));
        } else if (OP == 1) {  // FFMA2
            asm volatile("{\n\t.reg .b64 a, b, c;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %2};\n\t"
                         "mov.b64 c, {%3, %3};\n\tfma.rn.f32x2 a, a, b, c;\n\tmov.b64 {%0, %1}, a;\n}"
                         : "+f"(f[i]), "+f"(f[(i + 1) & 7])
                         : "f"(__uint_as_float(u[i])), "f"(__uint_as_float(k)));
        } else if (OP == 2) {  // FHFMA.BF16 (f32 += bf16 * bf16)
            asm volatile("{\n\t.reg .b16 a0, a1;\n\tmov.b32 {a0, a1}, %1;\n\t"
                         "fma.rn.f32.bf16 %0, a0, a1, %0;\n}"
                         : "+f"(f[i]) : "r"(u[i] ^ k));
        } else if (OP == 3) {  // FHADD.BF16 (f32 += bf16)
            asm volatile("{\n\t.reg .b16 a0, a1;\n\tmov.b32 {a0, a1}, %1;\n\t"
                         "add.f32.bf16 %0, a0, %0;\n}"
                         : "+f"(f[i]) : "r"(u[i] ^ k));
        } else if (OP == 4) {  // HSET2.BF16
            asm volatile("set.lt.bf16x2.bf16x2 %0, %0, %1;" : "+r"(u[i]) : "r"(k));
        } else if (OP == 5) {  // HFMA2.BF16
            asm volatile("fma.rn.bf16x2 %0, %0, %1, %2;" : "+r"(u[i]) : "r"(k), "r"(k ^ 0x3f803f80u));
        } else if (OP == 6) {  // FSEL
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\tselp.f32 %0, %0, %1, p;\n}"
                         : "+f"(f[i]) : "f"(__uint_as_float(u[i])), "r"(k));
        } else if (OP == 7) {  // unpack lo half: IMAD.U32 / SHF (x << 16)
            asm volatile("shl.b32 %0, %0, 16;" : "+r"(u[i]));
        } else if (OP == 8) {  // LOP3 (x & 0xffff0000)
            asm volatile("and.b32 %0, %0, %1;" : "+r"(u[i]) : "r"(k));
        } else if (OP == 9) {  // LDS.128 (conflict-free)
            uint4 v;
            asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                         : "r"(saddr + (uint32_t)i * 512u));
            u[i] ^= v.x ^ v.w;
        } else if (OP == 10) {  // FADD2
            asm volatile("{\n\t.reg .b64 a, b;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 b, {%2, %2};\n\t"
                         "add.rn.f32x2 a, a, b;\n\tmov.b64 {%0, %1}, a;\n}"
                         : "+f"(f[i]), "+f"(f[(i + 1) & 7])
                         : "f"(__uint_as_float(u[i])));
        } else if (OP == 11) {  // FSETP
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, 0f00000000;\n\tselp.u32 %0, 1, 0, p;\n}"
                         : "=r"(u[i]) : "f"(f[i]));
        } else if (OP == 12) {  // F2FP pack
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(f[i]), "f"(f[(i + 3) & 7]));
        }
    }
}

template <int OP>
__global__ void bench(unsigned long long* cyc, float* sink, uint32_t k) {
    __shared__ __align__(16) uint4 sm[8 * 32 * 2];
    float f[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = (float)(threadIdx.x + i);
        u[i] = threadIdx.x * 0x9e3779b9u + i;
    }
    for (int i = threadIdx.x; i < 8 * 32 * 2; i += blockDim.x) sm[i] = make_uint4(i, i, i, i);
    __syncthreads();
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) * 16u;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) op8<OP>(f, u, k, sa);
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = 0.f;
    for (int i = 0; i < 8; ++i) s += f[i] + (float)u[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms) {
    unsigned long long* cyc;
    float* sink;
    cudaMalloc(&cyc, sms * sizeof(unsigned long long));
    cudaMalloc(&sink, sms * 1024 * sizeof(float));
    printf("%-28s", name);
    for (int w : {1, 2, 4, 8}) {  // warps per SMSP
        const int threads = 128 * w;
        bench<OP><<<sms, threads>>>(cyc, sink, 7u);
        bench<OP><<<sms, threads>>>(cyc, sink, 7u);
        cudaDeviceSynchronize();
        unsigned long long c[1024];
        cudaMemcpy(c, cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < sms; ++i) avg += (double)c[i];
        avg /= sms;
        // warp-instructions of the op per SMSP: w warps x kIters x 8
        printf("  W=%d %6.2f", w, avg / ((double)w * kIters * 8));
    }
    printf("   cycles / warp-instr / SMSP\n");
    cudaFree(cyc);
    cudaFree(sink);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("FFMA", sms);
    run<1>("FFMA2", sms);
    run<10>("FADD2", sms);
    run<2>("FHFMA.BF16 (f32+=bf16*bf16)", sms);
    run<3>("FHADD.BF16 (f32+=bf16)", sms);
    run<4>("HSET2.BF16", sms);
    run<5>("HFMA2.BF16", sms);
    run<6>("FSEL (+ISETP)", sms);
    run<11>("FSETP (+SEL)", sms);
    run<7>("SHL (unpack lo)", sms);
    run<8>("LOP3 (unpack hi)", sms);
    run<12>("F2FP.BF16 pack", sms);
    run<9>("LDS.128", sms);
    return 0;
}
