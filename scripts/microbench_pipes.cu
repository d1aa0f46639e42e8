// Microbenchmark of per-SM instruction throughput on sm_100a for the softmax's instruction
// mix: MUFU.EX2, FFMA2, FADD2, F2FP (bf16x2 pack), FMNMX3, FFMA.  Each thread runs 8
// independent chains; clock64 around the loop; reports instructions/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_pipes.cu && /tmp/mb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) { uint64_t d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ uint32_t f2bf(float a, float b) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float r; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float r; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }

template <int OP>
__global__ void k(float* out, long long* cyc, float seed) {
    float x[8];
    uint64_t y[8];
    uint32_t u[8];
    for (int i = 0; i < 8; ++i) { x[i] = seed * (i + 1) * 1e-3f; y[i] = (uint64_t)__float_as_uint(x[i]) | ((uint64_t)__float_as_uint(x[i] + 1) << 32); u[i] = i; }
    const uint64_t c2 = y[3];
    __syncthreads();
    long long t0 = clock64();
#pragma unroll 4
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) x[i] = ex2(x[i]);
            if (OP == 1) y[i] = ffma2(y[i], c2, y[i]);
            if (OP == 2) y[i] = fadd2(y[i], c2);
            if (OP == 3) u[i] ^= f2bf(x[i], __uint_as_float(u[i]));
            if (OP == 4) x[i] = fmax3(x[i], x[(i + 1) & 7], seed);
            if (OP == 5) x[i] = ffma(x[i], seed, x[i]);
            if (OP == 6) { x[i] = ex2(x[i]); u[i] ^= f2bf(x[(i + 4) & 7], __uint_as_float(u[i])); }   // MUFU + F2FP
            if (OP == 7) { x[i] = ex2(x[i]); y[i] = ffma2(y[i], c2, y[i]); }                         // MUFU + FFMA2
            if (OP == 8) { x[i] = ex2(x[i]); u[i] = (u[i] + 0x7fffu + ((u[i] >> 16) & 1u)) & 0xffff0000u; }  // MUFU + ALU bf16 RNE
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float((uint32_t)y[i]) + __uint_as_float(u[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const char* names[] = {"MUFU.EX2", "FFMA2", "FADD2", "F2FP.BF16x2", "FMNMX3", "FFMA",
                           "EX2+F2FP", "EX2+FFMA2", "EX2+ALU-RNE"};
    float* out; long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 1024);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    for (int warps : {4, 8, 16, 32}) {
        for (int op = 0; op < 9; ++op) {
            auto run = [&]() {
                switch (op) {
                    case 0: k<0><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 1: k<1><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 2: k<2><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 3: k<3><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 4: k<4><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 5: k<5><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 6: k<6><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 7: k<7><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                    case 8: k<8><<<sms, warps * 32>>>(out, cyc, 0.5f); break;
                }
            };
            run();
            cudaDeviceSynchronize();
            run();
            cudaDeviceSynchronize();
            long long c;
            cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
            const double inst = (double)warps * ITERS * 8;       // warp-instructions per SM
            printf("warps/SM %2d  %-12s %8.3f warp-inst/clk/SM  (%6.2f clk per warp-inst per SMSP)\n",
                   warps, names[op], inst / c, 4.0 * c / inst);
        }
    }
    return 0;
}
