// probe_mufu.cu — measurement probe (not part of libproxyattn): MUFU.EX2 throughput per SM for
// ex2.approx.ftz.f32, ex2.approx.f16x2 and ex2.approx.ftz.bf16x2 (each lowers to MUFU.EX2
// instructions; the packed forms to two per pair), 16 warps per SM on independent chains.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/probe_mufu.cu -o /tmp/probe_mufu
#include <cstdint>
#include <cstdio>

template <int kMode>
__global__ void mufu_kernel(float* out, int n, long long* cycles) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
    uint32_t h0 = 0x3c003c00u ^ threadIdx.x, h1 = 0x3c003c01u, h2 = 0x3c003c02u, h3 = 0x3c003c03u;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (kMode == 1) {
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
        } else if (kMode == 2) {
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2));
            asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
        } else {
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
        }
    }
    const long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + __uint_as_float(h0 ^ h1 ^ h2 ^ h3);
}

int main() {
    float* dout;
    long long* dcyc;
    cudaMalloc(&dout, 148 * 512 * 4);
    cudaMalloc(&dcyc, 148 * 8);
    const char* names[3] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) mufu_kernel<0><<<148, 512>>>(dout, 4096, dcyc);
            if (mode == 1) mufu_kernel<1><<<148, 512>>>(dout, 4096, dcyc);
            if (mode == 2) mufu_kernel<2><<<148, 512>>>(dout, 4096, dcyc);
        }
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", names[mode], cudaGetErrorString(e)); return 1; }
        long long cyc;
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        const double instr = 4096.0 * 4 * 16;    // PTX instructions per SM (16 warps), per warp
        const double elems = instr * 32 * (mode ? 2 : 1);
        printf("%s: %.2f clk per PTX warp-instruction per SM, %.2f exp2 results/clk/SM\n", names[mode],
               cyc / instr, elems / cyc);
    }
    return 0;
}
