// Microbenchmark of tcgen05.mma throughput on sm_100a (one CTA per SM, back-to-back MMAs
// from a single thread, commit + wait at the end) for the operand modes the attention
// kernel can use: SS (A and B from shared memory) vs TS (A from TMEM), N = 128 / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o /tmp/mbu scripts/microbench_umma.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2509_24745_b200/csrc/sm100.cuh"

using namespace pa;

template <int MODE, int N>   // MODE 0 = SS, 1 = TS
__global__ void __launch_bounds__(128, 1) k(long long* cyc, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tb = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t idesc = idesc_bf16_f32(128, N, 0, MODE == 1 ? 1 : 0);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                if (MODE == 0)
                    umma_ss(tb, sdesc_sw128(a + off, 16, 1024), sdesc_sw128(b + off, 16, 1024), idesc, 1);
                else
                    umma_ts(tb, tb + 384 + kk * 8, sdesc_sw128(b + kk * 2048, 16384, 1024), idesc, 1);
            }
        }
        tc_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc(tb, 512); }
}

template <int MODE, int N>
void run(const char* name, int sms) {
    long long* cyc;
    cudaMalloc(&cyc, sizeof(long long) * sms);
    cudaFuncSetAttribute(k<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 2000;
    k<MODE, N><<<sms, 128, 100 * 1024>>>(cyc, iters);
    cudaDeviceSynchronize();
    k<MODE, N><<<sms, 128, 100 * 1024>>>(cyc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 16 * 8.0 * iters;
    printf("%-26s %s: %7.1f clk per MMA (K=16), %7.0f flop/clk/SM (%.0f%% of 8192)\n", name,
           cudaGetErrorString(e), c / (8.0 * iters), flops / c, 100.0 * flops / c / 8192.0);
    cudaFree(cyc);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 128>("SS M=128 N=128", sms);
    run<1, 128>("TS M=128 N=128 (B MN-major)", sms);
    run<0, 256>("SS M=128 N=256", sms);
    run<0, 64>("SS M=128 N=64", sms);
    return 0;
}
