// probe_f16p.cu — measurement probe (not part of libproxyattn): can the PV MMA take P as
// fp16 (A from TMEM) against bf16 V (B from shared memory) in one tcgen05.mma kind::f16,
// and what does ex2.approx.f16x2 cost on MUFU against ex2.approx.ftz.f32?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2509_24745_b200/csrc \
//        scripts/probe_f16p.cu -o scripts/probe_f16p && scripts/probe_f16p
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"
#include "tma_host.h"

using namespace pa;

constexpr int kBox = 128 * 64 * 2;
constexpr int kTile = 2 * kBox;

// C[128][128] = A[128][128] (fp16 or bf16 bits, staged in TMEM) x B[128][128] (bf16, MN-major)
__global__ void __launch_bounds__(128, 1) mixed_kernel(const __grid_constant__ CUtensorMap tmB,
                                                       const uint16_t* __restrict__ A, float* __restrict__ C,
                                                       uint32_t a_format) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sB = smem;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kTile);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&bar[2], 128);
        fence_barrier_init();
    }
    if (warp == 0) tmem_alloc(tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *tslot;
    const uint32_t lane_off = static_cast<uint32_t>(warp * 32) << 16;
    {
        const int rr = warp * 32 + lane;
        uint32_t pk[2][32];
        const uint32_t* arow = reinterpret_cast<const uint32_t*>(A + rr * 128);
#pragma unroll
        for (int c = 0; c < 64; ++c) pk[c >> 5][c & 31] = arow[c];
        tmem_st32(tbase + lane_off + 256, pk[0]);
        tmem_st32(tbase + lane_off + 256 + 32, pk[1]);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&bar[2]);
    }
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar[0], kTile);
        tma_load_2d(sB, &tmB, &bar[0], 0, 0);
        tma_load_2d(sB + kBox, &tmB, &bar[0], 64, 0);
        mbar_wait(&bar[0], 0);
        mbar_wait(&bar[2], 0);
        tc_fence_after();
        const uint32_t idesc = (1u << 4) | (a_format << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                               ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t b_addr = smem_u32(sB);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
            umma_ts(tbase, tbase + 256 + kk * 8, sdesc_sw128(b_addr + kk * 2048, kBox, 1024), idesc, kk > 0);
        tc_commit(&bar[1]);
    }
    __syncwarp();
    mbar_wait(&bar[1], 0);
    tc_fence_after();
    const int rr = warp * 32 + lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld32(tbase + lane_off + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) C[rr * 128 + c * 32 + e] = __uint_as_float(v[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

// MUFU throughput: each thread issues n ex2 instructions on independent chains
template <bool kF16x2>
__global__ void mufu_kernel(float* out, int n, long long* cycles) {
    float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
    uint32_t h0 = 0x3c003c00u, h1 = 0x3c003c01u, h2 = 0x3c003c02u, h3 = 0x3c003c03u;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (kF16x2) {
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2));
            asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
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
    std::vector<uint16_t> Ah(128 * 128), Ab(128 * 128), Bh(128 * 128);
    std::vector<float> Af(128 * 128), Bf(128 * 128);
    srand(1);
    for (int i = 0; i < 128 * 128; ++i) {
        // P-like values in (0, 1]: exactly representable in fp16 (11 bits), NOT in bf16 (8 bits)
        const float p = (1 + rand() % 2047) / 2048.0f;
        __half hp = __float2half_rn(p);
        Ah[i] = *reinterpret_cast<uint16_t*>(&hp);
        Af[i] = __half2float(hp);
        __nv_bfloat16 bp = __float2bfloat16_rn(p);
        Ab[i] = *reinterpret_cast<uint16_t*>(&bp);
        __nv_bfloat16 b = __float2bfloat16_rn((rand() % 2001 - 1000) / 250.0f);
        Bh[i] = *reinterpret_cast<uint16_t*>(&b);
        Bf[i] = __bfloat162float(b);
    }
    uint16_t *dA, *dB;
    float* dC;
    cudaMalloc(&dA, 128 * 128 * 2);
    cudaMalloc(&dB, 128 * 128 * 2);
    cudaMalloc(&dC, 128 * 128 * 4);
    cudaMemcpy(dB, Bh.data(), 128 * 128 * 2, cudaMemcpyHostToDevice);
    CUtensorMap mb;
    if (!make_map_bf16_sw128(&mb, dB, 128, 128, 128)) { printf("map failed\n"); return 1; }
    const size_t sm = 1024 + kTile + 64;
    cudaFuncSetAttribute(mixed_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    std::vector<float> C(128 * 128);
    for (int mode = 0; mode < 2; ++mode) {   // 0: A fp16 with a_format F16 (mixed), 1: A bf16 with BF16
        cudaMemcpy(dA, mode == 0 ? Ah.data() : Ab.data(), 128 * 128 * 2, cudaMemcpyHostToDevice);
        mixed_kernel<<<1, 128, sm>>>(mb, dA, dC, mode == 0 ? 0u : 1u);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(C.data(), dC, 128 * 128 * 4, cudaMemcpyDeviceToHost);
        double err = 0, ref_mag = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < 128; ++j) {
                double r = 0;
                for (int k = 0; k < 128; ++k) {
                    const double a = mode == 0 ? Af[i * 128 + k]
                                               : __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(&Ab[i * 128 + k]));
                    r += a * Bf[k * 128 + j];
                }
                err = fmax(err, fabs(r - C[i * 128 + j]));
                ref_mag = fmax(ref_mag, fabs(r));
            }
        printf("%s: max |C - ref| = %.3e (max |ref| %.2f)\n",
               mode == 0 ? "A fp16 (TMEM) x B bf16 (smem), a_format=F16, b_format=BF16"
                         : "A bf16 x B bf16 (control)", err, ref_mag);
    }
    float* dout;
    long long* dcyc;
    cudaMalloc(&dout, 148 * 512 * 4);
    cudaMalloc(&dcyc, 148 * 8);
    for (int f16 = 0; f16 < 2; ++f16) {
        for (int rep = 0; rep < 2; ++rep) {
            if (f16) mufu_kernel<true><<<148, 512>>>(dout, 4096, dcyc);
            else mufu_kernel<false><<<148, 512>>>(dout, 4096, dcyc);
        }
        cudaDeviceSynchronize();
        long long cyc;
        cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
        const double instr = 4096.0 * 4 * 16;    // warp-instructions per SM (16 warps)
        printf("%s: %.2f clk per warp-instruction per SM (%.2f elements/clk/SM)\n",
               f16 ? "ex2.approx.f16x2" : "ex2.approx.ftz.f32", cyc / instr,
               (f16 ? 64.0 : 32.0) * instr / cyc);
    }
    return 0;
}
