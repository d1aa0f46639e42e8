// debug_umma.cu — diagnostic tcgen05 GEMM tile that pins the descriptor encodings used by
// the attention and score kernels (proxyattn_debug_umma, tests/test_gpu_parity.py).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace pa {
namespace {

constexpr int kBox = 128 * 64 * 2;
constexpr int kTile = 2 * kBox;

// ------------------------------------------------------------ diagnostic GEMM --
__global__ void __launch_bounds__(128, 1)
debug_umma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __nv_bfloat16* __restrict__ A, float* __restrict__ Css,
                  float* __restrict__ Cts) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kTile;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 2 * kTile);
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
    // A (row-major [128][128]) into TMEM columns [256, 320) as packed bf16 pairs.
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
        mbar_expect_tx(&bar[0], 2 * kTile);
        tma_load_2d(sA, &tmA, &bar[0], 0, 0);
        tma_load_2d(sA + kBox, &tmA, &bar[0], 64, 0);
        tma_load_2d(sB, &tmB, &bar[0], 0, 0);
        tma_load_2d(sB + kBox, &tmB, &bar[0], 64, 0);
        mbar_wait(&bar[0], 0);
        mbar_wait(&bar[2], 0);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA), b_addr = smem_u32(sB);
        constexpr uint32_t idesc_ss = idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t idesc_ts = idesc_bf16_f32(128, 128, 0, 1);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
            umma_ss(tbase, sdesc_sw128(a_addr + off, 16, 1024), sdesc_sw128(b_addr + off, 16, 1024),
                    idesc_ss, kk > 0);
        }
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
            umma_ts(tbase + 128, tbase + 256 + kk * 8, sdesc_sw128(b_addr + kk * 2048, kBox, 1024),
                    idesc_ts, kk > 0);
        }
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
        for (int e = 0; e < 32; ++e) Css[rr * 128 + c * 32 + e] = __uint_as_float(v[e]);
        tmem_ld32(tbase + lane_off + 128 + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) Cts[rr * 128 + c * 32 + e] = __uint_as_float(v[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

}  // namespace

cudaError_t launch_debug_umma(const void* A, const void* B, float* C_ss, float* C_ts,
                              cudaStream_t st) {
    CUtensorMap ma, mb;
    if (!make_map_bf16_sw128(&ma, A, 128, 128, 128) || !make_map_bf16_sw128(&mb, B, 128, 128, 128))
        return cudaErrorInvalidValue;
    const size_t sm = 1024 + 2 * kTile + 64;
    cudaError_t e = cudaFuncSetAttribute(debug_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    debug_umma_kernel<<<1, 128, sm, st>>>(ma, mb, static_cast<const __nv_bfloat16*>(A), C_ss, C_ts);
    return cudaGetLastError();
}

}  // namespace pa
