// attn_tc.cu — bf16 block-sparse causal prefill attention on tcgen05 (A7, and A8 = dense).
//
// Method: O[h][t] = sum over keys k of the selected blocks, k <= t, of
// softmax(Q[h][t] K[kv(h)][k] / sqrt(d)) V[kv(h)][k],
// FlashAttention-style online softmax, causal mask only inside the diagonal block.
//
// One CTA per (local head, query block row m); CTAs are ordered longest row first.
// Warp roles (192 threads):
//   warp 0      TMA producer: Q tile once, then K/V tiles of each selected block into a
//               2-stage ring (128 x 128 bf16 tiles, two SWIZZLE_128B boxes each)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//               S_j = Q K_j^T (SS, K-major both)        -> TMEM S[j%2]  (128 cols fp32)
//               O  += P_j V_j (A = P_j from TMEM, B = V_j MN-major) -> TMEM O (128 cols)
//   warps 2-5   softmax: thread = query row (TMEM lane); tcgen05.ld S_j, scale, diagonal
//               mask, online max with lazy rescale (threshold 2^8), exp2, P_j packed to
//               bf16 and tcgen05.st over S_j's first 64 columns; O correction in TMEM when
//               the running max moved; epilogue O / l -> bf16 -> global.
// TMEM: S0 [0,128) S1 [128,256) O [256,384) of a 512-column allocation.
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace pa {
namespace {

constexpr int kTileRows = 128;                   // b = 128 query rows / keys per tile
constexpr int kBox = kTileRows * 64 * 2;         // 16 KB: [128 rows][64 bf16] SW128 box
constexpr int kTile = 2 * kBox;                  // 32 KB: a 128 x 128 bf16 tile
constexpr int kStages = 2;
constexpr int kThreads = 192;
constexpr float kRescaleThreshold = 8.0f;        // log2 units: P <= 2^8 before a rescale

struct __align__(8) Bars {
    uint64_t q_full;
    uint64_t k_full[kStages];
    uint64_t v_full[kStages];
    uint64_t kv_empty[kStages];
    uint64_t s_full[2];
    uint64_t p_full;
    uint64_t o_done;
    uint32_t tmem_base;
};

constexpr size_t kSmemBytes = 1024 /*align slack*/ + kTile * (1 + 2 * kStages) + sizeof(Bars);

__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
               const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O,
               const int* __restrict__ block_cnt, const int* __restrict__ block_idx, int N, int M,
               int Hl, int r, float scale_log2) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTile;                   // kStages tiles
    uint8_t* sV = smem + kTile * (1 + kStages);   // kStages tiles
    Bars* bars = reinterpret_cast<Bars*>(smem + kTile * (1 + 2 * kStages));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int bid = blockIdx.x;
    const int m = M - 1 - bid / Hl;               // longest rows first (LPT order)
    const int hl = bid % Hl;
    const int kvl = hl / r;
    const bool dense = (block_cnt == nullptr);
    const long long row = static_cast<long long>(hl) * M + m;
    const int cnt = dense ? (m + 1) : block_cnt[row];
    const int* list = dense ? nullptr : block_idx + row * M;

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->kv_empty[s], 1);
        }
        mbar_init(&bars->s_full[0], 1);
        mbar_init(&bars->s_full[1], 1);
        mbar_init(&bars->p_full, 128);
        mbar_init(&bars->o_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ producer --
        if (lane == 0) {
            tma_prefetch(&tmQ);
            tma_prefetch(&tmK);
            tma_prefetch(&tmV);
            const int qrow = hl * N + m * kTileRows;
            mbar_expect_tx(&bars->q_full, kTile);
            tma_load_2d(sQ, &tmQ, &bars->q_full, 0, qrow);
            tma_load_2d(sQ + kBox, &tmQ, &bars->q_full, 64, qrow);
            for (int j = 0; j < cnt; ++j) {
                const int s = j % kStages;
                if (j >= kStages) mbar_wait(&bars->kv_empty[s], ((j / kStages) - 1) & 1);
                const int n = dense ? j : __ldg(list + j);
                const int krow = kvl * N + n * kTileRows;
                uint8_t* k_dst = sK + s * kTile;
                uint8_t* v_dst = sV + s * kTile;
                mbar_expect_tx(&bars->k_full[s], kTile);
                tma_load_2d(k_dst, &tmK, &bars->k_full[s], 0, krow);
                tma_load_2d(k_dst + kBox, &tmK, &bars->k_full[s], 64, krow);
                mbar_expect_tx(&bars->v_full[s], kTile);
                tma_load_2d(v_dst, &tmV, &bars->v_full[s], 0, krow);
                tma_load_2d(v_dst + kBox, &tmV, &bars->v_full[s], 64, krow);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer --
        if (lane == 0) {
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
            const uint32_t tO = tbase + 256;
            const uint32_t q_addr = smem_u32(sQ);
            const uint32_t k_addr = smem_u32(sK);
            const uint32_t v_addr = smem_u32(sV);
            mbar_wait(&bars->q_full, 0);
            auto issue_s = [&](int j) {
                const int s = j % kStages;
                mbar_wait(&bars->k_full[s], (j / kStages) & 1);
                tc_fence_after();
                const uint32_t tS = tbase + (j & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {  // K = d = 128 in steps of 16
                    const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                    const uint64_t a = sdesc_sw128(q_addr + off, 16, 1024);
                    const uint64_t b = sdesc_sw128(k_addr + s * kTile + off, 16, 1024);
                    umma_ss(tS, a, b, idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit(&bars->s_full[j & 1]);
            };
            issue_s(0);
            for (int j = 0; j < cnt; ++j) {
                if (j + 1 < cnt) issue_s(j + 1);
                const int s = j % kStages;
                mbar_wait(&bars->p_full, j & 1);
                mbar_wait(&bars->v_full[s], (j / kStages) & 1);
                tc_fence_after();
                const uint32_t tP = tbase + (j & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {  // K = 128 keys in steps of 16
                    const uint64_t b = sdesc_sw128(v_addr + s * kTile + kk * 2048, kBox, 1024);
                    umma_ts(tO, tP + kk * 8, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
                }
                tc_commit(&bars->kv_empty[s]);
                tc_commit(&bars->o_done);
            }
        }
    } else {
        // ------------------------------------------------------------- softmax --
        const int quarter = warp & 3;                   // TMEM lane quarter of this warp
        const int rr = quarter * 32 + lane;             // query row within the block
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        float m_used = -INFINITY;                       // running max (log2 units)
        float l = 0.f;                                  // running denominator
        for (int j = 0; j < cnt; ++j) {
            const int n = dense ? j : __ldg(list + j);
            mbar_wait(&bars->s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            const uint32_t tS = tbase + lane_off + (j & 1) * 128;
            uint32_t raw[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, raw[c]);
            tmem_ld_wait();
            float x[128];
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e) x[c * 32 + e] = __uint_as_float(raw[c][e]) * scale_log2;
            if (n == m) {  // diagonal block: key index > row index is masked (causal)
#pragma unroll
                for (int e = 0; e < 128; ++e)
                    if (e > rr) x[e] = -INFINITY;
            }
            float rmax = x[0];
#pragma unroll
            for (int e = 1; e < 128; ++e) rmax = fmaxf(rmax, x[e]);
            const float m_new = fmaxf(m_used, rmax);
            const bool need = (m_new > m_used + kRescaleThreshold);
            const bool any = __any_sync(0xffffffffu, need);
            float factor = 1.f;
            if (any) {
                factor = ex2(m_used - m_new);  // 0 on the first block (m_used = -inf)
                m_used = m_new;
                l *= factor;
            }
            uint32_t pk[2][32];
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const float p0 = ex2(x[2 * c] - m_used);
                const float p1 = ex2(x[2 * c + 1] - m_used);
                l += p0 + p1;
                pk[c >> 5][c & 31] = pack_bf16(p0, p1);
            }
            tmem_st32(tS, pk[0]);
            tmem_st32(tS + 32, pk[1]);
            if (j > 0) {
                mbar_wait(&bars->o_done, (j - 1) & 1);  // PV_{j-1} finished writing O
                tc_fence_after();
                if (any) {
                    const uint32_t tO = tbase + lane_off + 256;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + c * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            o[e] = __float_as_uint(__uint_as_float(o[e]) * factor);
                        tmem_st32(tO + c * 32, o);
                    }
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&bars->p_full);
        }
        // ----------------------------------------------------------- epilogue --
        mbar_wait(&bars->o_done, (cnt - 1) & 1);
        tc_fence_after();
        const float inv = 1.f / l;
        const uint32_t tO = tbase + lane_off + 256;
        uint4* dst = reinterpret_cast<uint4*>(
            O + (static_cast<long long>(hl) * N + static_cast<long long>(m) * kTileRows + rr) * 128);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + c * 32, o);
            tmem_ld_wait();
            uint32_t pkd[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                pkd[e] = pack_bf16(__uint_as_float(o[2 * e]) * inv, __uint_as_float(o[2 * e + 1]) * inv);
#pragma unroll
            for (int v = 0; v < 4; ++v)
                dst[c * 4 + v] = make_uint4(pkd[4 * v], pkd[4 * v + 1], pkd[4 * v + 2], pkd[4 * v + 3]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

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

cudaError_t launch_attn_tc(const Dims& D, const void* Q, const void* K, const void* V,
                           const int* block_cnt, const int* block_idx, void* O, cudaStream_t st) {
    CUtensorMap mq, mk, mv;
    if (!make_map_bf16_sw128(&mq, Q, static_cast<uint64_t>(D.Hl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mk, K, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mv, V, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128))
        return cudaErrorInvalidValue;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D.d));
    const unsigned grid = static_cast<unsigned>(D.Hl) * static_cast<unsigned>(D.M);
    attn_tc_kernel<<<grid, kThreads, kSmemBytes, st>>>(
        mq, mk, mv, static_cast<__nv_bfloat16*>(O), block_cnt, block_idx, static_cast<int>(D.N),
        D.M, D.Hl, D.r, scale_log2);
    return cudaGetLastError();
}

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
