// attn_tc4.cu — bf16 block-sparse causal prefill attention on tcgen05 (A7 / A8), variant
// with double-buffered S and column-split softmax.
//
// Method: O[h][t] = sum over keys k of the selected blocks, k <= t, of
// softmax(Q[h][t] K[kv(h)][k] / sqrt(d)) V[kv(h)][k],
// FlashAttention-style online softmax, causal mask only inside the diagonal block.
//
// One CTA = one (local head, query block row m), 128 query rows; CTAs ordered kv-head
// major (L2 reuse of the kv head's K/V across the resident CTAs), heaviest rows first.
// Warp roles (320 threads):
//   warp 0      TMA producer: Q tile, then K (3-stage ring, two blocks ahead) and V (2-stage)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//               S_{j+2} = Q K_{j+2}^T is issued right after O += P_j V_j, so the tensor core
//               computes the next S while the softmax works on the current one
//   warps 2-9   softmax: warp (2 + 4c + q) owns TMEM lanes [32q, 32q+32) (query rows) and
//               key columns [64c, 64c+64); the two column halves of a row exchange their
//               partial max through shared memory (64-thread named barrier); each half
//               writes its P (bf16) into its own 32 TMEM columns and releases it to the
//               MMA separately; O correction (lazy, 2^8 threshold) and the epilogue are
//               split by the same column halves.
// TMEM (512 columns allocated): S_0 [0,128), S_1 [128,256), O [256,384).
//   P_j (half c) lives in S_{j&1} columns [64c, 64c+32) (inside the half's own S columns).
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace pa {
namespace {

constexpr int kTileRows = 128;
constexpr int kBox = kTileRows * 64 * 2;   // 16 KB: [128 rows][64 bf16] SW128 box
constexpr int kTile = 2 * kBox;            // 32 KB: a 128 x 128 bf16 tile
constexpr int kKStages = 3;   // K ring runs ahead: S is issued two blocks ahead of PV
constexpr int kVStages = 2;
constexpr int kThreads = 320;
constexpr float kRescaleThreshold = 8.0f;

struct __align__(8) Bars4 {
    uint64_t q_full;
    uint64_t k_full[kKStages];
    uint64_t k_empty[kKStages];
    uint64_t v_full[kVStages];
    uint64_t v_empty[kVStages];
    uint64_t s_full[2];
    uint64_t p_half[2];      // [column half]: P_j for keys [64c, 64c + 64) written
    uint64_t o_done;
    uint32_t tmem_base;
    float red[3][2][128];    // [j & 1 | 2 for l][column half][row]: partial max / sum exchange
};

constexpr size_t kSmemBytes = 1024 + kTile * (1 + kKStages + kVStages) + sizeof(Bars4);

__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <int kEmu>   // of every 4 column pairs, kEmu use the FMA-pipe exp2 (ex2_poly2)
__global__ void __launch_bounds__(kThreads, 1)
attn_tc4_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O,
                const int* __restrict__ block_cnt, const int* __restrict__ block_idx, int N, int M,
                int r, float scale_log2, long long* trace, int trace_bid) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTile;
    uint8_t* sV = smem + kTile * (1 + kKStages);
    Bars4* bars = reinterpret_cast<Bars4*>(smem + kTile * (1 + kKStages + kVStages));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int bid = blockIdx.x;
    const int per_kv = r * M;
    const int kvl = bid / per_kv, rem = bid % per_kv;
    const int m = M - 1 - rem / r;
    const int hl = kvl * r + rem % r;
    const bool dense = (block_cnt == nullptr);
    const long long row = static_cast<long long>(hl) * M + m;
    const int cnt = dense ? m + 1 : block_cnt[row];
    const int* list = dense ? nullptr : block_idx + row * M;

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        mbar_init(&bars->s_full[0], 1);
        mbar_init(&bars->s_full[1], 1);
        mbar_init(&bars->p_half[0], 128);
        mbar_init(&bars->p_half[1], 128);
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
            auto load_k = [&](int j) {
                const int st = j % kKStages;
                if (j >= kKStages) mbar_wait(&bars->k_empty[st], ((j / kKStages) - 1) & 1);
                const int n = dense ? j : __ldg(list + j);
                const int krow = kvl * N + n * kTileRows;
                mbar_expect_tx(&bars->k_full[st], kTile);
                tma_load_2d(sK + st * kTile, &tmK, &bars->k_full[st], 0, krow);
                tma_load_2d(sK + st * kTile + kBox, &tmK, &bars->k_full[st], 64, krow);
            };
            auto load_v = [&](int j) {
                const int st = j % kVStages;
                if (j >= kVStages) mbar_wait(&bars->v_empty[st], ((j / kVStages) - 1) & 1);
                const int n = dense ? j : __ldg(list + j);
                const int vrow = kvl * N + n * kTileRows;
                mbar_expect_tx(&bars->v_full[st], kTile);
                tma_load_2d(sV + st * kTile, &tmV, &bars->v_full[st], 0, vrow);
                tma_load_2d(sV + st * kTile + kBox, &tmV, &bars->v_full[st], 64, vrow);
            };
            // K runs up to two blocks ahead of V (S_{j+2} is issued right after PV_j).
            if (cnt > 0) load_k(0);
            if (cnt > 1) load_k(1);
            for (int j = 0; j < cnt; ++j) {
                load_v(j);
                if (j + 2 < cnt) load_k(j + 2);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer --
        if (lane == 0) {
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
            const uint32_t q_addr = smem_u32(sQ);
            const uint32_t k_addr = smem_u32(sK);
            const uint32_t v_addr = smem_u32(sV);
            const uint32_t tO = tbase + 256;
            mbar_wait(&bars->q_full, 0);
            auto issue_s = [&](int j) {
                const int st = j % kKStages;
                mbar_wait(&bars->k_full[st], (j / kKStages) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                    umma_ss(tbase + (j & 1) * 128, sdesc_sw128(q_addr + off, 16, 1024),
                            sdesc_sw128(k_addr + st * kTile + off, 16, 1024), idesc_qk,
                            kk > 0 ? 1u : 0u);
                }
                tc_commit(&bars->k_empty[st]);
                tc_commit(&bars->s_full[j & 1]);
            };
            issue_s(0);
            if (cnt > 1) issue_s(1);
            for (int j = 0; j < cnt; ++j) {
                const int st = j % kVStages;
                const uint32_t tP = tbase + (j & 1) * 128;
                mbar_wait(&bars->v_full[st], (j / kVStages) & 1);
#pragma unroll
                long long* tr = (trace && blockIdx.x == trace_bid && j < 256) ? trace + (j * 2) * 8 : nullptr;
                if (tr) tr[0] = clock64();
                for (int c = 0; c < 2; ++c) {   // keys [64c, 64c + 64): P at S cols [64c, 64c+32)
                    mbar_wait(&bars->p_half[c], j & 1);
                    if (tr) tr[1 + c] = clock64();
                    tc_fence_after();
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4) {
                        const int kk = c * 4 + k4;
                        const uint64_t b = sdesc_sw128(v_addr + st * kTile + kk * 2048, kBox, 1024);
                        umma_ts(tO, tP + c * 64 + k4 * 8, b, idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                tc_commit(&bars->v_empty[st]);
                tc_commit(&bars->o_done);
                if (j + 2 < cnt) issue_s(j + 2);   // overwrites S_{j&1} = P_j: after PV_j (in order)
                if (tr) tr[3] = clock64();
            }
        }
    } else {
        // ------------------------------------------------------------- softmax --
        const int q4 = warp & 3;                        // TMEM lane quarter
        const int ch = (warp - 2) >> 2;                 // column half
        const int rr = q4 * 32 + lane;                  // query row within the block
        const uint32_t lane_off = static_cast<uint32_t>(q4 * 32) << 16;
        const uint32_t tO = tbase + lane_off + 256 + ch * 64;
        float m_used = -INFINITY;                       // running max (log2 units)
        float l = 0.f;                                  // partial denominator (own columns)
        int n_next = cnt > 0 ? (list ? __ldg(list) : 0) : 0;
        for (int j = 0; j < cnt; ++j) {
            const int n = n_next;
            if (j + 1 < cnt) n_next = list ? __ldg(list + j + 1) : j + 1;
            long long* tr = (trace && blockIdx.x == trace_bid && lane == 0 && q4 == 2 && j < 256)
                                ? trace + 256 * 16 + (j * 2 + ch) * 8 : nullptr;
            if (tr) tr[0] = clock64();
            mbar_wait(&bars->s_full[j & 1], (j >> 1) & 1);
            tc_fence_after();
            if (tr) tr[1] = clock64();
            const uint32_t tS = tbase + lane_off + (j & 1) * 128 + ch * 64;
            uint32_t raw[2][32];
            tmem_ld32(tS, raw[0]);
            tmem_ld32(tS + 32, raw[1]);
            tmem_ld_wait();
            if (n == m) {  // diagonal block: key index > row index is masked (causal)
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (ch * 64 + c * 32 + e > rr) raw[c][e] = 0xff800000u;
            }
            float mx[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) mx[k] = __uint_as_float(raw[k >> 1][(k & 1) * 16]);
#pragma unroll
            for (int c = 0; c < 2; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    mx[c * 2 + (e >> 4)] = fmaxf(mx[c * 2 + (e >> 4)], __uint_as_float(raw[c][e]));
            const float pmax = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
            // exchange the partial max with the other column half of the same rows
            if (tr) tr[2] = clock64();
            bars->red[j & 1][ch][rr] = pmax;
            named_bar(1 + q4, 64);
            if (tr) tr[3] = clock64();
            const float rmax = fmaxf(pmax, bars->red[j & 1][ch ^ 1][rr]);
            const float m_new = fmaxf(m_used, rmax * scale_log2);
            const bool need = (m_new > m_used + kRescaleThreshold);
            const bool any = __any_sync(0xffffffffu, need);   // same rows in both halves
            float factor = 1.f;
            if (any) {
                factor = ex2(m_used - m_new);
                m_used = m_new;
                l *= factor;
            }
            const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
            const uint64_t nm2 = f2_pack(-m_used, -m_used);
            uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const int e0 = 2 * c;
                const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(raw[e0 >> 5][e0 & 31]),
                                                   __uint_as_float(raw[e0 >> 5][(e0 & 31) + 1])),
                                           sc2, nm2);
                float p0, p1;
                if ((c & 3) < kEmu) {
                    ex2_poly2(x2, p0, p1);
                } else {
                    float x0, x1;
                    f2_unpack(x2, x0, x1);
                    p0 = ex2(x0);
                    p1 = ex2(x1);
                }
                ls[c & 3] = f2_add(ls[c & 3], f2_pack(p0, p1));
                pk[c] = pack_bf16(p0, p1);
            }
            if (tr) tr[4] = clock64();
            tmem_st32(tS, pk);                           // P for this half's 64 keys
            {
                const uint64_t t = f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3]));
                float a, b;
                f2_unpack(t, a, b);
                l += a + b;
            }
            if (j > 0) {
                mbar_wait(&bars->o_done, (j - 1) & 1);   // PV_{j-1} finished writing O
                tc_fence_after();
                if (any) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
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
            mbar_arrive(&bars->p_half[ch]);
            if (tr) tr[5] = clock64();
        }
        // ----------------------------------------------------------- epilogue --
        if (cnt > 0) {
            bars->red[2][ch][rr] = l;
            named_bar(1 + q4, 64);
            const float inv = 1.f / (l + bars->red[2][ch ^ 1][rr]);
            mbar_wait(&bars->o_done, (cnt - 1) & 1);
            tc_fence_after();
            uint4* dst = reinterpret_cast<uint4*>(
                O + (static_cast<long long>(hl) * N + static_cast<long long>(m) * kTileRows + rr) * 128 +
                ch * 64);
#pragma unroll
            for (int c = 0; c < 2; ++c) {
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
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tbase, 512);
    }
}

int attn4_exp_emu() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("PROXYATTN_EXP_EMU");
        v = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : 0;
    }
    return v;
}

}  // namespace

cudaError_t launch_attn_tc4(const Dims& D, const void* Q, const void* K, const void* V,
                            const int* block_cnt, const int* block_idx, void* O, cudaStream_t st) {
    CUtensorMap mq, mk, mv;
    if (!make_map_bf16_sw128(&mq, Q, static_cast<uint64_t>(D.Hl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mk, K, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mv, V, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128))
        return cudaErrorInvalidValue;
    const int emu = attn4_exp_emu();
    auto kern = emu == 0 ? attn_tc4_kernel<0> : emu == 1 ? attn_tc4_kernel<1>
              : emu == 2 ? attn_tc4_kernel<2> : attn_tc4_kernel<3>;
    static bool attr_set[4] = {false, false, false, false};
    if (!attr_set[emu]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set[emu] = true;
    }
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D.d));
    const unsigned grid = static_cast<unsigned>(D.Hl) * static_cast<unsigned>(D.M);
    static long long* trace = nullptr;
    static int trace_bid = -1;
    if (trace_bid < 0) {
        const char* e = getenv("PROXYATTN_TRACE");
        trace_bid = e ? atoi(e) : 1 << 30;
        if (e && cudaMalloc(&trace, 2 * 256 * 2 * 8 * sizeof(long long)) != cudaSuccess) trace = nullptr;
    }
    if (trace) {
        cudaMemsetAsync(trace, 0, 2 * 256 * 2 * 8 * sizeof(long long), st);
        attn_trace_ptr() = trace;
    }
    kern<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, static_cast<__nv_bfloat16*>(O), block_cnt,
                                             block_idx, static_cast<int>(D.N), D.M, D.r, scale_log2,
                                             trace, trace_bid);
    return cudaGetLastError();
}

}  // namespace pa
