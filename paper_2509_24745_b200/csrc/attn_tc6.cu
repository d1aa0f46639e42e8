// attn_tc6.cu — bf16 block-sparse causal prefill attention on tcgen05 (A7 / A8), variant v6:
// one (head, query block row) per CTA with its key blocks split into TWO INDEPENDENT STREAMS
// (even / odd positions of the row's ascending list).  Each stream owns an S buffer, an O
// accumulator and its own online-softmax state (running max, denominator), so the two
// S -> softmax -> PV chains overlap on the tensor core without the union-walk coupling of
// two query rows (attn_tc.cu): every iteration carries a full tile for its stream.  The
// epilogue merges the streams: O = (O_0 2^(m_0-m) + O_1 2^(m_1-m)) / (l_0 2^(m_0-m) + l_1 2^(m_1-m)).
//
// Method: O[h][t] = sum over keys k of the selected blocks, k <= t, of
// softmax(Q[h][t] K[kv(h)][k] / sqrt(d)) V[kv(h)][k]; causal
// mask only in the diagonal block (it also masks the padded keys of a ragged last block).
//
// Warp roles (320 threads):
//   warp 0      TMA producer: the Q tile, then K tiles (3-stage ring, two blocks ahead) and
//               V tiles (2-stage ring) in list order
//   warp 1      TMEM allocator + tcgen05.mma issuer, run warp-uniformly (descriptors in
//               uniform registers, MMA / commit under elect.sync): for block j of stream
//               s = j & 1: wait P_j -> O_s += P_j V_j -> S_s = Q K_{j+2}^T
//   warps 2-5   softmax of stream 0, warps 6-9 of stream 1 (thread = query row = TMEM lane):
//               tcgen05.ld S, mask, 8-chain max, lazy rescale (2^8), exp2, P (bf16) stored
//               over S's first 64 columns in two halves released separately to the PV MMA.
// TMEM (512 columns): S_0 [0,128) S_1 [128,256) O_0 [256,384) O_1 [384,512).
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
constexpr int kKStages = 3;
constexpr int kVStages = 2;
constexpr int kThreads = 320;
constexpr float kRescaleThreshold = 8.0f;

struct __align__(8) Bars6 {
    uint64_t q_full;
    uint64_t k_full[kKStages];
    uint64_t k_empty[kKStages];
    uint64_t v_full[kVStages];
    uint64_t v_empty[kVStages];
    uint64_t s_full[2];
    uint64_t p_half[2][2];   // [stream][half]
    uint64_t o_done[2];
    uint32_t tmem_base;
    float red_m[128];        // stream 1's final (max, denominator) per row, for the merge
    float red_l[128];
};

constexpr size_t kSmemBytes = 1024 + kTile * (1 + kKStages + kVStages) + sizeof(Bars6);

template <int kEmu>   // of every 8 key-column pairs, kEmu use the FMA-pipe exp2 (ex2_poly2)
__global__ void __launch_bounds__(kThreads, 1)
attn_tc6_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O,
                const int* __restrict__ block_cnt, const int* __restrict__ block_idx, int N, int M,
                int r, float scale_log2, int row_lo, int row_hi, long long* trace, int trace_bid) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTile;
    uint8_t* sV = smem + kTile * (1 + kKStages);
    Bars6* bars = reinterpret_cast<Bars6*>(smem + kTile * (1 + kKStages + kVStages));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // work item: kv-head major, heaviest rows first within a kv head
    const int nrows = row_hi - row_lo;
    const int per_kv = r * nrows;
    const int kvl = blockIdx.x / per_kv, rem = blockIdx.x % per_kv;
    const int m = row_hi - 1 - rem / r;
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
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->p_half[s][0], 128);
            mbar_init(&bars->p_half[s][1], 128);
            mbar_init(&bars->o_done[s], 1);
        }
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
            if (cnt > 0) load_k(0);
            if (cnt > 1) load_k(1);
            for (int j = 0; j < cnt; ++j) {
                if (j + 2 < cnt) load_k(j + 2);
                load_v(j);
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------- MMA issuer --
        constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
        const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
        const uint64_t dv = sdesc_sw128(smem_u32(sV), kBox, 1024);
        const bool leader = elect_one();
        mbar_wait(&bars->q_full, 0);
        auto issue_s = [&](int j) {   // S_{j&1} = Q K_j^T
            const int st = j % kKStages;
            mbar_wait(&bars->k_full[st], (j / kKStages) & 1);
            tc_fence_after();
            if (leader) {
                const uint64_t b0 = dk + (st * kTile >> 4);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
                    umma_ss(tbase + (j & 1) * 128, dq + off, b0 + off, idesc_qk, kk > 0 ? 1u : 0u);
                }
                tc_commit(&bars->k_empty[st]);
                tc_commit(&bars->s_full[j & 1]);
            }
            __syncwarp();
        };
        if (cnt > 0) issue_s(0);
        if (cnt > 1) issue_s(1);
        for (int j = 0; j < cnt; ++j) {
            const int s = j & 1;
            const int js = j >> 1;                        // position within the stream
            const int st = j % kVStages;
            const uint32_t tP = tbase + s * 128;
            const uint32_t tO = tbase + 256 + s * 128;
            long long* tr = (trace && blockIdx.x == trace_bid && j < 512 && leader) ? trace + j * 8 : nullptr;
            if (tr) tr[0] = clock64();                             // MMA: start waiting for V, P
            mbar_wait(&bars->v_full[st], (j / kVStages) & 1);
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                mbar_wait(&bars->p_half[s][half], js & 1);
                if (tr) tr[1 + half] = clock64();                  // MMA: P half ready
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = dv + (st * kTile >> 4);
#pragma unroll
                    for (int k4 = 0; k4 < 4; ++k4) {
                        const int kk = half * 4 + k4;
                        umma_ts(tO, tP + kk * 8, b0 + (kk * 2048 >> 4), idesc_pv,
                                (js > 0 || kk > 0) ? 1u : 0u);
                    }
                }
                __syncwarp();
            }
            if (leader) {
                tc_commit(&bars->v_empty[st]);
                tc_commit(&bars->o_done[s]);
            }
            __syncwarp();
            if (j + 2 < cnt) issue_s(j + 2);   // overwrites S_s = P_j after PV_j (in order)
            if (tr) tr[3] = clock64();                             // MMA: PV + next S issued
        }
    } else {
        // ------------------------------------------------------------- softmax --
        const int s = (warp - 2) >> 2;                  // stream
        const int quarter = warp & 3;
        const int rr = quarter * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + s * 128;
        const uint32_t tO = tbase + lane_off + 256 + s * 128;
        const int my_cnt = (cnt - s + 1) >> 1;         // blocks j = s, s + 2, ...
        float m_used = -INFINITY;                       // running max (log2 units)
        float l = 0.f;
        int n_next = (my_cnt > 0) ? (list ? __ldg(list + s) : s) : 0;
        for (int js = 0; js < my_cnt; ++js) {
            const int j = 2 * js + s;
            const int n = n_next;
            if (js + 1 < my_cnt) n_next = list ? __ldg(list + j + 2) : j + 2;
            long long* tr = (trace && blockIdx.x == trace_bid && lane == 0 && quarter == 2 && js < 256)
                                ? trace + 512 * 8 + (js * 2 + s) * 8 : nullptr;
            if (tr) tr[0] = clock64();                             // SM: start waiting for S
            mbar_wait(&bars->s_full[s], js & 1);
            if (tr) tr[1] = clock64();                             // SM: S ready
            tc_fence_after();
            uint32_t raw[4][32];
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, raw[c]);
            tmem_ld_wait();
            if (n == m) {  // diagonal block: causal mask (also masks padded keys)
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        if (c * 32 + e > rr) raw[c][e] = 0xff800000u;
            }
            float mx[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) mx[k] = __uint_as_float(raw[k >> 1][(k & 1) * 16]);
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    mx[c * 2 + (e >> 4)] = fmaxf(mx[c * 2 + (e >> 4)], __uint_as_float(raw[c][e]));
            const float rmax = fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                     fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
            const float m_new = fmaxf(m_used, rmax * scale_log2);
            const bool need = (m_new > m_used + kRescaleThreshold);
            const bool any = __any_sync(0xffffffffu, need);
            float factor = 1.f;
            if (any) {
                factor = ex2(m_used - m_new);
                m_used = m_new;
                l *= factor;
            }
            if (tr) tr[2] = clock64();                             // SM: S loaded + row max
            const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
            const uint64_t nm2 = f2_pack(-m_used, -m_used);
            uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                uint32_t pk[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    const int e0 = half * 64 + 2 * c;
                    const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(raw[e0 >> 5][e0 & 31]),
                                                       __uint_as_float(raw[e0 >> 5][(e0 & 31) + 1])),
                                               sc2, nm2);
                    float p0, p1;
                    if ((c & 7) < kEmu) {
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
                if (tr) tr[5 + half] = clock64();                  // SM: exps of this half done
                tmem_st32(tS + half * 32, pk);
                if (half == 0 && js > 0) {
                    mbar_wait(&bars->o_done[s], (js - 1) & 1);   // PV of the stream's previous block
                    if (tr) tr[7] = clock64();                     // SM: O ready for correction
                    tc_fence_after();
                    if (any) {
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
                mbar_arrive(&bars->p_half[s][half]);
                if (tr) tr[3 + half] = clock64();                  // SM: P half released
            }
            {
                const uint64_t t = f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3]));
                float a, b;
                f2_unpack(t, a, b);
                l += a + b;
            }
        }
        // ------------------------------------------------- merge + epilogue --
        if (s == 1) {
            bars->red_m[rr] = m_used;
            bars->red_l[rr] = l;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");       // the 8 softmax warps
        if (s == 0) {
            const float m1 = bars->red_m[rr], l1 = bars->red_l[rr];
            const float mm = fmaxf(m_used, m1);
            const float f0 = (my_cnt > 0) ? ex2(m_used - mm) : 0.f;
            const float f1 = (cnt > 1) ? ex2(m1 - mm) : 0.f;
            const float inv = 1.f / (l * f0 + l1 * f1);
            const float w0 = f0 * inv, w1 = f1 * inv;
            if (my_cnt > 0) {
                mbar_wait(&bars->o_done[0], (my_cnt - 1) & 1);
                if (cnt > 1) mbar_wait(&bars->o_done[1], (((cnt >> 1)) - 1) & 1);
            }
            tc_fence_after();
            const bool row_valid = static_cast<long long>(m) * kTileRows + rr < N;
            uint4* dst = reinterpret_cast<uint4*>(
                O + (static_cast<long long>(hl) * N + static_cast<long long>(m) * kTileRows + rr) * 128);
            const uint32_t tO1 = tbase + lane_off + 384;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t o0[32], o1[32];
                tmem_ld32(tO + c * 32, o0);
                tmem_ld32(tO1 + c * 32, o1);
                tmem_ld_wait();
                uint32_t pkd[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const float a = __uint_as_float(o0[2 * e]) * w0 + (cnt > 1 ? __uint_as_float(o1[2 * e]) * w1 : 0.f);
                    const float b = __uint_as_float(o0[2 * e + 1]) * w0 +
                                    (cnt > 1 ? __uint_as_float(o1[2 * e + 1]) * w1 : 0.f);
                    pkd[e] = pack_bf16(a, b);
                }
                if (row_valid) {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        dst[c * 4 + v] = make_uint4(pkd[4 * v], pkd[4 * v + 1], pkd[4 * v + 2], pkd[4 * v + 3]);
                }
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

}  // namespace

cudaError_t launch_attn_tc6(const Dims& D, const void* Q, const void* K, const void* V,
                            const int* block_cnt, const int* block_idx, void* O, cudaStream_t st) {
    CUtensorMap mq, mk, mv;
    if (!make_map_bf16_sw128(&mq, Q, static_cast<uint64_t>(D.Hl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mk, K, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128) ||
        !make_map_bf16_sw128(&mv, V, static_cast<uint64_t>(D.Hkvl) * D.N, 128, 128))
        return cudaErrorInvalidValue;
    static int emu = -1;
    if (emu < 0) {   // PROXYATTN_EXP_EMU=0..4: x/8 of the exponentials on the FMA pipe
        const char* e = getenv("PROXYATTN_EXP_EMU");
        emu = (e && e[0] >= '0' && e[0] <= '4') ? e[0] - '0' : 2;
    }
    auto kern = emu == 0 ? attn_tc6_kernel<0> : emu == 1 ? attn_tc6_kernel<1>
              : emu == 2 ? attn_tc6_kernel<2> : emu == 3 ? attn_tc6_kernel<3> : attn_tc6_kernel<4>;
    static bool attr_set[5] = {false, false, false, false, false};
    if (!attr_set[emu]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set[emu] = true;
    }
    // PROXYATTN_TRACE=<cta>: per-event clock64 timeline of one CTA (diagnostics only), read
    // back with proxyattn_debug_trace(): [512 j][8] MMA events, then [256 js][2 s][8] softmax.
    constexpr size_t kTraceBytes = 2 * 512 * 8 * sizeof(long long);
    static long long* trace = nullptr;
    static int trace_bid = -1;
    if (trace_bid < 0) {
        const char* e = getenv("PROXYATTN_TRACE");
        trace_bid = e ? atoi(e) : 1 << 30;
        if (e && cudaMalloc(&trace, kTraceBytes) != cudaSuccess) trace = nullptr;
    }
    if (trace) cudaMemsetAsync(trace, 0, kTraceBytes, st);
    attn_trace_ptr() = trace;
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D.d));
    const unsigned grid = static_cast<unsigned>(D.Hl) * static_cast<unsigned>(D.re - D.rb);
    kern<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, static_cast<__nv_bfloat16*>(O),
                                                        block_cnt, block_idx, static_cast<int>(D.N),
                                                        D.M, D.r, scale_log2, D.rb, D.re, trace, trace_bid);
    return cudaGetLastError();
}

}  // namespace pa
