// score_tc.cu — tcgen05 score kernels of the estimation (bf16 build, b in {64, 128},
// d in {64, 128}, b/s in {16, 32, 64, 128}):
//
//   A2  proxy_lse     Eq. 1 softmax normaliser of the proxy logits over the sampled causal
//                     keys (Z4): per (sampled row, key chunk) online (max, sum) in
//                     log2 units; the same pass stores each row's window maxima W (the
//                     raw-logit max over the b/s sampled keys of every key block).
//   A3  max-pool      Eq. 1 max-pool (Z6): maxpool_from_windows_kernel combines the
//                     rows' chunk partials into lse and takes L[c][m][n] = max over the block
//                     row's sampled rows of (W - lse), no second GEMM pass.
//   A4  budget        Alg. 1 line 1-2 (Z7, Z8): per head, last block's b queries
//                     against every key block: per (row t, block n) max m_tn and
//                     s_tn = sum_k exp2(x_tk - m_tn); combined + sorted afterwards.  With
//                     b = 64 the A tile's rows 64-127 are padding and each 128-key tile
//                     holds two key blocks (one partial per 64-column half).
//
// Both passes share one warp-specialised tile engine (320 threads, 2 CTAs / SM):
//   warp 0 TMA producer (A tile once, then 128-key B tiles into a 2-stage ring),
//   warp 1 TMEM allocator + single-thread tcgen05.mma issuer (S = A B^T, K = d,
//          SS operands K-major SWIZZLE_128B, fp32 accumulators double-buffered in TMEM),
//   warps 2-5 / 6-9 two epilogue warpgroups, one per S buffer (even / odd tiles): thread =
//          tile row (TMEM lane), the tile read in two 64-column halves, mode math.
#include <cuda_bf16.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace pa {
namespace {

constexpr int kBox = 128 * 64 * 2;   // one [128 rows][64 bf16] SWIZZLE_128B box
constexpr int kTile = 2 * kBox;      // 128 x 128 bf16
constexpr int kStages = 2;
constexpr int kThreads = 320;   // TMA warp, MMA warp, two epilogue warpgroups
constexpr int kChunk = 16;           // default key tiles per CTA (proxy / budget)

enum Mode { kLse = 0, kBudget = 2 };

struct __align__(8) SBars {
    uint64_t a_full;
    uint64_t b_full[kStages];
    uint64_t b_empty[kStages];
    uint64_t s_full[2];
    uint64_t s_empty[2];
    uint32_t tmem_base;
    float red_m[128];       // LSE: the second epilogue warpgroup's (max, sum) per row
    float red_s[128];
};
constexpr size_t kSmem = 1024 + kTile * (1 + kStages) + sizeof(SBars);

struct ScoreParams {
    int mode;
    int Ns;          // proxy: sampled rows per group
    int N, M;        // budget: tokens, blocks
    int n_tr;        // proxy: tile rows per group (Ns / 128)
    int tr_lo, tr_hi;   // proxy: tile rows computed (row-range estimate), [0, n_tr) by default
    int chunk;          // key tiles per CTA
    int n_chunks;    // chunks per tile row (proxy) / per head (budget)
    int r;           // budget: GQA ratio (local head -> local kv head)
    int bs;          // proxy: sampled rows (= keys) per block, b / s
    int d;           // head dim (64 or 128; the kernel's kD)
    int b;           // budget: block size (64 or 128); key tiles hold 128 / b blocks
    int n_kt;        // budget: 128-key tiles
    float sc2;       // logit scale in log2 units
    float* part_m;   // LSE: [gl][Ns][n_chunks]; BUDGET: [Hl][M][128]
    float* part_s;
    float* W;           // LSE (optional): [gl][n_tr][Ns][nwin] raw-logit max of each row over
                        // the bs sampled keys of block n = u * nwin + w of key tile u (causal
                        // mask applied); tile-major so a warp's store of its 32 rows' windows
                        // is one contiguous 32 * nwin * 4-byte segment
};

// kEmu: of every 4 column pairs, kEmu use the FMA-pipe exp2 (degree 4); kB64: budget pass
// with b = 64 (two key blocks per 128-key tile); kD: head dim (K of the MMAs)
template <int kEmu, bool kB64, int kD, int kMode>
__global__ void __launch_bounds__(kThreads, 2)
score_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                ScoreParams p) {
    // ---------------------------------------------------------------- problem --
    int a_row, b_row0, u_begin, u_end, diag_u, prob;  // prob: group (proxy) / local head
    int a_head = 0, b_head = 0;                        // budget: 3-D maps (any Q/K layout)
    int tr = 0;                                        // proxy tile row
    if (kMode == kBudget) {
        prob = blockIdx.x / p.n_chunks;
        const int k = blockIdx.x % p.n_chunks;
        u_begin = k * p.chunk;
        u_end = min(u_begin + p.chunk, p.n_kt);
        a_row = (p.M - 1) * p.b;                   // the last block's query rows (Alg. 1)
        a_head = prob;
        b_row0 = 0;
        b_head = prob / p.r;
        diag_u = p.n_kt - 1;
    } else {
        const int per_group = (p.tr_hi - p.tr_lo) * p.n_chunks;
        prob = blockIdx.x / per_group;
        const int rem = blockIdx.x % per_group;
        tr = p.tr_hi - 1 - rem / p.n_chunks;       // long rows first
        const int k = rem % p.n_chunks;
        u_begin = k * p.chunk;
        if (u_begin > tr) return;                  // chunk beyond the causal diagonal
        u_end = min(u_begin + p.chunk, tr + 1);
        a_row = prob * p.Ns + tr * 128;
        b_row0 = prob * p.Ns;
        diag_u = tr;
    }
    const int nt = u_end - u_begin;

    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base, derived from the __shared__ array by pointer arithmetic so that
    // the compiler keeps the shared state space (LDS/STS, not generic loads, for the barriers
    // and exchange arrays)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kTile;
    SBars* bars = reinterpret_cast<SBars*>(smem + kTile * (1 + kStages));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(&bars->a_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&bars->b_full[s], 1);
            mbar_init(&bars->b_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&bars->s_full[s], 1);
            mbar_init(&bars->s_empty[s], 128);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bars->tmem_base, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            tma_prefetch(&tmA);
            tma_prefetch(&tmB);
            auto load = [&](uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int col, int row, int head) {
                if (kMode == kBudget) tma_load_3d(dst, map, bar, col, row, head);
                else tma_load_2d(dst, map, bar, col, row);
            };
            constexpr int nbox = kD / 64;
            mbar_expect_tx(&bars->a_full, nbox * kBox);
            for (int ch = 0; ch < nbox; ++ch) load(sA + ch * kBox, &tmA, &bars->a_full, ch * 64, a_row, a_head);
            for (int j = 0; j < nt; ++j) {
                const int s = j % kStages;
                if (j >= kStages) mbar_wait(&bars->b_empty[s], ((j / kStages) - 1) & 1);
                const int brow = b_row0 + (u_begin + j) * 128;
                mbar_expect_tx(&bars->b_full[s], nbox * kBox);
                for (int ch = 0; ch < nbox; ++ch)
                    load(sB + s * kTile + ch * kBox, &tmB, &bars->b_full[s], ch * 64, brow, b_head);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
            const uint32_t a_addr = smem_u32(sA), b_addr = smem_u32(sB);
            mbar_wait(&bars->a_full, 0);
            for (int j = 0; j < nt; ++j) {
                const int s = j % kStages;
                mbar_wait(&bars->b_full[s], (j / kStages) & 1);
                if (j >= 2) mbar_wait(&bars->s_empty[j & 1], ((j >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t tS = tbase + (j & 1) * 128;
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
                    umma_ss(tS, sdesc_sw128(a_addr + off, 16, 1024),
                            sdesc_sw128(b_addr + s * kTile + off, 16, 1024), idesc, kk > 0 ? 1u : 0u);
                }
                tc_commit(&bars->b_empty[s]);
                tc_commit(&bars->s_full[j & 1]);
            }
        }
    } else {
        // Two epilogue warpgroups (warps 2-5 and 6-9), one per S buffer: warpgroup e takes the
        // tiles j with j % 2 == e.  A thread is a tile row (TMEM lane); a tile's 128 columns are
        // read in two 64-column halves, which keeps a thread within the register budget of two
        // warpgroups (16 epilogue warps per SM at 2 CTAs) to hide the MUFU / FMNMX latencies.
        const int eg = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int rr = quarter * 32 + lane;                  // tile row
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        float m_run = -INFINITY, s_run = 0.f;                // kLse: online (max, sum), log2 units
        // diagonal tile: key column c is masked when c > rr + diag_off (key position past the
        // query's); 0 except in the b = 64 budget pass, where the last block can sit in the
        // second half of its 128-key tile (diag_off = 64)
        const int diag_off = kB64 && kMode == kBudget ? a_row - diag_u * 128 : 0;
        // rows past the end (partial last tile / block): padded, excluded from every output
        const bool row_ok = (kMode == kBudget) ? (rr < p.b && a_row + rr < p.N) : (tr * 128 + rr < p.Ns);
        const uint64_t sc2 = f2_pack(p.sc2, p.sc2);
        for (int j = eg; j < nt; j += 2) {
            const int u = u_begin + j;
            mbar_wait(&bars->s_full[eg], (j >> 1) & 1);
            tc_fence_after();
            const bool diag = (u == diag_u);
            float h8[8];                                     // 16-column group maxima (raw logits)
            float tm[2], ac[2];                              // budget: per-half max (log2) and sum
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t raw[2][32];
                tmem_ld32(tbase + lane_off + eg * 128 + hf * 64, raw[0]);
                tmem_ld32(tbase + lane_off + eg * 128 + hf * 64 + 32, raw[1]);
                tmem_ld_wait();
                if (hf == 1) {                               // S read out: the next MMA may reuse it
                    tc_fence_before();
                    mbar_arrive(&bars->s_empty[eg]);
                }
                if (diag) {
                    const int thr = rr + diag_off - hf * 64;
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (c * 32 + e > thr) raw[c][e] = 0xff800000u;   // -inf
                }
#pragma unroll
                for (int g = 0; g < 4; ++g) {                // 16-column maxima: 8 FMNMX3 each
                    const uint32_t* v = &raw[g >> 1][(g & 1) * 16];
                    auto f = [&](int e) { return __uint_as_float(v[e]); };
                    const float a0 = fmax3(f(0), f(1), f(2)), a1 = fmax3(f(3), f(4), f(5));
                    const float a2 = fmax3(f(6), f(7), f(8)), a3 = fmax3(f(9), f(10), f(11));
                    const float a4 = fmax3(f(12), f(13), f(14));
                    h8[hf * 4 + g] = fmax3(fmax3(a0, a1, a2), fmax3(a3, a4, f(15)), -INFINITY);
                }
                const float hmax = fmax3(fmax3(h8[hf * 4], h8[hf * 4 + 1], h8[hf * 4 + 2]), h8[hf * 4 + 3],
                                         -INFINITY) * p.sc2;
                // exps of the half relative to ref (log2 units)
                const float ref = (kMode == kLse) ? fmaxf(m_run, hmax) : hmax;
                float acc = 0.f;
                if (ref > -INFINITY) {
                    const uint64_t nref = f2_pack(-ref, -ref);
                    uint64_t acc2[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const int e0 = 2 * q;
                        const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(raw[e0 >> 5][e0 & 31]),
                                                           __uint_as_float(raw[e0 >> 5][(e0 & 31) + 1])),
                                                   sc2, nref);
                        float e0v, e1v;
                        if ((q & 3) < kEmu) {
                            ex2_poly2_d4(x2, e0v, e1v);
                        } else {
                            float x0, x1;
                            f2_unpack(x2, x0, x1);
                            e0v = ex2(x0);
                            e1v = ex2(x1);
                        }
                        acc2[q & 3] = f2_add(acc2[q & 3], f2_pack(e0v, e1v));
                    }
                    float a0, a1;
                    f2_unpack(f2_add(f2_add(acc2[0], acc2[1]), f2_add(acc2[2], acc2[3])), a0, a1);
                    acc = a0 + a1;
                }
                if (kMode == kLse) {
                    if (ref > -INFINITY) {
                        s_run = (m_run > -INFINITY ? s_run * ex2(m_run - ref) : 0.f) + acc;
                        m_run = ref;
                    }
                } else if (kB64) {                          // b = 64: the half is key block 2u + hf
                    const int n = 2 * u + hf;
                    if (n < p.M) {
                        const long long o = (static_cast<long long>(prob) * p.M + n) * 128 + rr;
                        const bool ok = row_ok && hmax > -INFINITY;
                        p.part_m[o] = ok ? hmax : -INFINITY;   // padded rows carry no mass
                        p.part_s[o] = ok ? acc : 0.f;
                    }
                } else {
                    tm[hf] = hmax;
                    ac[hf] = acc;
                }
            }
            if (kMode == kBudget && !kB64) {                // b = 128: the tile is key block u
                const float mm = fmaxf(tm[0], tm[1]);
                float ss = 0.f;
                if (mm > -INFINITY) {
                    ss = (tm[0] > -INFINITY ? ac[0] * ex2(tm[0] - mm) : 0.f) +
                         (tm[1] > -INFINITY ? ac[1] * ex2(tm[1] - mm) : 0.f);
                }
                const long long o = (static_cast<long long>(prob) * p.M + u) * 128 + rr;
                p.part_m[o] = row_ok ? mm : -INFINITY;       // padded rows carry no mass
                p.part_s[o] = row_ok ? ss : 0.f;
            }
            if (kMode == kLse && p.W != nullptr && row_ok) {
                // A3 by-product: the window maxima (16-column groups folded to b/s columns);
                // the max-pool itself runs afterwards from W and the row lse
                const int nwin = 128 / p.bs;
                float* wrow = p.W + ((static_cast<long long>(prob) * p.n_tr + u) * p.Ns + tr * 128 + rr) * nwin;
                float win[8];
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    win[c] = p.bs == 16 ? h8[c]
                           : p.bs == 32 ? fmaxf(h8[(2 * c) & 7], h8[(2 * c + 1) & 7])
                           : p.bs == 64 ? fmaxf(fmaxf(h8[(4 * c) & 7], h8[(4 * c + 1) & 7]),
                                                fmaxf(h8[(4 * c + 2) & 7], h8[(4 * c + 3) & 7]))
                                        : fmaxf(fmaxf(fmaxf(h8[0], h8[1]), fmaxf(h8[2], h8[3])),
                                                fmaxf(fmaxf(h8[4], h8[5]), fmaxf(h8[6], h8[7])));
                if (nwin == 8) {
                    reinterpret_cast<float4*>(wrow)[0] = make_float4(win[0], win[1], win[2], win[3]);
                    reinterpret_cast<float4*>(wrow)[1] = make_float4(win[4], win[5], win[6], win[7]);
                } else if (nwin == 4) {
                    *reinterpret_cast<float4*>(wrow) = make_float4(win[0], win[1], win[2], win[3]);
                } else if (nwin == 2) {
                    *reinterpret_cast<float2*>(wrow) = make_float2(win[0], win[1]);
                } else {
                    *wrow = win[0];
                }
            }
        }
        if (kMode == kLse) {
            // the two warpgroups' (max, sum) of each row -> one partial (fixed order: WG0 then WG1)
            if (eg == 1) {
                bars->red_m[rr] = m_run;
                bars->red_s[rr] = s_run;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (eg == 0 && row_ok) {
                const float m1 = bars->red_m[rr], s1 = bars->red_s[rr];
                const float mm = fmaxf(m_run, m1);
                const float ss = (m_run > -INFINITY ? s_run * ex2(m_run - mm) : 0.f) +
                                 (m1 > -INFINITY ? s1 * ex2(m1 - mm) : 0.f);
                const int k = u_begin / p.chunk;
                const long long o = (static_cast<long long>(prob) * p.Ns + tr * 128 + rr) * p.n_chunks + k;
                p.part_m[o] = mm;
                p.part_s[o] = ss;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        tc_fence_after();
        tmem_dealloc(tbase, 256);
    }
}


// A3 from the window maxima of the lse pass: L[c][m][n] = ln2 * max over the block's valid
// sampled rows i of (W[c][i][n] * sc2 - lse2[c][i]) for n <= m, -inf above the diagonal.
// The operations of a second max-pool GEMM pass (window max of raw logits, scale, subtract lse,
// max over rows, ln2) without the pass.  One CTA per (group, block row), a thread per key block.
// The block's row lse (A2's normaliser) is combined here from the lse pass's per-chunk (max,
// sum) partials (fixed chunk order), so no separate combine launch sits on the critical path.
__global__ void __launch_bounds__(256) maxpool_from_windows_kernel(int M, int Ns, int bs, int n_tr, float sc2,
                                                                   const float* __restrict__ W,
                                                                   const float* __restrict__ part_m,
                                                                   const float* __restrict__ part_s,
                                                                   int chunk, int n_chunks,
                                                                   float* __restrict__ lse_nat,
                                                                   float* __restrict__ L, int rb, int re) {
    __shared__ float lse_s[128];
    const int m = rb + blockIdx.x % (re - rb), c = blockIdx.x / (re - rb);   // block rows [rb, re)
    const int i0 = m * bs, i1 = min(i0 + bs, Ns);
    if (threadIdx.x < i1 - i0) {                       // lse2 of the block's rows from the chunk partials
        const long long i = static_cast<long long>(c) * Ns + i0 + threadIdx.x;
        const int nk = ((i0 + static_cast<int>(threadIdx.x)) / 128 + chunk) / chunk;
        const float* pm = part_m + i * n_chunks;
        const float* ps = part_s + i * n_chunks;
        float mx = -INFINITY, sum = 0.f;
        if (nk <= 16) {                                // all partials in flight at once
            float vm[16], vs[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                vm[k] = k < nk ? __ldg(pm + k) : -INFINITY;
                vs[k] = k < nk ? __ldg(ps + k) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) mx = fmaxf(mx, vm[k]);
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (k < nk) sum += vs[k] * ex2(vm[k] - mx);
        } else {
            for (int k = 0; k < nk; ++k) mx = fmaxf(mx, pm[k]);
            for (int k = 0; k < nk; ++k) sum += ps[k] * ex2(pm[k] - mx);
        }
        const float l2 = mx + __log2f(sum);
        lse_s[threadIdx.x] = l2;
        if (lse_nat) lse_nat[i] = l2 * kLn2;
    }
    __syncthreads();
    // thread per key block n <= m: max over the block's rows of W[c][n / nwin][i][n % nwin]
    const int nwin = 128 / bs;
    float* Lrow = L + (static_cast<long long>(c) * M + m) * M;
    const float* Wc = W + static_cast<long long>(c) * n_tr * Ns * nwin;
    for (int n = threadIdx.x; n < M; n += blockDim.x) {
        float w = -INFINITY;
        if (n <= m) {
            const float* Wn = Wc + (static_cast<long long>(n / nwin) * Ns) * nwin + (n % nwin);
            int i = i0;
#pragma unroll 1
            for (; i + 4 <= i1; i += 4) {              // four rows' loads in flight
                const float a0 = __ldg(Wn + static_cast<long long>(i) * nwin);
                const float a1 = __ldg(Wn + static_cast<long long>(i + 1) * nwin);
                const float a2 = __ldg(Wn + static_cast<long long>(i + 2) * nwin);
                const float a3 = __ldg(Wn + static_cast<long long>(i + 3) * nwin);
                w = fmaxf(w, fmaf(a0, sc2, -lse_s[i - i0]));
                w = fmaxf(w, fmaf(a1, sc2, -lse_s[i + 1 - i0]));
                w = fmaxf(w, fmaf(a2, sc2, -lse_s[i + 2 - i0]));
                w = fmaxf(w, fmaf(a3, sc2, -lse_s[i + 3 - i0]));
            }
            for (; i < i1; ++i) w = fmaxf(w, fmaf(__ldg(Wn + static_cast<long long>(i) * nwin), sc2, -lse_s[i - i0]));
            w *= kLn2;
        }
        Lrow[n] = w;
    }
}


// Alg. 1 lines 1-2 from the per-(block u, row t) partials (m_tu, s_tu) of the budget pass,
// in two grid-wide phases (the single-CTA-per-head version left 116 of 148 SMs idle):
//   phase 1: per (head, chunk of kCombChunks blocks) and row t, the online (max, sum) of
//            the chunk's partials -> cm/cs [Hl][n_chunks][128]
//   phase 2: per (head, chunk): row lse_t from the chunk partials (fixed order), then the
//            block masses a[u] = (1/b^2) sum_t s_tu 2^(m_tu - lse_t) of the chunk's blocks.
constexpr int kCombChunk = 16;   // blocks per chunk

__global__ void __launch_bounds__(128) budget_part_kernel(int M, int n_chunks, const float* __restrict__ part_m,
                                                          const float* __restrict__ part_s,
                                                          float* __restrict__ cm, float* __restrict__ cs) {
    const int hl = blockIdx.x / n_chunks, k = blockIdx.x % n_chunks;
    const int t = threadIdx.x;
    const int u0 = k * kCombChunk, u1 = min(u0 + kCombChunk, M);
    const float* pm = part_m + static_cast<long long>(hl) * M * 128;
    const float* ps = part_s + static_cast<long long>(hl) * M * 128;
    float m = -INFINITY, sum = 0.f;
#pragma unroll 4
    for (int u = u0; u < u1; ++u) {
        const float mu = __ldg(pm + static_cast<long long>(u) * 128 + t);
        const float su = __ldg(ps + static_cast<long long>(u) * 128 + t);
        if (!(su > 0.f)) continue;                  // padded row (no mass)
        if (mu > m) {
            sum = sum * ex2(m - mu) + su;
            m = mu;
        } else {
            sum += su * ex2(mu - m);
        }
    }
    const long long o = (static_cast<long long>(hl) * n_chunks + k) * 128 + t;
    cm[o] = m;
    cs[o] = sum;
}

__global__ void __launch_bounds__(256) budget_mass_kernel(int M, int n_chunks, const float* __restrict__ part_m,
                                                          const float* __restrict__ part_s,
                                                          const float* __restrict__ cm,
                                                          const float* __restrict__ cs,
                                                          float* __restrict__ bmass) {
    __shared__ float lse_s[128];
    const int hl = blockIdx.x / n_chunks, k = blockIdx.x % n_chunks;
    if (threadIdx.x < 128) {
        const int t = threadIdx.x;
        const float* pcm = cm + static_cast<long long>(hl) * n_chunks * 128 + t;
        const float* pcs = cs + static_cast<long long>(hl) * n_chunks * 128 + t;
        float mx = -INFINITY;
        for (int q = 0; q < n_chunks; ++q) mx = fmaxf(mx, pcm[q * 128]);
        float s2 = 0.f;
        for (int q = 0; q < n_chunks; ++q) {
            const float sq = pcs[q * 128];
            s2 += (sq > 0.f) ? sq * ex2(pcm[q * 128] - mx) : 0.f;
        }
        lse_s[t] = (s2 > 0.f) ? mx + __log2f(s2) : INFINITY;   // padded row: no mass
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    float l4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) l4[q] = lse_s[lane + 32 * q];
    const float* pm = part_m + static_cast<long long>(hl) * M * 128;
    const float* ps = part_s + static_cast<long long>(hl) * M * 128;
    const int u1 = min((k + 1) * kCombChunk, M);
    for (int u = k * kCombChunk + w; u < u1; u += 8) {
        const float* pmu = pm + static_cast<long long>(u) * 128;
        const float* psu = ps + static_cast<long long>(u) * 128;
        float a = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float sv = __ldg(psu + lane + 32 * q);
            if (sv > 0.f) a += sv * ex2(__ldg(pmu + lane + 32 * q) - l4[q]);
        }
        a = warp_sum(a);
        if (lane == 0) bmass[static_cast<long long>(hl) * M + u] = a / (128.f * 128.f);
    }
}

// Exp2 split between MUFU and the FMA pipe in the score epilogues: 1/4 of the column pairs
// on the FMA-pipe polynomial (A2 pass 213 -> 198 us, Alg. 1 pass 178 -> 166 us at 128K).
#ifndef PA_SCORE_EMU
#define PA_SCORE_EMU 1
#endif
constexpr int kScoreEmu = PA_SCORE_EMU;

// Key tiles per CTA of the score passes; PROXYATTN_SCORE_CHUNK=16/32/64 overrides.
// Key tiles per CTA of the proxy (A2) pass: the default unless the causal grid of this
// config would leave the GPU under-filled (short N), then the largest of 8 / 4 / 2 that gives
// >= 2 CTAs per SM (128 / 64 / 32-row proxies at 16K: 48 CTAs at 16 tiles each otherwise).
int proxy_chunk(const Dims& D, int base) {
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const long long n_tr = (D.Ns + 127) / 128;
    int c = base;
    while (c > 2) {
        long long ctas = 0;
        for (long long tr = 0; tr < n_tr; ++tr) ctas += (tr + c) / c;
        if (ctas * D.gl >= 2LL * n_sm) break;
        c >>= 1;
    }
    return c;
}

constexpr int score_chunk() { return kChunk; }


using ScoreKernel = void (*)(const CUtensorMap, const CUtensorMap, ScoreParams);

// mode: kLse (the A2 pass) or kBudget (Alg. 1; b64 = block size 64)
ScoreKernel score_kernel(int d, int mode, bool b64 = false) {
    if (mode == kLse) return d == 64 ? score_tc_kernel<0, false, 64, kLse> : score_tc_kernel<kScoreEmu, false, 128, kLse>;
    if (d == 64) return b64 ? score_tc_kernel<0, true, 64, kBudget> : score_tc_kernel<0, false, 64, kBudget>;
    return b64 ? score_tc_kernel<0, true, 128, kBudget> : score_tc_kernel<kScoreEmu, false, 128, kBudget>;
}

bool set_smem_attr() {
    for (int d : {64, 128})
        for (int mode : {static_cast<int>(kLse), static_cast<int>(kBudget)})
            for (bool b64 : {false, true})
                if (ensure_smem_attr(reinterpret_cast<const void*>(score_kernel(d, mode, b64)),
                                     static_cast<int>(kSmem)) != cudaSuccess)
                    return false;
    return true;
}

}  // namespace

bool score_tc_supported(const Dims& D) {
    return !D.fp32 && (D.d == 64 || D.d == 128) && (D.b == 64 || D.b == 128) &&
           (D.bs == 16 || D.bs == 32 || D.bs == 64 || D.bs == 128);
}

size_t score_tc_scratch_bytes(const Dims& D) {
    const int n_tr = static_cast<int>((D.Ns + 127) / 128);
    const int chunk = proxy_chunk(D, kChunk);
    const int n_chunks = (n_tr + chunk - 1) / chunk;
    // A2/A3: lse partials, lse2, window maxima W [gl][Ns][M]
    const size_t nwin = 128 / (D.bs > 0 ? D.bs : 1);
    return 2ull * D.gl * D.Ns * n_chunks * 4 + 2ull * D.gl * D.Ns * 4 + 32 +
           static_cast<size_t>(D.gl) * n_tr * D.Ns * nwin * 4;   // W [gl][n_tr][Ns][nwin], aligned
}

size_t score_tc_budget_scratch_bytes(const Dims& D) {
    // A4: (m, s) partials [Hl][M][128] + the combine's chunk partials (own region: the
    // budget pass may run concurrently with A2/A3)
    const size_t n_comb = (D.M + kCombChunk - 1) / kCombChunk;
    return 2ull * D.Hl * D.M * 128 * 4 + 2ull * D.Hl * n_comb * 128 * 4;
}

// A2 + A3 on tcgen05.  scratch: score_tc_scratch_bytes(D); lse_nat (may be null) receives
// the natural-log lse for inspection.
cudaError_t launch_proxy_tc(const Dims& D, const void* Pq, const void* Pk, float* scratch,
                            float* lse_nat, float* L, cudaStream_t st, int tr0, int tr1) {
    if (!set_smem_attr()) return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    const uint64_t rows = static_cast<uint64_t>(D.gl) * D.Ns;
    if (!make_map_bf16_sw128(&ma, Pq, rows, D.d, 128) || !make_map_bf16_sw128(&mb, Pk, rows, D.d, 128))
        return cudaErrorInvalidValue;
    ScoreParams p{};
    p.d = D.d;
    p.b = D.b;
    p.Ns = static_cast<int>(D.Ns);
    p.M = D.M;
    p.n_tr = static_cast<int>((D.Ns + 127) / 128);
    p.chunk = proxy_chunk(D, score_chunk());
    p.n_chunks = (p.n_tr + p.chunk - 1) / p.chunk;
    p.tr_lo = tr0;
    p.tr_hi = tr1 < 0 ? p.n_tr : tr1;
    p.bs = D.bs;
    // Eq. 2 means + 1/sqrt(d) folded into the scale (Z2, Z5), in log2 units.
    p.sc2 = has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD)
                ? kLog2e / sqrtf(static_cast<float>(D.d))
                : kLog2e / (static_cast<float>(D.gq) * static_cast<float>(D.gk) * sqrtf(static_cast<float>(D.d)));
    float* part_m = scratch;
    float* part_s = part_m + static_cast<size_t>(D.gl) * D.Ns * p.n_chunks;
    float* lse2 = part_s + static_cast<size_t>(D.gl) * D.Ns * p.n_chunks;
    p.part_m = part_m;
    p.part_s = part_s;
    // W: 32-byte aligned (its rows are stored as float4 / float2 vectors)
    const uintptr_t w_addr = reinterpret_cast<uintptr_t>(lse2 + static_cast<size_t>(D.gl) * D.Ns);
    p.W = reinterpret_cast<float*>((w_addr + 31) & ~static_cast<uintptr_t>(31));
    const unsigned grid = static_cast<unsigned>(D.gl) * (p.tr_hi - p.tr_lo) * p.n_chunks;
    p.mode = kLse;
    score_kernel(D.d, kLse)<<<grid, kThreads, kSmem, st>>>(ma, mb, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // A3: the max-pool (with the row lse combine) from the window maxima, block rows [rb, re)
    maxpool_from_windows_kernel<<<static_cast<unsigned>(D.gl) * (D.re - D.rb), 256, 0, st>>>(
        D.M, p.Ns, p.bs, p.n_tr, p.sc2, p.W, part_m, part_s, p.chunk, p.n_chunks, lse_nat, L, D.rb, D.re);
    return cudaGetLastError();
}

// A4 on tcgen05: per-(row, block) partials, then combine into block masses bmass[Hl][M].
cudaError_t launch_budget_tc(const Dims& D, const void* Q, const void* K, float* scratch,
                             float* bmass, cudaStream_t st) {
    if (!set_smem_attr()) return cudaErrorInvalidValue;
    CUtensorMap ma, mb;
    if (!make_map_bf16_sw128_3d(&ma, Q, D.Hl, D.N, D.q_ts, D.q_hs, 128, D.d) ||
        !make_map_bf16_sw128_3d(&mb, K, D.Hkvl, D.N, D.kv_ts, D.kv_hs, 128, D.d))
        return cudaErrorInvalidValue;
    ScoreParams p{};
    p.mode = kBudget;
    p.d = D.d;
    p.b = D.b;
    p.N = static_cast<int>(D.N);
    p.M = D.M;
    p.r = D.r;
    p.n_kt = static_cast<int>((static_cast<long long>(D.M) * D.b + 127) / 128);
    p.chunk = score_chunk();
    p.n_chunks = (p.n_kt + p.chunk - 1) / p.chunk;
    p.sc2 = kLog2e / sqrtf(static_cast<float>(D.d));
    p.part_m = scratch;
    p.part_s = scratch + static_cast<size_t>(D.Hl) * D.M * 128;
    const unsigned grid = static_cast<unsigned>(D.Hl) * p.n_chunks;
    score_kernel(D.d, kBudget, D.b == 64)<<<grid, kThreads, kSmem, st>>>(ma, mb, p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int n_comb = (D.M + kCombChunk - 1) / kCombChunk;
    float* cm = p.part_s + static_cast<size_t>(D.Hl) * D.M * 128;
    float* cs = cm + static_cast<size_t>(D.Hl) * n_comb * 128;
    budget_part_kernel<<<D.Hl * n_comb, 128, 0, st>>>(D.M, n_comb, p.part_m, p.part_s, cm, cs);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    budget_mass_kernel<<<D.Hl * n_comb, 256, 0, st>>>(D.M, n_comb, p.part_m, p.part_s, cm, cs, bmass);
    return cudaGetLastError();
}

}  // namespace pa
