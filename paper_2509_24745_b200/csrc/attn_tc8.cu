// attn_tc8.cu — bf16 block-sparse causal prefill attention on tcgen05 (A7 / A8), variant v8:
// the attn_tc7 pipeline (two key-block streams sharing one O under a fixed per-row softmax
// reference, separate P buffers, S released right after tcgen05.ld) made PERSISTENT: one
// CTA per SM pulls (head, block-row) items from an atomic counter, and the ring / barrier
// phases run on across items, so the next row's Q/K loads, its first S MMAs and its softmax
// overlap the previous row's last PVs and its epilogue (dedicated epilogue warps).  In
// attn_tc7 that per-row prologue/epilogue cost ~5 us per CTA, ~8 % of the launch at 128K.
//
// Method: O[h][t] = sum over keys k of the selected blocks, k <= t, of
// softmax(Q[h][t] K[kv(h)][k] / sqrt(d)) V[kv(h)][k],
// evaluated as sum 2^(x - m_ref) V / sum 2^(x - m_ref) with m_ref the max of the row's two
// first blocks (softmax is shift invariant).  A row on which some P would exceed 2^32 is
// appended to a list during the fast launch (its output is then overwritten) and the exact
// launch recomputes the listed rows with m_ref = the true row max (max-only sweep, then the
// fixed pass), so the result never depends on the fast path's bound.
//
// Warp roles (512 threads, 4 warpgroups):
//   warp 0      item scheduler (atomic counter) + TMA producer of Q and K (3-stage ring)
//   warp 1      TMEM allocator + S issuer          warp 2   PV issuer
//   warp 3      TMA producer of V (2-stage ring)
//   warps 4-7   epilogue: O (TMEM) * 1/l -> bf16 -> global; releases O for the next row
//   warps 8-11  softmax of stream 0, warps 12-15 of stream 1 (thread = row = TMEM lane)
// TMEM (512 columns): O [0,128)  S_0 [128,256)  S_1 [256,384)  P_0 [384,448)  P_1 [448,512).
// (kB = 64: each stream's S and P regions hold two buffers, so a stream's next S and P
// never wait for its previous block's PV.)
//
// Shapes (template <kEmu, kD, kB>): head_dim kD in {64, 128}, block kB in {64, 128}.  The
// 128 query rows of a work unit are the 128 TMEM lanes.  kB = 128: one (head, block row).
// kB = 64: a PAIR of adjacent 64-row block rows (2q, 2q+1) of one head (lanes 0-63 row 2q,
// 64-127 row 2q+1), so every S = Q K^T tile is still M = 128 (an M = 64 tcgen05.mma costs
// the issue slot of an M = 128 one).  The pair walks the UNION of its two ascending lists
// (1.12x the mean list at the 128K bench inputs; pairing two heads of one KV head instead
// measured 1.41x, scripts/pair_union_stats.py); a block that is not in a half's list gets
// P = 0 for that half.  The fixed reference of a half is the max over its member blocks
// among the two first blocks, else (neither is a member) the raw max of those blocks; rows
// whose sum would then underflow (l < 2^-60) or overflow are re-run by the exact launch,
// as for kB = 128.
#include <cuda_bf16.h>

#include <climits>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"
#include "tma_host.h"

// Energy-attribution experiments (never in the shipped build; scripts/attn_experiments.sh
// builds them with PROXYATTN_NVCC_DEFINES and times the launch): each removes one component
// of the per-block work and so produces WRONG outputs.  PA_X_NOMUFU: P = x instead of 2^x;
// PA_X_NOLOAD: K/V TMA loads skipped after the rings are filled; PA_X_NOQK / PA_X_NOPV: the
// S / PV tcgen05.mma skipped (commits kept); PA_X_EXBF16: ex2.approx.ftz.bf16x2 on a bf16
// argument; PA_X_HALFLOAD: every other K and V load skipped (half the L2 -> SMEM traffic);
// PA_X_NOKLOAD / PA_X_NOVLOAD: only the K / only the V loads skipped.  Any of them also disables the overflow flagging (no exact re-run).
#if defined(PA_X_NOMUFU) || defined(PA_X_NOLOAD) || defined(PA_X_NOQK) || defined(PA_X_NOPV) || \
    defined(PA_X_EXBF16) || defined(PA_X_HALFLOAD) || defined(PA_X_NOKLOAD) || defined(PA_X_NOVLOAD)
#define PA_X_ANY 1
#endif

namespace pa {
namespace {

constexpr int kTileRows = 128;
constexpr int kBox = kTileRows * 64 * 2;   // 16 KB: [128 rows][64 bf16] SW128 box
constexpr float kUnderflow = -60.0f;       // log2 floor of a row sum under a non-attained reference
#ifndef PA_KSTAGES
#define PA_KSTAGES 3
#endif
#ifndef PA_VSTAGES
#define PA_VSTAGES 2
#endif
// exp2 split per shape (of every 8 key-column pairs, this many on the FMA-pipe cubic); build
// defines so the split can be re-measured without editing the dispatch
#ifndef PA_EMU_D128
#define PA_EMU_D128 0
#endif
#ifndef PA_EMU_D64
#define PA_EMU_D64 2
#endif
#ifndef PA_EMU_B64
#define PA_EMU_B64 0
#endif
// bf16 pack of P (build define for A/B timing): 0 F2FP (RNE)
#ifndef PA_PACK
#define PA_PACK 0
#endif
constexpr int kKStages = PA_KSTAGES;   // K ring (3) and V ring (2) stages of 32 KB tiles
constexpr int kVStages = PA_VSTAGES;
constexpr int kItemSlots = 4;
constexpr int kThreads = 512;
constexpr float kOverflow = 32.0f;         // log2 headroom of P over the fast reference
constexpr uint32_t kColO = 0, kColS = 128, kColP = 384;
constexpr int kItemConsumers = 1 + 1 + 1 + 4 + 8;   // S, PV, V, epilogue warps, softmax warps

struct Item {
    int item;   // -1: no more work
    int cnt;
};

struct __align__(8) Bars8 {
    uint64_t q_full, q_empty;
    uint64_t k_full[kKStages];
    uint64_t k_empty[kKStages];
    uint64_t v_full[kVStages];
    uint64_t v_empty[kVStages];
    uint64_t s_full[2][2];   // [stream][buffer] (kB = 64: two 64-column S buffers per stream)
    uint64_t s_free[2][2];
    uint64_t p_full[2][2];   // kB = 128: [stream][half]; kB = 64: [stream][buffer]
    uint64_t p_free[2][2];   // [stream][buffer]
    uint64_t o_final, o_free;
    uint64_t l_ready[2];     // per item parity: both streams' row sums written
    uint64_t item_full[kItemSlots];
    uint64_t item_empty[kItemSlots];
    Item items[kItemSlots];
    uint32_t tmem_base;
    float red[2][128];       // first-block / true row max exchange between the streams
    float red_u[2][128];     // kB = 64: the same without the membership mask
    float lsum[2][2][128];   // [item parity][stream][row] row sums for the epilogue
};

template <int kD, int kB>
struct Shape {
    static constexpr int kQTile = (kD / 64) * kBox;      // Q: 128 rows x kD (64-col boxes at kBox)
    static constexpr int kKBox = kB * 128;               // K / V: [kB rows][64 bf16] box
    static constexpr int kKTile = (kD / 64) * kKBox;
    static constexpr int kChunks = kB / 32;               // 32-column S chunks per block
    static constexpr int kHalves = kB / 64;               // P halves (4 PV MMAs of K = 16 each)
    static constexpr size_t kSmem = 1024 + kQTile + kKTile * (kKStages + kVStages) + sizeof(Bars8);
    static_assert(kSmem <= 232448, "shared memory budget");
};

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

struct Sched {        // device-side scheduler state of one launch pair (zeroed before launch)
    int next[2];      // item counters of the fast and the exact launch
    int n_flagged;    // rows appended by the fast launch
    int pad;
};

// Block-list walk of a kB = 64 work unit: the ascending union of the pair's two lists, with
// each element's membership (bit 0: row A = lanes 0-63, bit 1: row B = lanes 64-127).
struct PairWalk {
    const int* a;
    const int* b;
    int ca, cb, pa, pb, j;
    bool dense;
    __device__ __forceinline__ int next(int& mem) {
        if (dense) {   // lists 0..ca-1 and 0..cb-1, walked diagonal-first (see block_n below)
            const int n = max(ca, cb) - 1 - j++;
            mem = (n < ca ? 1 : 0) | (n < cb ? 2 : 0);
            return n;
        }
        const int x = pa < ca ? __ldg(a + pa) : INT_MAX;
        const int y = pb < cb ? __ldg(b + pb) : INT_MAX;
        const int n = min(x, y);
        mem = (x == n ? 1 : 0) | (y == n ? 2 : 0);
        pa += (x == n);
        pb += (y == n);
        return n;
    }
};

// kEmu: of every 8 key-column pairs, kEmu use the FMA-pipe exp2; kVar: varlen (packed sequences)
template <int kEmu, int kD, int kB, bool kVar = false>
__global__ void __launch_bounds__(kThreads, 1)
attn_tc8_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O,
                const int* __restrict__ block_cnt, const int* __restrict__ block_idx, int N, int M,
                int r, float scale_log2, int row_lo, int row_hi, int n_total, Sched* sched,
                int* flagged, int exact, long long o_hs, long long o_ts, const int* __restrict__ ucnt,
                const int* __restrict__ kvperm, const SeqDesc* __restrict__ seqs,
                int n_seqs) {
    using Sh = Shape<kD, kB>;
    constexpr bool kPair = (kB == 64);
    constexpr int kNB = kPair ? 2 : 1;   // S / P buffers per stream (a 64-key S is 64 columns)
    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned base, derived from the __shared__ array by pointer arithmetic so that
    // the compiler keeps the shared state space (LDS/STS, not generic loads, for the barriers
    // and exchange arrays)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = smem;
    uint8_t* sK = smem + Sh::kQTile;
    uint8_t* sV = sK + Sh::kKTile * kKStages;
    Bars8* bars = reinterpret_cast<Bars8*>(sV + Sh::kKTile * kVStages);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nrows = row_hi - row_lo;
    // kB = 64: row pairs q in [q_lo, q_hi) cover the block rows [row_lo, row_hi)
    const int q_lo = row_lo >> 1, q_hi = (row_hi + 1) >> 1;
    const int per_kv = r * (kPair ? q_hi - q_lo : nrows);   // work units per kv head
    const int n_items = exact ? sched->n_flagged : n_total;
    const bool dense = (block_cnt == nullptr);
    const int passes = exact ? 2 : 1;   // exact: max sweep, then the fixed pass

    if (threadIdx.x == 0) {
        mbar_init(&bars->q_full, 1);
        mbar_init(&bars->q_empty, 1);
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(&bars->k_full[s], 1);
            mbar_init(&bars->k_empty[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&bars->v_full[s], 1);
            mbar_init(&bars->v_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            for (int k = 0; k < 2; ++k) {
                mbar_init(&bars->s_full[s][k], 1);
                mbar_init(&bars->s_free[s][k], 128);
                mbar_init(&bars->p_full[s][k], 128);
                mbar_init(&bars->p_free[s][k], 1);
            }
            mbar_init(&bars->l_ready[s], 256);
        }
        mbar_init(&bars->o_final, 1);
        mbar_init(&bars->o_free, 128);
        for (int i = 0; i < kItemSlots; ++i) {
            mbar_init(&bars->item_full[i], 1);
            mbar_init(&bars->item_empty[i], kItemConsumers);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;

    // The current item's sequence (varlen: n_seqs > 0, one packed launch over all sequences;
    // each role decodes every item it handles, so these are per-thread): token offset, length,
    // block rows and the base of its block lists.
    long long c_tok = 0;
    int c_N = N, c_M = M;
    const int* c_cnt = block_cnt;
    const int* c_idx = block_idx;
    // item decode (kv-head major — KV heads in decreasing total work when kvperm is given, so
    // the last heads scheduled are the lightest — heavy rows first): head hl, its block row mA (kB = 128), or
    // its row pair (mA, mB) = (2q, 2q+1) (kB = 64; -1 for a row outside [row_lo, row_hi))
    auto decode = [&](int item, int& hl, int& mA, int& mB, int& kvl) {
        int pk = per_kv, rhi = row_hi;
        if (kVar && n_seqs > 0) {  // varlen (kB = 128): sequence s holds items [item0_s, item0_{s+1})
            int lo = 0, hi = n_seqs - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (__ldg(&seqs[mid].item0) <= item) lo = mid;
                else hi = mid - 1;
            }
            c_tok = __ldg(&seqs[lo].tok0);
            c_N = __ldg(&seqs[lo].N);
            c_M = __ldg(&seqs[lo].M);
            c_cnt = block_cnt + __ldg(&seqs[lo].cnt_off);
            c_idx = block_idx + __ldg(&seqs[lo].idx_off);
            item -= __ldg(&seqs[lo].item0);
            pk = r * c_M;
            rhi = c_M;
        }
        kvl = kvperm ? __ldg(kvperm + item / pk) : item / pk;
        const int rem = item % pk;
        hl = kvl * r + rem % r;
        if (kPair) {
            const int q = q_hi - 1 - rem / r;
            mA = (2 * q >= row_lo) ? 2 * q : -1;
            mB = (2 * q + 1 < row_hi) ? 2 * q + 1 : -1;
        } else {
            mA = rhi - 1 - rem / r;
            mB = -1;
        }
    };
    auto get_item = [&](int it) -> Item {         // consumers: wait for slot, read, release
        const int slot = it % kItemSlots;
        mbar_wait(&bars->item_full[slot], (it / kItemSlots) & 1);
        const Item x = bars->items[slot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->item_empty[slot]);
        return x;
    };
    auto list_of = [&](int hl, int m) -> const int* {
        return dense ? nullptr : c_idx + (static_cast<long long>(hl) * c_M + m) * c_M;
    };
    auto count_of = [&](int hl, int m) -> int {
        return m < 0 ? 0 : dense ? m + 1 : __ldg(c_cnt + static_cast<long long>(hl) * c_M + m);
    };
    auto walk_of = [&](int hl, int mA, int mB) -> PairWalk {
        PairWalk w;
        w.dense = dense;
        w.a = mA >= 0 ? list_of(hl, mA) : nullptr;
        w.b = mB >= 0 ? list_of(hl, mB) : nullptr;
        w.ca = count_of(hl, mA);
        w.cb = count_of(hl, mB);
        w.pa = w.pb = w.j = 0;
        return w;
    };

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
        if (warp == 0) {
            // ---------------------------------------- scheduler + Q/K producer --
            if (lane == 0) {
                tma_prefetch(&tmQ);
                tma_prefetch(&tmK);
                int gk = 0;
                for (int it = 0;; ++it) {
                    const int slot = it % kItemSlots;
                    if (it >= kItemSlots) mbar_wait(&bars->item_empty[slot], ((it / kItemSlots) - 1) & 1);
                    int k = atomicAdd(&sched->next[exact], 1);
                    Item x{-1, 0};
                    if (k < n_items) {
                        x.item = exact ? flagged[k] : k;
                        int hl, mA, mB, kvl;
                        decode(x.item, hl, mA, mB, kvl);
                        // ucnt is indexed by the natural (unpermuted) kv-head-major item
                        x.cnt = !kPair ? count_of(hl, mA)
                              : dense ? max(count_of(hl, mA), count_of(hl, mB))
                                      : __ldg(ucnt + kvl * per_kv + x.item % per_kv);
                    }
                    bars->items[slot] = x;
                    mbar_arrive(&bars->item_full[slot]);   // release semantics publish x
                    if (x.item < 0) break;
                    int hl, mA, mB, kvl;
                    decode(x.item, hl, mA, mB, kvl);
                    if (it > 0) mbar_wait(&bars->q_empty, (it - 1) & 1);   // last S of it-1 done
                    // the unit's 128 query rows (kB = 64: rows 2q*64 .. 2q*64+127)
                    const int q_row0 = static_cast<int>(c_tok) + (kPair ? (mA >= 0 ? mA : mB - 1) * kB : mA * kTileRows);
                    mbar_expect_tx(&bars->q_full, Sh::kQTile);
#pragma unroll
                    for (int ch = 0; ch < kD / 64; ++ch)
                        tma_load_3d(sQ + ch * kBox, &tmQ, &bars->q_full, ch * 64, q_row0, hl);
                    const int* list = list_of(hl, mA);
                    for (int pass = 0; pass < passes; ++pass) {
                        PairWalk w = walk_of(hl, mA, mB);
                        for (int j = 0; j < x.cnt; ++j, ++gk) {
                            const int st = gk % kKStages;
                            if (gk >= kKStages) mbar_wait(&bars->k_empty[st], ((gk / kKStages) - 1) & 1);
                            int mem;
                            const int n = kPair ? w.next(mem) : dense ? mA - j : __ldg(list + j);
#if defined(PA_X_NOLOAD) || defined(PA_X_NOKLOAD) || defined(PA_X_HALFLOAD)
#ifdef PA_X_HALFLOAD
                            if (gk >= kKStages && (j & 1)) {
#else
                            if (gk >= kKStages) {
#endif
                                mbar_arrive(&bars->k_full[st]);
                                continue;
                            }
#endif
                            mbar_expect_tx(&bars->k_full[st], Sh::kKTile);
#pragma unroll
                            for (int ch = 0; ch < kD / 64; ++ch)
                                tma_load_3d(sK + st * Sh::kKTile + ch * Sh::kKBox, &tmK, &bars->k_full[st],
                                            ch * 64, static_cast<int>(c_tok) + n * kB, kvl);
                        }
                    }
                }
            }
        } else if (warp == 3) {
            // ------------------------------------------------------- V producer --
            if (lane == 0) tma_prefetch(&tmV);
            int gv = 0;
            for (int it = 0;; ++it) {
                const Item x = get_item(it);
                if (x.item < 0) break;
                if (lane == 0) {
                    int hl, mA, mB, kvl;
                    decode(x.item, hl, mA, mB, kvl);
                    const int* list = list_of(hl, mA);
                    PairWalk w = walk_of(hl, mA, mB);
                    for (int j = 0; j < x.cnt; ++j, ++gv) {
                        const int st = gv % kVStages;
                        if (gv >= kVStages) mbar_wait(&bars->v_empty[st], ((gv / kVStages) - 1) & 1);
                        int mem;
                        const int n = kPair ? w.next(mem) : dense ? mA - j : __ldg(list + j);
#if defined(PA_X_NOLOAD) || defined(PA_X_NOVLOAD) || defined(PA_X_HALFLOAD)
#ifdef PA_X_HALFLOAD
                        if (gv >= kVStages && (j & 1)) {
#else
                        if (gv >= kVStages) {
#endif
                            mbar_arrive(&bars->v_full[st]);
                            continue;
                        }
#endif
                        mbar_expect_tx(&bars->v_full[st], Sh::kKTile);
#pragma unroll
                        for (int ch = 0; ch < kD / 64; ++ch)
                            tma_load_3d(sV + st * Sh::kKTile + ch * Sh::kKBox, &tmV, &bars->v_full[st],
                                        ch * 64, static_cast<int>(c_tok) + n * kB, kvl);
                    }
                }
                __syncwarp();
            }
        } else if (warp == 1) {
            // -------------------------------------------------------- S issuer --
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, kB, 0, 0);
            const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
            const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
            const bool leader = elect_one();
            int gk = 0, gs0 = 0, gs1 = 0;   // per-stream S counts (scalars: no local-memory array)
            for (int it = 0;; ++it) {
                const Item x = get_item(it);
                if (x.item < 0) break;
                mbar_wait(&bars->q_full, it & 1);
                for (int pass = 0; pass < passes; ++pass) {
                    for (int j = 0; j < x.cnt; ++j, ++gk) {
                        const int s = j & 1;
                        const int gss = s ? gs1 : gs0;
                        const int sb = gss % kNB;         // this stream's S buffer
                        if (gss >= kNB) mbar_wait(&bars->s_free[s][sb], ((gss / kNB) - 1) & 1);
                        if (s) ++gs1;
                        else ++gs0;
                        const int st = gk % kKStages;
                        mbar_wait(&bars->k_full[st], (gk / kKStages) & 1);
                        tc_fence_after();
                        if (leader) {
                            const uint64_t b0 = dk + (st * Sh::kKTile >> 4);
#pragma unroll
                            for (int kk = 0; kk < kD / 16; ++kk) {
                                const uint32_t offq = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
                                const uint32_t offk = ((kk >> 2) * Sh::kKBox + (kk & 3) * 32) >> 4;
#ifndef PA_X_NOQK
                                umma_ss(tbase + kColS + s * 128 + sb * 64, dq + offq, b0 + offk, idesc_qk,
                                        kk > 0 ? 1u : 0u);
#endif
                            }
                            tc_commit(&bars->k_empty[st]);
                            tc_commit(&bars->s_full[s][sb]);
                        }
                        __syncwarp();
                    }
                }
                if (leader) tc_commit(&bars->q_empty);   // Q may be replaced by the next row's
                __syncwarp();
            }
        } else {
            // ------------------------------------------------------- PV issuer --
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, kD, 0, 1);
            const uint64_t dv = sdesc_sw128(smem_u32(sV), Sh::kKBox, 1024);
            const bool leader = elect_one();
            int gv = 0, gp0 = 0, gp1 = 0;   // per-stream P counts
            for (int it = 0;; ++it) {
                const Item x = get_item(it);
                if (x.item < 0) break;
                for (int j = 0; j < x.cnt; ++j, ++gv) {
                    const int s = j & 1;
                    const int st = gv % kVStages;
                    mbar_wait(&bars->v_full[st], (gv / kVStages) & 1);
                    if (j == 0 && it > 0) mbar_wait(&bars->o_free, (it - 1) & 1);   // O read out
                    const int gps = s ? gp1 : gp0;
                    const int pb = gps % kNB;             // this stream's P buffer
#pragma unroll
                    for (int half = 0; half < Sh::kHalves; ++half) {
                        mbar_wait(&bars->p_full[s][kPair ? pb : half], (gps / kNB) & 1);
                        tc_fence_after();
                        if (leader) {
                            const uint64_t b0 = dv + (st * Sh::kKTile >> 4);
#pragma unroll
                            for (int k4 = 0; k4 < 4; ++k4) {
                                const int kk = half * 4 + k4;
#ifndef PA_X_NOPV
                                umma_ts(tbase + kColO, tbase + kColP + s * 64 + pb * 32 + kk * 8,
                                        b0 + (kk * 2048 >> 4), idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
#endif
                            }
                        }
                        __syncwarp();
                    }
                    if (s) ++gp1;
                    else ++gp0;
                    if (leader) {
                        tc_commit(&bars->v_empty[st]);
                        tc_commit(&bars->p_free[s][pb]);
                    }
                    __syncwarp();
                }
                if (leader) tc_commit(&bars->o_final);
                __syncwarp();
            }
        }
    } else if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
        // ------------------------------------------------------------- epilogue --
        const int quarter = warp & 3;
        const int rr = quarter * 32 + lane;
        const uint32_t tO = tbase + (static_cast<uint32_t>(quarter * 32) << 16) + kColO;
        for (int it = 0;; ++it) {
            const Item x = get_item(it);
            if (x.item < 0) break;
            int hl, mA, mB, kvl;
            decode(x.item, hl, mA, mB, kvl);
            const int m = (kPair && rr >= 64) ? mB : mA;         // the row's block row (-1: none)
            const long long pos = static_cast<long long>(m) * kB + (rr & (kB - 1));
            mbar_wait(&bars->l_ready[it & 1], (it >> 1) & 1);
            const float l0 = bars->lsum[it & 1][0][rr], l1 = bars->lsum[it & 1][1][rr];
            const float inv = 1.f / (l0 + l1);
#ifndef PA_X_ANY
            if (!exact) {   // a row whose P exceeded the bound (l = +inf marker): exact re-run
                bool bad = !(l0 + l1 <= 2.f * exp2f(kOverflow));
                if (kPair) bad = bad || (m >= 0 && l0 + l1 < exp2f(kUnderflow));
                if (__any_sync(0xffffffffu, bad) && lane == 0)
                    flagged[atomicAdd(&sched->n_flagged, 1)] = x.item;   // <= 4 duplicates, benign
            }
#endif
            mbar_wait(&bars->o_final, it & 1);
            tc_fence_after();
            const bool row_valid = m >= 0 && pos < c_N;
            uint4* dst = reinterpret_cast<uint4*>(O + static_cast<long long>(hl) * o_hs + (c_tok + (m < 0 ? 0 : pos)) * o_ts);
#pragma unroll
            for (int h2 = 0; h2 < kD / 64; ++h2) {
                uint32_t o[2][32];
                tmem_ld32(tO + h2 * 64, o[0]);
                tmem_ld32(tO + h2 * 64 + 32, o[1]);
                tmem_ld_wait();
                if (h2 == kD / 64 - 1) {
                    tc_fence_before();
                    mbar_arrive(&bars->o_free);           // the next row's PV may overwrite O
                }
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t pkd[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        pkd[e] = pack_bf16(__uint_as_float(o[c][2 * e]) * inv,
                                           __uint_as_float(o[c][2 * e + 1]) * inv);
                    if (row_valid) {
#pragma unroll
                        for (int v = 0; v < 4; ++v)
                            dst[h2 * 8 + c * 4 + v] =
                                make_uint4(pkd[4 * v], pkd[4 * v + 1], pkd[4 * v + 2], pkd[4 * v + 3]);
                    }
                }
            }
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 184;\n" ::: "memory");
        // -------------------------------------------------------------- softmax --
        const int s = (warp - 8) >> 2;                  // stream
        const int quarter = warp & 3;
        const int rr = quarter * 32 + lane;
        const int qrow = rr & (kB - 1);                 // query row within the block
        const int hp = kPair ? (quarter >> 1) : 0;      // kB = 64: this warp's row of the pair
        const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t tS = tbase + lane_off + kColS + s * 128;
        const uint32_t tP = tbase + lane_off + kColP + s * 64;
        const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
        int gs = 0, gp = 0;                             // this stream's S / P counters
        int sb = 0;                                     // S buffer of the block being read
        float xhi = -INFINITY;

        auto p_chunk = [&](const uint32_t (&x)[32], uint64_t nm2, uint64_t (&ls)[4], uint32_t tdst,
                           bool wait_free) {
            uint32_t pk[16];
#pragma unroll
            for (int p = 0; p < 16; ++p) {
                const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(x[2 * p]), __uint_as_float(x[2 * p + 1])),
                                           sc2, nm2);
                float p0, p1;
                if ((p & 7) < kEmu) {
                    float x0, x1;
                    f2_unpack(x2, x0, x1);
                    xhi = fmaxf(xhi, fmaxf(x0, x1));      // the poly wraps for x >= 128
                    ex2_poly2(x2, p0, p1);
                } else {
                    float x0, x1;
                    f2_unpack(x2, x0, x1);
#if defined(PA_X_NOMUFU)
                    p0 = x0;
                    p1 = x1;
#elif defined(PA_X_EXBF16)
                    uint32_t hb;
                    asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(hb) : "r"(pack_bf16(x0, x1)));
                    p0 = __uint_as_float(hb << 16);
                    p1 = __uint_as_float(hb & 0xffff0000u);
                    ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
                    pk[p] = hb;
                    continue;
#else
                    p0 = ex2(x0);
                    p1 = ex2(x1);
#endif
                }
#if PA_PACK == 1          // truncating pack (one PRMT), row sum of the fp32 values
                ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
                pk[p] = __byte_perm(__float_as_uint(p0), __float_as_uint(p1), 0x7632);
#elif PA_PACK == 2        // round half up on the integer pipe (RNE except exact ties)
                ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
                pk[p] = __byte_perm(__float_as_uint(p0) + 0x8000u, __float_as_uint(p1) + 0x8000u, 0x7632);
#elif PA_PACK == 3        // truncating pack, row sum of the truncated values
                pk[p] = __byte_perm(__float_as_uint(p0), __float_as_uint(p1), 0x7632);
                ls[p & 3] = f2_add(ls[p & 3], f2_pack(__uint_as_float(pk[p] << 16), __uint_as_float(pk[p] & 0xffff0000u)));
#else
                ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
                pk[p] = pack_bf16(p0, p1);
#endif
            }
            if (wait_free && gp >= kNB) {                // the PV kNB blocks back has read the buffer
                mbar_wait(&bars->p_free[s][gp % kNB], ((gp / kNB) - 1) & 1);
                tc_fence_after();
            }
            tmem_st16(tdst, pk);
        };
        auto mask_chunk = [&](uint32_t (&x)[32], int c) {
#pragma unroll
            for (int e = 0; e < 32; ++e)
                if (c * 32 + e > qrow) x[e] = 0xff800000u;
        };
        auto release_p = [&](int half) {
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&bars->p_full[s][kPair ? gp % kNB : half]);
        };
        auto sum_ls = [&](uint64_t (&ls)[4]) {
            const uint64_t t = f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3]));
            float a, b;
            f2_unpack(t, a, b);
            return a + b;
        };
        auto wait_s = [&]() {
            sb = gs % kNB;
            mbar_wait(&bars->s_full[s][sb], (gs / kNB) & 1);
            ++gs;
            tc_fence_after();
        };
        auto release_s = [&]() {
            tc_fence_before();
            mbar_arrive(&bars->s_free[s][sb]);
        };
        // P of the block in S_s (already landed), with the reference known: chunked TMEM
        // loads overlapped with the exp2s; S released once its last chunk is in registers.
        // A block outside this half's list (kB = 64 pairs) contributes P = 0.
        auto block_exps = [&](float m_ref, bool diag, bool mine) -> float {
            if (kPair && !mine) {
                release_s();
                if (gp >= kNB) {
                    mbar_wait(&bars->p_free[s][gp % kNB], ((gp / kNB) - 1) & 1);
                    tc_fence_after();
                }
                uint32_t z[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) z[e] = 0u;
#pragma unroll
                for (int c = 0; c < Sh::kChunks; ++c) tmem_st16(tP + (gp % kNB) * 32 + c * 16, z);
#pragma unroll
                for (int h = 0; h < Sh::kHalves; ++h) release_p(h);
                ++gp;
                return 0.f;
            }
            const uint64_t nm2 = f2_pack(-m_ref, -m_ref);
            uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
            uint32_t xb[2][32];
            const uint32_t tSb = tS + sb * 64, tPb = tP + (gp % kNB) * 32;
            tmem_ld32(tSb, xb[0]);
#pragma unroll
            for (int c = 0; c < Sh::kChunks; ++c) {
                tmem_ld_wait_regs(xb[c & 1]);
                if (c + 1 < Sh::kChunks) tmem_ld32(tSb + 32 * (c + 1), xb[(c + 1) & 1]);
                else release_s();
                if (diag) mask_chunk(xb[c & 1], c);
                p_chunk(xb[c & 1], nm2, ls, tPb + 16 * c, c == 0);
                if (c & 1) release_p(c >> 1);
            }
            ++gp;
            return sum_ls(ls);
        };
        // row max of the block in S_s (raw logits), chunked; S stays in TMEM
        auto block_max = [&](bool diag) -> float {
            float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
            uint32_t xb[2][32];
            auto fold = [&](uint32_t (&x)[32], int c) {
                if (diag) mask_chunk(x, c);
#pragma unroll
                for (int e = 0; e < 32; e += 2)
                    mx[(e >> 1) & 3] = fmaxf(mx[(e >> 1) & 3], fmaxf(__uint_as_float(x[e]), __uint_as_float(x[e + 1])));
            };
            const uint32_t tSb = tS + sb * 64;
            tmem_ld32(tSb, xb[0]);
#pragma unroll
            for (int c = 0; c < Sh::kChunks; ++c) {
                tmem_ld_wait_regs(xb[c & 1]);
                if (c + 1 < Sh::kChunks) tmem_ld32(tSb + 32 * (c + 1), xb[(c + 1) & 1]);
                fold(xb[c & 1], c);
            }
            return fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        };
        // the two streams' maxima -> the shared reference (log2 units); kB = 64: the max over
        // member blocks `vm`, else (no member among the first blocks) the raw max `vu`
        auto exchange_max = [&](float vm, float vu) {
            bars->red[s][rr] = vm;
            if (kPair) bars->red_u[s][rr] = vu;
            softmax_bar();
            float r2 = fmaxf(bars->red[0][rr], bars->red[1][rr]);
            if (kPair && r2 == -INFINITY) r2 = fmaxf(bars->red_u[0][rr], bars->red_u[1][rr]);
            softmax_bar();
            return r2 * scale_log2;
        };

        for (int it = 0;; ++it) {
            const Item x = get_item(it);
            if (x.item < 0) break;
            int hl, mA, mB, kvl;
            decode(x.item, hl, mA, mB, kvl);
            const int m = hp ? mB : mA;                 // this warp's block row (its diagonal block)
            const int* list = list_of(hl, mA);
            const int my_cnt = (x.cnt - s + 1) >> 1;   // blocks j = s, s + 2, ...
            // kB = 64: this stream's positions of the pair's union walk, with membership
            PairWalk w = walk_of(hl, mA, mB);
            int dummy;
            auto next_mine = [&](bool& mine) -> int {
                int mem;
                const int n = w.next(mem);
                w.next(dummy);                          // the other stream's position
                mine = (mem >> hp) & 1;
                return n;
            };
            if (kPair && s == 1) w.next(dummy);
            // dense (b = 128): blocks in DESCENDING order, so the two streams' first blocks — the
            // fixed softmax reference — are the diagonal and its neighbour, where a causal row's
            // largest scores usually sit (ascending, the sink-side reference let rows overflow 2^32
            // and re-run exactly: 11.7 of 117 ms at 128K)
            auto block_n = [&](int js) { return dense ? m - (2 * js + s) : __ldg(list + 2 * js + s); };
            float l = 0.f;
            float m_ref;
            if (!exact) {
                // reference = max of the two streams' first blocks (read twice from TMEM)
                float rmax = -INFINITY, rmax_u = -INFINITY;
                bool mine0 = true;
                int n0 = -1;
                if (my_cnt > 0) {
                    n0 = kPair ? next_mine(mine0) : block_n(0);
                    wait_s();
                    rmax_u = block_max(n0 == m);
                    rmax = mine0 ? rmax_u : -INFINITY;
                }
                m_ref = exchange_max(rmax, rmax_u);
                xhi = -INFINITY;
                if (my_cnt > 0) l = block_exps(m_ref, n0 == m, mine0);
                if (kPair) {
                    for (int js = 1; js < my_cnt; ++js) {
                        bool mine;
                        const int n = next_mine(mine);
                        wait_s();
                        l += block_exps(m_ref, n == m, mine);
                    }
                } else {
                    int n_next = (my_cnt > 1) ? block_n(1) : 0;
                    for (int js = 1; js < my_cnt; ++js) {
                        const int n = n_next;
                        if (js + 1 < my_cnt) n_next = block_n(js + 1);
                        wait_s();
                        l += block_exps(m_ref, n == m, true);
                    }
                }
#ifndef PA_X_ANY
                if (!(l <= exp2f(kOverflow)) || xhi > kOverflow) l = INFINITY;   // flag the row
#endif
            } else {
                // exact: the row's true max over its own blocks first (S only), then the fixed pass
                float tmax = -INFINITY;
                for (int js = 0; js < my_cnt; ++js) {
                    bool mine = true;
                    const int n = kPair ? next_mine(mine) : block_n(js);
                    wait_s();
                    if (mine) tmax = fmaxf(tmax, block_max(n == m));
                    release_s();
                }
                m_ref = exchange_max(tmax, tmax);
                if (kPair) {
                    w = walk_of(hl, mA, mB);
                    if (s == 1) w.next(dummy);
                }
                for (int js = 0; js < my_cnt; ++js) {
                    bool mine = true;
                    const int n = kPair ? next_mine(mine) : block_n(js);
                    wait_s();
                    l += block_exps(m_ref, n == m, mine);
                }
            }
            bars->lsum[it & 1][s][rr] = l;
            mbar_arrive(&bars->l_ready[it & 1]);
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

// kB = 64: union size of each row pair's two lists, |A| + |B| - |A n B| (a warp per work
// unit; B marked in a per-warp bitmap and A tested, or A's elements binary-searched in the
// ascending B when the bitmap does not fit).  Same item order as the kernel.
__global__ void pair_union_kernel(const int* __restrict__ block_cnt, const int* __restrict__ block_idx,
                                  int M, int r, int row_lo, int row_hi, int n_items, int* __restrict__ ucnt,
                                  int use_bitmap) {
    const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (item >= n_items) return;
    const int q_lo = row_lo >> 1, q_hi = (row_hi + 1) >> 1;
    const int per_kv = r * (q_hi - q_lo);
    const int rem = item % per_kv;
    const int hl = (item / per_kv) * r + rem % r;
    const int q = q_hi - 1 - rem / r;
    const int mA = (2 * q >= row_lo) ? 2 * q : -1, mB = (2 * q + 1 < row_hi) ? 2 * q + 1 : -1;
    const int ca = mA < 0 ? 0 : __ldg(block_cnt + static_cast<long long>(hl) * M + mA);
    const int cb = mB < 0 ? 0 : __ldg(block_cnt + static_cast<long long>(hl) * M + mB);
    int inter = 0;
    extern __shared__ unsigned pair_bits[];           // a (M+31)/32-word bitmap per warp, or none
    const int words = (M + 31) >> 5;
    if (ca > 0 && cb > 0 && use_bitmap) {
        // |A n B| by marking B's columns in a bitmap and testing A's: coalesced, independent loads
        const int* A = block_idx + (static_cast<long long>(hl) * M + mA) * M;
        const int* B = block_idx + (static_cast<long long>(hl) * M + mB) * M;
        unsigned* bm = pair_bits + (threadIdx.x >> 5) * words;
        const int nw = (mB >> 5) + 1;                  // B's columns are <= mB
        for (int w = lane; w < nw; w += 32) bm[w] = 0u;
        __syncwarp();
        for (int i = lane; i < cb; i += 32) {
            const int v = __ldg(B + i);
            atomicOr(bm + (v >> 5), 1u << (v & 31));
        }
        __syncwarp();
        for (int i = lane; i < ca; i += 32) {
            const int v = __ldg(A + i);
            inter += (bm[v >> 5] >> (v & 31)) & 1u;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    } else if (ca > 0 && cb > 0) {
        const int* A = block_idx + (static_cast<long long>(hl) * M + mA) * M;
        const int* B = block_idx + (static_cast<long long>(hl) * M + mB) * M;
        for (int i = lane; i < ca; i += 32) {
            const int v = __ldg(A + i);
            int lo = 0, hi = cb;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (__ldg(B + mid) < v) lo = mid + 1;
                else hi = mid;
            }
            inter += (lo < cb && __ldg(B + lo) == v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) inter += __shfl_xor_sync(0xffffffffu, inter, o);
    }
    if (lane == 0) ucnt[item] = ca + cb - inter;
}

// KV-head order of the persistent schedule: decreasing total selected blocks over the launch's
// rows (stable).  Items stay KV-head-major (a KV head's K/V stay hot in L2) while the
// heaviest rows of the launch are no longer left to the end when they belong to a late KV head
// (the tail that limited row-sharded launches at 8 ranks).  One CTA per KV head sums its
// counts; the last CTA to finish ranks the sums (kvsum / done live in the scheduler buffer,
// `done` returns to 0 for the next launch).
__global__ void __launch_bounds__(1024) kv_order_kernel(const int* __restrict__ block_cnt, int M, int r,
                                                        int row_lo, int row_hi, int n_kv,
                                                        long long* __restrict__ kvsum, int* __restrict__ done,
                                                        int* __restrict__ kvperm) {
    __shared__ long long warp_part[32];
    __shared__ bool last;
    const int kv = blockIdx.x;
    long long acc = 0;
    for (int h = kv * r; h < (kv + 1) * r; ++h)
        for (int m = row_lo + threadIdx.x; m < row_hi; m += blockDim.x)
            acc += __ldg(block_cnt + static_cast<long long>(h) * M + m);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) warp_part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += warp_part[w];
        kvsum[kv] = t;
        __threadfence();
        last = atomicAdd(done, 1) == n_kv - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < n_kv) {
        const int me = threadIdx.x;
        const long long tm = *(volatile long long*)(kvsum + me);
        int rank = 0;
        for (int j = 0; j < n_kv; ++j) {
            const long long tj = *(volatile long long*)(kvsum + j);
            rank += (tj > tm) || (tj == tm && j < me);
        }
        kvperm[rank] = me;
    }
    if (threadIdx.x == 0) *done = 0;
}

// Per-(device, stream) scheduler state + flagged-row list + kB = 64 union counts.  A launch
// captured into a CUDA graph keeps these pointers in its kernel parameters, so a buffer is
// NEVER freed: when a larger launch needs more room, the old arrays are retired (kept
// allocated until exit) and new ones are made.  Graphs captured on one stream share the
// `sched` counters: replay them one at a time on that stream (stream order serialises them).
struct SchedBuf {
    Sched* sched = nullptr;
    int* flagged = nullptr;
    int* ucnt = nullptr;
    int* kvperm = nullptr;   // [64]
    long long* kvsum = nullptr;   // [64]
    int* kvdone = nullptr;
    size_t cap = 0;
};

SchedBuf* sched_for(cudaStream_t st, size_t n_items) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, SchedBuf> bufs;
    static std::vector<void*> retired;   // superseded arrays a captured graph may still use
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    SchedBuf& b = bufs[{dev, st}];
    if (!b.sched && cudaMalloc(&b.sched, sizeof(Sched)) != cudaSuccess) return nullptr;
    if (!b.kvperm) {
        if (cudaMalloc(&b.kvperm, 64 * sizeof(int)) != cudaSuccess) return nullptr;
        if (cudaMalloc(&b.kvsum, 64 * sizeof(long long)) != cudaSuccess) return nullptr;
        if (cudaMalloc(&b.kvdone, sizeof(int)) != cudaSuccess) return nullptr;
        if (cudaMemset(b.kvdone, 0, sizeof(int)) != cudaSuccess) return nullptr;
    }
    if (b.cap < n_items) {   // each row can be appended by up to 4 epilogue warps
        int* fl = nullptr;
        int* uc = nullptr;
        const size_t cap = std::max(n_items, 2 * b.cap);
        if (cudaMalloc(&fl, 4 * cap * sizeof(int)) != cudaSuccess) return nullptr;
        if (cudaMalloc(&uc, cap * sizeof(int)) != cudaSuccess) {
            cudaFree(fl);
            return nullptr;
        }
        if (b.flagged) retired.push_back(b.flagged);
        if (b.ucnt) retired.push_back(b.ucnt);
        b.flagged = fl;
        b.ucnt = uc;
        b.cap = cap;
    }
    return &b;
}

using AttnKernel = void (*)(const CUtensorMap, const CUtensorMap, const CUtensorMap, __nv_bfloat16*,
                            const int*, const int*, int, int, int, float, int, int, int, Sched*, int*,
                            int, long long, long long, const int*, const int*, const SeqDesc*, int);

template <int kD, int kB, int kEmu, bool kVar = false>
AttnKernel kernel_with_attr() {
    if (ensure_smem_attr(reinterpret_cast<const void*>(attn_tc8_kernel<kEmu, kD, kB, kVar>),
                         static_cast<int>(Shape<kD, kB>::kSmem)) != cudaSuccess)
        return nullptr;
    return attn_tc8_kernel<kEmu, kD, kB, kVar>;
}

}  // namespace

namespace {
cudaError_t launch_tc8(const Dims& D, const void* Q, const void* K, const void* V, const int* block_cnt,
                       const int* block_idx, void* O, cudaStream_t st, const SeqDesc* seqs, int n_seqs,
                       int varlen_items) {
    if (!((D.d == 64 || D.d == 128) && (D.b == 64 || D.b == 128))) return cudaErrorInvalidValue;
    if (n_seqs > 0 && (D.b != 128 || !block_cnt)) return cudaErrorInvalidValue;   // varlen: sparse, b = 128
    CUtensorMap mq, mk, mv;
    if (!make_map_bf16_sw128_3d(&mq, Q, D.Hl, D.N, D.q_ts, D.q_hs, 128, D.d) ||
        !make_map_bf16_sw128_3d(&mk, K, D.Hkvl, D.N, D.kv_ts, D.kv_hs, D.b, D.d) ||
        !make_map_bf16_sw128_3d(&mv, V, D.Hkvl, D.N, D.kv_ts, D.kv_hs, D.b, D.d))
        return cudaErrorInvalidValue;
    // Exp2 split (of every 8 key-column pairs, kEmu on the FMA-pipe polynomial), measured at
    // 128K: d = 128 all-MUFU (under the power cap 18.84-18.94 ms vs 18.85-19.06 at 1/8 and
    // 19.18-19.28 at 2/8); d = 64 (exp-bound: half the tensor work per exp2) 2/8 (13.2-13.3 ms
    // vs 13.4-13.6 at 3/8 and 13.8 at 4/8); b = 64 all-MUFU.
    AttnKernel kern = nullptr;
    constexpr int e128 = PA_EMU_D128, e64 = PA_EMU_D64, eb64 = PA_EMU_B64;
    if (n_seqs > 0) {          // varlen instantiations (b = 128; d = 128 is attn_tc9's)
#if PA_ATTN_V9
        kern = D.d == 128 ? nullptr : kernel_with_attr<64, 128, e64, true>();
#else
        kern = D.d == 128 ? kernel_with_attr<128, 128, e128, true>() : kernel_with_attr<64, 128, e64, true>();
#endif
    }
    else if (D.d == 128)
#if PA_ATTN_V9 && PA_ATTN_V9_DENSE
        kern = D.b == 128 ? nullptr : kernel_with_attr<128, 64, eb64>();   // d = b = 128: attn_tc9
#else
        kern = D.b == 128 ? kernel_with_attr<128, 128, e128>() : kernel_with_attr<128, 64, eb64>();
#endif
    else
        kern = D.b == 128 ? kernel_with_attr<64, 128, e64>() : kernel_with_attr<64, 64, e64>();
    if (!kern) return cudaErrorInvalidValue;
    int dev = 0, n_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    const bool pair = D.b == 64;
    // work units: (head, block row), or (head, row pair) for b = 64
    const int nrows = pair ? (D.re + 1) / 2 - D.rb / 2 : D.re - D.rb;
    const size_t n_items = n_seqs > 0 ? static_cast<size_t>(varlen_items)
                                      : static_cast<size_t>(D.Hl) * static_cast<size_t>(nrows);
    SchedBuf* sb = sched_for(st, n_items);
    if (!sb) return cudaErrorMemoryAllocation;
    cudaError_t e = cudaMemsetAsync(sb->sched, 0, sizeof(Sched), st);
    if (e != cudaSuccess) return e;
    if (pair && block_cnt) {
        // bitmap intersection while 8 warps' bitmaps fit in 16 KB (M <= 16384), else binary search
        const int words = (D.M + 31) / 32;
        const bool bitmap = words * 8 * 4 <= 16384;
        pair_union_kernel<<<static_cast<unsigned>((n_items * 32 + 255) / 256), 256,
                            bitmap ? static_cast<size_t>(words) * 8 * 4 : 0, st>>>(
            block_cnt, block_idx, D.M, D.r, D.rb, D.re, static_cast<int>(n_items), sb->ucnt, bitmap ? 1 : 0);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // KV heads in decreasing work (sparse launches with more than one local KV head, <= 64)
    const int* kvperm = nullptr;
    if (block_cnt && n_seqs == 0 && D.Hkvl > 1 && D.Hkvl <= 64) {
        kv_order_kernel<<<D.Hkvl, 1024, 0, st>>>(block_cnt, D.M, D.r, D.rb, D.re, D.Hkvl, sb->kvsum,
                                                 sb->kvdone, sb->kvperm);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        kvperm = sb->kvperm;
    }
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D.d));
    const size_t smem = D.d == 128 ? (D.b == 128 ? Shape<128, 128>::kSmem : Shape<128, 64>::kSmem)
                                   : (D.b == 128 ? Shape<64, 128>::kSmem : Shape<64, 64>::kSmem);
    // fast launch over every row, then the exact launch over the rows it flagged (usually
    // none: its CTAs find an empty list and exit)
    for (int exact = 0; exact < 2; ++exact) {
        const int grid = exact ? n_sm : static_cast<int>(n_items < static_cast<size_t>(n_sm) ? n_items : n_sm);
        kern<<<grid, kThreads, smem, st>>>(
            mq, mk, mv, static_cast<__nv_bfloat16*>(O), block_cnt, block_idx, static_cast<int>(D.N),
            D.M, D.r, scale_log2, D.rb, D.re, static_cast<int>(n_items), sb->sched, sb->flagged, exact,
            D.q_hs, D.q_ts, sb->ucnt, kvperm, seqs, n_seqs);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

}  // namespace

// Shared with attn_tc9.cu: the per-(device, stream) scheduler state for a launch pair of
// n_items work units, zeroed on `st`, and (sparse, 1 < Hkvl <= 64) the KV-head order over the
// launch's rows.  Returns the device pointers through the out-parameters.
cudaError_t attn_sched_prepare(const Dims& D, const int* block_cnt, size_t n_items, cudaStream_t st,
                               void** sched, int** flagged, const int** kvperm) {
    SchedBuf* sb = sched_for(st, n_items);
    if (!sb) return cudaErrorMemoryAllocation;
    cudaError_t e = cudaMemsetAsync(sb->sched, 0, sizeof(Sched), st);
    if (e != cudaSuccess) return e;
    *kvperm = nullptr;
    if (block_cnt && D.Hkvl > 1 && D.Hkvl <= 64) {
        kv_order_kernel<<<D.Hkvl, 1024, 0, st>>>(block_cnt, D.M, D.r, D.rb, D.re, D.Hkvl, sb->kvsum,
                                                 sb->kvdone, sb->kvperm);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        *kvperm = sb->kvperm;
    }
    *sched = sb->sched;
    *flagged = sb->flagged;
    return cudaSuccess;
}

cudaError_t launch_attn_tc8(const Dims& D, const void* Q, const void* K, const void* V,
                            const int* block_cnt, const int* block_idx, void* O, cudaStream_t st) {
    return launch_tc8(D, Q, K, V, block_cnt, block_idx, O, st, nullptr, 0, 0);
}

namespace {
struct DescChunk {
    SeqDesc d[64];
    int n;
};
__global__ void write_descs_kernel(SeqDesc* dst, const __grid_constant__ DescChunk c) {
    if (static_cast<int>(threadIdx.x) < c.n) dst[threadIdx.x] = c.d[threadIdx.x];
}
}  // namespace

cudaError_t write_seq_descs(SeqDesc* dst, const SeqDesc* host, int n, cudaStream_t st) {
    for (int i = 0; i < n; i += 64) {
        DescChunk c{};
        c.n = n - i < 64 ? n - i : 64;
        for (int k = 0; k < c.n; ++k) c.d[k] = host[i + k];
        write_descs_kernel<<<1, 64, 0, st>>>(dst + i, c);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_attn_tc8_varlen(const Dims& D, const void* Q, const void* K, const void* V,
                                   const int* block_cnt, const int* block_idx, void* O,
                                   const SeqDesc* seqs, int n_seqs, int n_items, cudaStream_t st) {
    return launch_tc8(D, Q, K, V, block_cnt, block_idx, O, st, seqs, n_seqs, n_items);
}

}  // namespace pa
