// attn_tc7.cu — bf16 block-sparse causal prefill attention on tcgen05 (A7 / A8), variant v7:
// one (head, query block row) per CTA, its key blocks split into two streams (even / odd list
// positions) that accumulate into ONE shared O with a per-row reference max that is FIXED
// for the whole row.  Fixing the reference removes the online rescale, so the two streams
// can share O, which frees TMEM for separate P buffers: an S buffer is released as soon as
// the softmax has loaded it and the next S of that stream is issued while the softmax is
// still computing P.  Nothing in the per-stream chain waits for the PV of the same block.
//
// Method: O[h][t] = sum over keys k of the selected blocks, k <= t, of
// softmax(Q[h][t] K[kv(h)][k] / sqrt(d)) V[kv(h)][k].
// softmax is shift invariant: P = 2^(x - m_ref), x = s log2(e)/sqrt(d), O = sum P V / sum P
// for ANY per-row m_ref, as long as nothing overflows.  Pass 0 takes m_ref = the row max of
// the first block of each stream (an attained value, so sum P >= 1); if a later block
// exceeds m_ref by more than kOverflow (2^32 bounds P, sum P <= 2^49, no fp32/bf16 overflow)
// the CTA sets a flag and re-runs the row (pass 1) with m_ref = the exact row max gathered in
// pass 0, where x <= m_ref always holds.  Pass 1 is for adversarial score ranges only.
//
// Warp roles (384 threads):
//   warp 0      TMA producer of Q and K (4-stage ring)
//   warp 1      TMEM allocator + S issuer: S_{j&1} = Q K_j^T once the softmax of block j-2
//               has loaded S_{j&1} (s_free) and K_j has landed
//   warp 2      PV issuer: O += P_{j&1} V_j per P half as soon as it is released
//   warp 3      TMA producer of V (2-stage ring)
//   warps 4-7   softmax of stream 0, warps 8-11 of stream 1 (thread = query row = TMEM lane):
//               tcgen05.ld S, release S, mask, 8-chain max, exp2 (MUFU + FMA-pipe poly),
//               P (bf16) into the stream's own P buffer in two halves
// TMEM (512 columns): O [0,128)  S_0 [128,256)  S_1 [256,384)  P_0 [384,448)  P_1 [448,512).
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
constexpr int kKStages = 4;
constexpr int kVStages = 2;
constexpr int kThreads = 384;
constexpr float kOverflow = 32.0f;         // log2 headroom of P over the pass-0 reference

constexpr uint32_t kColO = 0, kColS = 128, kColP = 384;

struct __align__(8) Bars7 {
    uint64_t q_full;
    uint64_t k_full[kKStages];
    uint64_t k_empty[kKStages];
    uint64_t v_full[kVStages];
    uint64_t v_empty[kVStages];
    uint64_t s_full[2];
    uint64_t s_free[2];
    uint64_t p_full[2][2];   // [stream][half]
    uint64_t p_free[2];
    uint64_t o_final;
    uint32_t tmem_base;
    int overflow;
    float red[2][128];       // per-stream row values exchanged between the streams
};

constexpr size_t kSmemBytes = 1024 + kTile * (1 + kKStages + kVStages) + sizeof(Bars7);
static_assert(kSmemBytes <= 232448, "shared memory budget");

__device__ __forceinline__ void softmax_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int kEmu>   // of every 8 key-column pairs, kEmu use the FMA-pipe exp2 (ex2_poly2)
__global__ void __launch_bounds__(kThreads, 1)
attn_tc7_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ O,
                const int* __restrict__ block_cnt, const int* __restrict__ block_idx, int N, int M,
                int r, float scale_log2, int row_lo, int row_hi, long long* trace, int trace_bid,
                long long* cta_times) {
    long long t_start = 0;
    if (cta_times && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTile;
    uint8_t* sV = smem + kTile * (1 + kKStages);
    Bars7* bars = reinterpret_cast<Bars7*>(smem + kTile * (1 + kKStages + kVStages));

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
            mbar_init(&bars->s_free[s], 128);
            mbar_init(&bars->p_full[s][0], 128);
            mbar_init(&bars->p_full[s][1], 128);
            mbar_init(&bars->p_free[s], 1);
        }
        mbar_init(&bars->o_final, 1);
        bars->overflow = 0;
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(&bars->tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = bars->tmem_base;

    // Passes: 0 = fixed reference from the first blocks; only if pass 0 overflowed (flag):
    // 1 = max sweep (S and row max only, no P / PV), 2 = full pass with the exact row max.
    // Ring / barrier phases continue across passes through per-role block counters.
    const int cnt_s[2] = {(cnt + 1) >> 1, cnt >> 1};   // blocks of stream 0 / 1

    if (warp < 4) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 56;\n" ::: "memory");
      for (int pass = 0; pass < 3; ++pass) {
        const bool pv_pass = (pass != 1);
        if (warp == 0) {
            // ------------------------------------------------------- K producer --
            if (lane == 0) {
                if (pass == 0) {
                    tma_prefetch(&tmQ);
                    tma_prefetch(&tmK);
                    const int qrow = hl * N + m * kTileRows;
                    mbar_expect_tx(&bars->q_full, kTile);
                    tma_load_2d(sQ, &tmQ, &bars->q_full, 0, qrow);
                    tma_load_2d(sQ + kBox, &tmQ, &bars->q_full, 64, qrow);
                }
                for (int j = 0; j < cnt; ++j) {
                    const int g = pass * cnt + j;
                    const int st = g % kKStages;
                    if (g >= kKStages) mbar_wait(&bars->k_empty[st], ((g / kKStages) - 1) & 1);
                    const int n = dense ? j : __ldg(list + j);
                    const int krow = kvl * N + n * kTileRows;
                    mbar_expect_tx(&bars->k_full[st], kTile);
                    tma_load_2d(sK + st * kTile, &tmK, &bars->k_full[st], 0, krow);
                    tma_load_2d(sK + st * kTile + kBox, &tmK, &bars->k_full[st], 64, krow);
                }
            }
        } else if (warp == 3) {
            // ------------------------------------------------------- V producer --
            if (lane == 0 && pv_pass) {
                if (pass == 0) tma_prefetch(&tmV);
                for (int j = 0; j < cnt; ++j) {
                    const int g = (pass == 2 ? cnt : 0) + j;
                    const int st = g % kVStages;
                    if (g >= kVStages) mbar_wait(&bars->v_empty[st], ((g / kVStages) - 1) & 1);
                    const int n = dense ? j : __ldg(list + j);
                    const int vrow = kvl * N + n * kTileRows;
                    mbar_expect_tx(&bars->v_full[st], kTile);
                    tma_load_2d(sV + st * kTile, &tmV, &bars->v_full[st], 0, vrow);
                    tma_load_2d(sV + st * kTile + kBox, &tmV, &bars->v_full[st], 64, vrow);
                }
            }
        } else if (warp == 1) {
            // -------------------------------------------------------- S issuer --
            constexpr uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
            const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
            const uint64_t dk = sdesc_sw128(smem_u32(sK), 16, 1024);
            const bool leader = elect_one();
            if (pass == 0) mbar_wait(&bars->q_full, 0);
            for (int j = 0; j < cnt; ++j) {
                const int g = pass * cnt + j;
                const int s = j & 1;
                const int gs = pass * cnt_s[s] + (j >> 1);          // stream block counter
                if (gs > 0) mbar_wait(&bars->s_free[s], (gs - 1) & 1);
                const int st = g % kKStages;
                mbar_wait(&bars->k_full[st], (g / kKStages) & 1);
                tc_fence_after();
                if (leader) {
                    const uint64_t b0 = dk + (st * kTile >> 4);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const uint32_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
                        umma_ss(tbase + kColS + s * 128, dq + off, b0 + off, idesc_qk, kk > 0 ? 1u : 0u);
                    }
                    tc_commit(&bars->k_empty[st]);
                    tc_commit(&bars->s_full[s]);
                }
                __syncwarp();
            }
        } else if (warp == 2 && pv_pass) {
            // ------------------------------------------------------- PV issuer --
            constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
            const uint64_t dv = sdesc_sw128(smem_u32(sV), kBox, 1024);
            const bool leader = elect_one();
            for (int j = 0; j < cnt; ++j) {
                const int g = (pass == 2 ? cnt : 0) + j;
                const int s = j & 1;
                const int gs = (pass == 2 ? cnt_s[s] : 0) + (j >> 1);
                const int st = g % kVStages;
                long long* tr = (trace && blockIdx.x == trace_bid && j < 512 && leader && pass == 0)
                                    ? trace + j * 8 : nullptr;
                if (tr) tr[0] = clock64();                         // PV: start waiting for V, P
                mbar_wait(&bars->v_full[st], (g / kVStages) & 1);
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    mbar_wait(&bars->p_full[s][half], gs & 1);
                    if (tr) tr[1 + half] = clock64();              // PV: P half ready
                    tc_fence_after();
                    if (leader) {
                        const uint64_t b0 = dv + (st * kTile >> 4);
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {
                            const int kk = half * 4 + k4;
                            umma_ts(tbase + kColO, tbase + kColP + s * 64 + kk * 8, b0 + (kk * 2048 >> 4),
                                    idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
                        }
                    }
                    __syncwarp();
                }
                if (leader) {
                    tc_commit(&bars->v_empty[st]);
                    tc_commit(&bars->p_free[s]);
                }
                __syncwarp();
                if (tr) tr[3] = clock64();                         // PV: issued
            }
            if (leader) tc_commit(&bars->o_final);
            __syncwarp();
        }
        __syncthreads();
        if (pass == 2 || !bars->overflow) break;
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 216;\n" ::: "memory");
      // ------------------------------------------------------------ softmax --
      const int s = (warp - 4) >> 2;                  // stream
      const int quarter = warp & 3;
      const int rr = quarter * 32 + lane;
      const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
      const uint32_t tS = tbase + lane_off + kColS + s * 128;
      const uint32_t tP = tbase + lane_off + kColP + s * 64;
      const int my_cnt = cnt_s[s];                    // blocks j = s, s + 2, ...
      const uint64_t sc2 = f2_pack(scale_log2, scale_log2);
      float m_ref = 0.f;
      float l = 0.f;
      float xhi = -INFINITY;                          // max exponent seen by the FMA-pipe exp2

      // P = 2^(S log2e/sqrt(d) - m_ref) of one 32-column chunk (diagonal mask applied by the
      // caller), row sum into ls, bf16 pairs into the P buffer (16 columns).
      auto p_chunk = [&](const uint32_t (&x)[32], uint64_t nm2, uint64_t (&ls)[4], uint32_t tdst,
                         int wait_gp = 0) {
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
                  p0 = ex2(x0);
                  p1 = ex2(x1);
              }
              ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
              pk[p] = pack_bf16(p0, p1);
          }
          if (wait_gp > 0) {                            // the previous PV has read P_s
              mbar_wait(&bars->p_free[s], (wait_gp - 1) & 1);
              tc_fence_after();
          }
          tmem_st16(tdst, pk);
      };
      auto mask_chunk = [&](uint32_t (&x)[32], int c) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
              if (c * 32 + e > rr) x[e] = 0xff800000u;
      };
      auto release_p = [&](int half) {
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bars->p_full[s][half]);
      };
      auto add_l = [&](uint64_t (&ls)[4]) {
          const uint64_t t = f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3]));
          float a, b;
          f2_unpack(t, a, b);
          l += a + b;
      };
      // one block with the reference known: chunked TMEM loads overlapped with the exps
      auto block_fixed = [&](int gs, int gp, bool diag) {
          mbar_wait(&bars->s_full[s], gs & 1);
          tc_fence_after();
          const uint64_t nm2 = f2_pack(-m_ref, -m_ref);
          uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
          uint32_t xa[32], xb[32];
          tmem_ld32(tS, xa);
          tmem_ld_wait_regs(xa);
          tmem_ld32(tS + 32, xb);
          if (diag) mask_chunk(xa, 0);
          p_chunk(xa, nm2, ls, tP, gp);
          tmem_ld_wait_regs(xb);
          tmem_ld32(tS + 64, xa);
          if (diag) mask_chunk(xb, 1);
          p_chunk(xb, nm2, ls, tP + 16);
          release_p(0);
          tmem_ld_wait_regs(xa);
          tmem_ld32(tS + 96, xb);
          if (diag) mask_chunk(xa, 2);
          p_chunk(xa, nm2, ls, tP + 32);
          tmem_ld_wait_regs(xb);
          tc_fence_before();
          mbar_arrive(&bars->s_free[s]);                // S buffer free for block j+2
          if (diag) mask_chunk(xb, 3);
          p_chunk(xb, nm2, ls, tP + 48);
          release_p(1);
          add_l(ls);
      };
      // one block loaded whole: row max (all 128 columns), S released; P optional
      auto block_max = [&](int gs, bool diag, uint32_t (&raw)[4][32]) -> float {
          mbar_wait(&bars->s_full[s], gs & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 4; ++c) tmem_ld32(tS + c * 32, raw[c]);
          tmem_ld_wait();
          tc_fence_before();
          mbar_arrive(&bars->s_free[s]);
          if (diag) {
#pragma unroll
              for (int c = 0; c < 4; ++c) mask_chunk(raw[c], c);
          }
          float mx[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) mx[k] = __uint_as_float(raw[k >> 1][(k & 1) * 16]);
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int e = 0; e < 32; ++e)
                  mx[c * 2 + (e >> 4)] = fmaxf(mx[c * 2 + (e >> 4)], __uint_as_float(raw[c][e]));
          return fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      };
      auto block_n = [&](int js) { return dense ? 2 * js + s : __ldg(list + 2 * js + s); };
      auto exchange_max = [&](float v) {
          bars->red[s][rr] = v;
          softmax_bar();
          const float r = fmaxf(bars->red[0][rr], bars->red[1][rr]) * scale_log2;
          softmax_bar();
          return r;
      };

      // ---- pass 0: reference = max of the two streams' first blocks
      {
          uint32_t raw[4][32];
          float rmax = -INFINITY;
          if (my_cnt > 0) {
              long long* tr = (trace && blockIdx.x == trace_bid && lane == 0 && quarter == 2)
                                  ? trace + 512 * 8 + s * 8 : nullptr;
              if (tr) tr[1] = clock64();
              rmax = block_max(0, block_n(0) == m, raw);
              if (tr) tr[2] = clock64();
          }
          m_ref = exchange_max(rmax);
          if (my_cnt > 0) {
              const uint64_t nm2 = f2_pack(-m_ref, -m_ref);
              uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
              p_chunk(raw[0], nm2, ls, tP);
              p_chunk(raw[1], nm2, ls, tP + 16);
              release_p(0);
              p_chunk(raw[2], nm2, ls, tP + 32);
              p_chunk(raw[3], nm2, ls, tP + 48);
              release_p(1);
              add_l(ls);
          }
          int n_next = (my_cnt > 1) ? block_n(1) : 0;
          for (int js = 1; js < my_cnt; ++js) {
              const int n = n_next;
              if (js + 1 < my_cnt) n_next = block_n(js + 1);
              long long* tr = (trace && blockIdx.x == trace_bid && lane == 0 && quarter == 2 && js < 256)
                                  ? trace + 512 * 8 + (js * 2 + s) * 8 : nullptr;
              if (tr) tr[0] = clock64();
              block_fixed(js, js, n == m);
              if (tr) tr[4] = clock64();
          }
          // P <= 2^kOverflow for every element <=> safe; a larger (or non-finite) row sum, or
          // a polynomial exp2 argument above the bound, means some block exceeded the
          // reference: redo the row exactly
          if (!(l <= exp2f(kOverflow)) || xhi > kOverflow) bars->overflow = 1;
      }
      __syncthreads();
      if (bars->overflow) {
          // ---- pass 1: exact row max over the stream's blocks (S only)
          float tmax = -INFINITY;
          for (int js = 0; js < my_cnt; ++js) {
              uint32_t raw[4][32];
              tmax = fmaxf(tmax, block_max(my_cnt + js, block_n(js) == m, raw));
          }
          m_ref = exchange_max(tmax);
          __syncthreads();
          // ---- pass 2: full pass with the exact reference (x <= m_ref: no overflow)
          l = 0.f;
          for (int js = 0; js < my_cnt; ++js) block_fixed(2 * my_cnt + js, my_cnt + js, block_n(js) == m);
          __syncthreads();
      }

      // ----------------------------------------------------------- epilogue --
      bars->red[s][rr] = l;
      softmax_bar();
      const float inv = 1.f / (bars->red[0][rr] + bars->red[1][rr]);
      mbar_wait(&bars->o_final, bars->overflow ? 1 : 0);
      tc_fence_after();
      const bool row_valid = static_cast<long long>(m) * kTileRows + rr < N;
      uint4* dst = reinterpret_cast<uint4*>(
          O + (static_cast<long long>(hl) * N + static_cast<long long>(m) * kTileRows + rr) * 128 + s * 64);
      uint32_t o[2][32];
      tmem_ld32(tbase + lane_off + kColO + s * 64, o[0]);
      tmem_ld32(tbase + lane_off + kColO + s * 64 + 32, o[1]);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 2; ++c) {
          uint32_t pkd[16];
#pragma unroll
          for (int e = 0; e < 16; ++e)
              pkd[e] = pack_bf16(__uint_as_float(o[c][2 * e]) * inv, __uint_as_float(o[c][2 * e + 1]) * inv);
          if (row_valid) {
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
    if (cta_times && threadIdx.x == 0) {   // diagnostics: per-CTA [start, end, sm, blocks]
        long long t_end;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        long long* c = cta_times + 4ll * blockIdx.x;
        c[0] = t_start;
        c[1] = t_end;
        c[2] = smid;
        c[3] = cnt + (bars->overflow ? 1 << 20 : 0);
    }
}

}  // namespace

cudaError_t launch_attn_tc7(const Dims& D, const void* Q, const void* K, const void* V,
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
    auto kern = emu == 0 ? attn_tc7_kernel<0> : emu == 1 ? attn_tc7_kernel<1>
              : emu == 2 ? attn_tc7_kernel<2> : emu == 3 ? attn_tc7_kernel<3> : attn_tc7_kernel<4>;
    static bool attr_set[5] = {false, false, false, false, false};
    if (!attr_set[emu]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(kSmemBytes));
        if (e != cudaSuccess) return e;
        attr_set[emu] = true;
    }
    // PROXYATTN_TRACE=<cta>: per-event clock64 timeline of one CTA (diagnostics only), read
    // back with proxyattn_debug_trace(): [512 j][8] PV-issuer events, then [256 js][2 s][8].
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
    // PROXYATTN_CTA_TIMES=1: per-CTA [start ns, end ns, SM, blocks (+2^20 if re-run)] of the
    // last launch, read back with proxyattn_debug_trace() (diagnostics only).
    static long long* cta_times = nullptr;
    static size_t cta_cap = 0;
    const size_t ncta = static_cast<size_t>(D.Hl) * static_cast<size_t>(D.re - D.rb);
    if (!trace && getenv("PROXYATTN_CTA_TIMES")) {
        if (cta_cap < ncta) {
            if (cta_times) cudaFree(cta_times);
            cta_times = nullptr;
            if (cudaMalloc(&cta_times, ncta * 4 * sizeof(long long)) == cudaSuccess) cta_cap = ncta;
        }
        attn_trace_ptr() = cta_times;
    }
    const float scale_log2 = kLog2e / sqrtf(static_cast<float>(D.d));
    const unsigned grid = static_cast<unsigned>(D.Hl) * static_cast<unsigned>(D.re - D.rb);
    kern<<<grid, kThreads, kSmemBytes, st>>>(mq, mk, mv, static_cast<__nv_bfloat16*>(O), block_cnt,
                                             block_idx, static_cast<int>(D.N), D.M, D.r, scale_log2,
                                             D.rb, D.re, trace, trace_bid,
                                             (!trace && cta_times) ? cta_times : nullptr);
    return cudaGetLastError();
}

}  // namespace pa
