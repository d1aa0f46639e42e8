/*
 * proxyattn.h — C-ABI of libproxyattn, the B200 (sm_100a) hot path of ProxyAttn
 * (arXiv 2509.24745, "ProxyAttn: Guided Sparse Attention via Representative Heads").
 *
 * Citations: P:<line> = PAPER.md line (section / equation), S:<line> = SPEC.md line.
 * Steps A1-A8 are SURVEY.md §8(a); readings Z1-Z24 are listed in DESIGN.md.
 *
 * Conventions (every entry point):
 *  - All tensor pointers are caller-owned DEVICE memory (e.g. torch tensors), 16-byte
 *    aligned.  Default layout is head-major and contiguous: Q [Hl][N][d], K/V [Hkv_l][N][d],
 *    O [Hl][N][d], where Hl = q_head_end - q_head_begin is the local query-head shard and
 *    Hkv_l = Hl / r (r = Hq/Hkv) the kv heads it uses, starting at kv head q_head_begin / r.
 *    With PROXYATTN_FLAG_TOKEN_MAJOR the layout is token-major with a token stride (the
 *    packed [tokens][heads][d] layout of serving engines): element (local head h, token t,
 *    i) of Q / O is at Q[t * q_token_stride + h * d + i], of K / V at
 *    K[t * kv_token_stride + h_kv * d + i]; Q, O, K, V point at the first LOCAL head.
 *    Strides 0 mean the packed defaults Hl * d and Hkv_l * d.
 *  - Element type: bf16 (__nv_bfloat16) by default; fp32 when PROXYATTN_FLAG_FP32_DEBUG.
 *  - Per-head outputs (kstar, budget, block_cnt, block_idx) are indexed by local head.
 *  - All work is enqueued on `stream` (a cudaStream_t, passed as void*); no call
 *    synchronises the host except proxyattn_forward_host and the validation flags
 *    (PROXYATTN_FLAG_CHECK, PROXYATTN_FLAG_CHECK_FINITE).  proxyattn_estimate forks Alg. 1
 *    onto a library-owned helper stream and joins it back to `stream` by events before
 *    returning, so its completion is still ordered on `stream` and the call is capturable
 *    in a CUDA graph.  Helper streams are created once per (device, caller stream): calls
 *    from different threads on different streams never share one.
 *  - Scratch comes from the caller's workspace.  The only memory the library allocates is
 *    the attention launch's scheduler state, once per (device, stream) on the first
 *    prefill / forward on that stream (work counter, KV-head order, the exact-launch row
 *    list: 20 bytes per work item).  When a later launch on that stream needs more items,
 *    new arrays are made and the old ones are kept (never freed while the process lives),
 *    so a graph captured earlier keeps valid pointers.  Hence CUDA-graph capture: make one
 *    call on the capture stream first (as bench.py and tests/test_gpu_graphs.py do); every
 *    call is then asynchronous and capturable, including proxyattn_forward_varlen.  Graphs
 *    captured on one stream share its work counter: replay them in that stream's order, not
 *    concurrently on other streams.
 *  - Return codes: PROXYATTN_OK or one of the negative PROXYATTN_E_* codes; a
 *    human-readable reason is available from proxyattn_last_error() (thread-local).
 *    Validation errors are raised before anything is enqueued.
 *  - Determinism: identical inputs give bit-identical outputs (no float atomics,
 *    fixed reduction orders).
 */
#ifndef PROXYATTN_H
#define PROXYATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- config -- */

/* AttnConfig.  Invariants: Hq % Hkv == 0, Hkv % g == 0, b % s == 0,
 * 0 < gamma <= 1, min_budget_tokens >= 0.  N need not be a multiple of b: M = ceil(N/b)
 * blocks, the last one zero-padded with its padded keys masked and no output for padded
 * rows; sampled positions are i*s < N, N/s rounded up.
 * bf16 build supports d in {64, 128} and b in {64, 128} (tcgen05 kernels; the estimation's
 * tensor-core passes also need b/s in {16, 32, 64, 128}, else SIMT kernels run them);
 * FP32_DEBUG supports d % 32 == 0, d <= 128, any b with b % s == 0 (SIMT kernels, for the
 * 1e-4 parity contract). */
typedef struct {
    int32_t  n_q_heads;          /* Hq (global) */
    int32_t  n_kv_heads;         /* Hkv (global) */
    int32_t  head_dim;           /* d */
    int64_t  seq_len;            /* N; ceil(N / b) <= 16384 block rows (A4/A6 sort a row in
                                    shared memory), else PROXYATTN_E_UNSUPPORTED */
    int32_t  block_size;         /* b (Z18) */
    int32_t  stride;             /* s, strided q/k sampling */
    int32_t  n_groups;           /* g, proxy heads */
    float    gamma;              /* cumulative threshold of Alg. 1 */
    int32_t  min_budget_tokens;  /* per-row floor ceil(tokens/b) blocks (Z13/Z14) */
    uint32_t flags;              /* PROXYATTN_FLAG_* */
    int32_t  q_head_begin;       /* local shard [begin, end) of query heads; end == 0 means all */
    int32_t  q_head_end;
    int32_t  static_kstar;       /* > 0: static top-K baseline (Fig. 6c): every head uses
                                    K* = static_kstar instead of Alg. 1's dynamic budget; 0 = Alg. 1 */
    int32_t  row_begin;          /* prefill / dense_prefill / estimate / select: compute query
                                    block rows [row_begin, row_end) only (row_end == 0: all rows);
                                    other rows of O / block_cnt / block_idx are left untouched
                                    (zig-zag row sharding); kstar / budget always
                                    cover every local head */
    int32_t  row_end;
    int64_t  q_token_stride;     /* TOKEN_MAJOR only: elements between consecutive tokens of Q / O
                                    (>= Hl * d, a multiple of 8; 0 = Hl * d) */
    int64_t  kv_token_stride;    /* TOKEN_MAJOR only: the same for K / V (>= Hkv_l * d; 0 = Hkv_l * d) */
} proxyattn_cfg;

#define PROXYATTN_FLAG_FP32_DEBUG  0x1u  /* fp32 Q/K/V/O, SIMT FFMA kernels (1e-4 contract)   */
#define PROXYATTN_FLAG_CHECK       0x2u  /* prefill validates block lists on the device (E_SHAPE) */
/* Method variants (readings Z1, Z12, Z16), off by default: */
#define PROXYATTN_FLAG_FORCE_SINK  0x4u  /* block 0 always selected, counted toward K (Z16 alternative) */
#define PROXYATTN_FLAG_CONSTANT_K  0x8u  /* Eq. 3 K = ceil(b_i M) on every row, capped at m+1 (Z12 alt.) */
#define PROXYATTN_FLAG_DESIGNATED_HEAD 0x10u /* proxy = the group's first query / kv head instead of
                                                the Eq. 2 mean ("a designated head"; Z1 alt.) */
/* Layout: token-major Q/K/V/O with token strides (see Conventions). */
#define PROXYATTN_FLAG_TOKEN_MAJOR 0x20u
/* estimate only: kstar is an INPUT (from an earlier call over another row range of the same
 * layer); Alg. 1 is skipped and budget is left untouched. */
#define PROXYATTN_FLAG_KSTAR_GIVEN 0x40u
/* estimate only: run A1-A3 (and Alg. 1 unless KSTAR_GIVEN) but not the selection; the block
 * scores L stay in the workspace for proxyattn_select_ws (block_cnt / block_idx may be NULL).
 * Lets a caller overlap the scores with a K* exchange (multi-GPU) and select afterwards. */
#define PROXYATTN_FLAG_SCORES_ONLY 0x80u
/* Validation ("all values finite"; S:49 / S:319 "non-finite input -> validation error"):
 * every call that reads Q / K / V first counts their NaN / Inf elements on the device,
 * synchronises `stream` and returns PROXYATTN_E_NONFINITE (nothing else enqueued) if any. */
#define PROXYATTN_FLAG_CHECK_FINITE 0x100u

#define PROXYATTN_OK               0
#define PROXYATTN_E_CONFIG        -1  /* divisibility, gamma range, shard alignment */
#define PROXYATTN_E_UNSUPPORTED   -2  /* head_dim / block size not supported by this build        */
#define PROXYATTN_E_SHAPE         -3  /* invalid block list (empty, unsorted, out of range, acausal) */
#define PROXYATTN_E_WORKSPACE     -4  /* workspace missing or too small                             */
#define PROXYATTN_E_CUDA          -5  /* CUDA launch / runtime failure                              */
#define PROXYATTN_E_NONFINITE     -6  /* NaN / Inf input, only with PROXYATTN_FLAG_CHECK_FINITE */

/* ------------------------------------------------------------- workspace -- */

/* Bytes of device scratch proxyattn_estimate needs (pooled proxies, row log-sum-exps,
 * the log-domain block map, budget partials).  Returns E_CONFIG on an invalid config. */
int proxyattn_workspace_bytes(const proxyattn_cfg* cfg, size_t* out_bytes);

/* ------------------------------------------------------- fused estimate -- */

/* A1-A6: proxy pooling (Eq. 2), strided sampling, proxy block
 * scores (Eq. 1), Alg. 1 budgets and Eq. 3 per-head top-k masks
 * (P:308-320).  Inputs Q, K (local shard layout above).  Outputs, all device memory:
 *   kstar     [Hl]        int32   K*_h, blocks needed by the last query block (1..M)
 *   budget    [Hl]        float   b_h = K*_h / M
 *   block_cnt [Hl][M]     int32   K_{h,m} = min(m+1, max(ceil(K*_h (m+1)/M), F, 1)) (Z12)
 *   block_idx [Hl][M][M]  int32   row stride M; first block_cnt entries valid, ascending,
 *                                 diagonal block m always included (Z15)
 * Requires every proxy group touched by the shard to be fully inside it (else E_CONFIG;
 * use the staged entries with an all-reduce of the pooled sums instead). */
int proxyattn_estimate(const proxyattn_cfg* cfg, const void* Q, const void* K,
                       void* workspace, size_t workspace_bytes,
                       int32_t* kstar, float* budget, int32_t* block_cnt, int32_t* block_idx,
                       void* stream);

/* ---------------------------------------------------------------- attention -- */

/* A7: block-sparse causal attention.  For every local head
 * h and query block m: O[h][t] = softmax over keys k in the listed blocks with k <= t of
 * Q[h][t]·K[kv(h)][k]/sqrt(d), times V.  Accepts ANY valid lists (non-empty, ascending,
 * in range, n <= m), so oracle masks can be injected.  With PROXYATTN_FLAG_CHECK the
 * lists are validated on the device first and E_SHAPE is returned on a violation
 * (this flag synchronises the stream).  b = 64 and d = b = 128 work on row PAIRS (2q, 2q+1)
 * of a head (b = 64: one 128-lane tile; d = b = 128: shared K/V tiles): a [row_begin,
 * row_end) range aligned to even rows gives outputs bit-identical to the full launch; an
 * unaligned one splits a pair (results within the bf16 tolerance, not bitwise). */
int proxyattn_prefill(const proxyattn_cfg* cfg, const void* Q, const void* K, const void* V,
                      const int32_t* block_cnt, const int32_t* block_idx, void* O,
                      void* stream);

/* A8: dense causal attention, the same engine with every causal block;
 * the same-run baseline for "speedup vs dense". */
int proxyattn_dense_prefill(const proxyattn_cfg* cfg, const void* Q, const void* K,
                            const void* V, void* O, void* stream);

/* ---------------------------------------------------------- staged entries -- */

/* A1 (Eq. 2 + stride): fp32 pooled SUMS over the shard's heads, qsum/ksum [g_l][N/s][d],
 * g_l = proxy groups touched by the shard.  With g < #shards the sums are partial and the
 * caller all-reduces them (the only cross-GPU step). */
int proxyattn_pool(const proxyattn_cfg* cfg, const void* Q, const void* K,
                   float* qsum, float* ksum, void* stream);

/* A2-A3 (Eq. 1): from complete fp32 pooled sums, rounds them to the proxy precision
 * (bf16 RNE; fp32 in FP32_DEBUG), then writes the log-domain block map
 * L [g_l][M][M] float, L[c][m][n] = max over sampled i in block m, j in block n, j <= i of
 * z_ij - lse_i (Z6), -inf for n > m.  Uses the workspace of proxyattn_workspace_bytes. */
int proxyattn_proxy_scores(const proxyattn_cfg* cfg, const float* qsum, const float* ksum,
                           void* workspace, size_t workspace_bytes, float* L, void* stream);

/* A4 (Alg. 1): per local head, kstar/budget from its own last-block queries (Z7-Z11). */
int proxyattn_budgets(const proxyattn_cfg* cfg, const void* Q, const void* K,
                      void* workspace, size_t workspace_bytes,
                      int32_t* kstar, float* budget, void* stream);

/* A5-A6 (Eq. 3): per (local head, block row) top-K_{h,m} columns of the shared row of L,
 * diagonal forced and counted, ties to the lower index (Z15, Z17), emitted ascending. */
int proxyattn_select(const proxyattn_cfg* cfg, const float* L, const int32_t* kstar,
                     int32_t* block_cnt, int32_t* block_idx, void* stream);

/* A5-A6 from the L a PROXYATTN_FLAG_SCORES_ONLY estimate left in `workspace` (same cfg,
 * rows [row_begin, row_end)); kstar [Hl] is an input. */
int proxyattn_select_ws(const proxyattn_cfg* cfg, const void* workspace, size_t workspace_bytes,
                        const int32_t* kstar, int32_t* block_cnt, int32_t* block_idx, void* stream);

/* -------------------------------------------------------------- host path -- */

/* End-to-end call on HOST buffers (pinned or pageable): copies Q/K/V to the device
 * workspace, runs estimate + prefill, copies O (and kstar when non-NULL) back, and
 * synchronises `stream` before returning.  device_ws must hold
 * proxyattn_forward_host_workspace_bytes(cfg) bytes.  Pipelined over query-block-row chunks,
 * last rows first (K, the last Q chunk, V, then the other Q chunks on an upload stream; each
 * chunk's row-range estimate and attention as soon as it lands; O chunks down on a third
 * stream); outputs equal the device-resident estimate + prefill bit for bit.  Needs every
 * proxy group of the shard to be local and no row range. */
int proxyattn_forward_host_workspace_bytes(const proxyattn_cfg* cfg, size_t* out_bytes);
int proxyattn_forward_host(const proxyattn_cfg* cfg, const void* Q_host, const void* K_host,
                           const void* V_host, void* O_host, int32_t* kstar_host,
                           void* device_ws, size_t device_ws_bytes, void* stream);

/* ---------------------------------------------------------------- varlen -- */

/* Variable-length batch (batch / varlen packing): n_seqs independent
 * sequences packed along the token axis, sequence i = tokens [cu_seqlens[i],
 * cu_seqlens[i+1]) (cu_seqlens: HOST int64 array of n_seqs + 1 entries, cu_seqlens[0] = 0,
 * non-decreasing).  Requires PROXYATTN_FLAG_TOKEN_MAJOR (Q/K/V/O are [total][heads][d] with
 * the cfg's token strides); cfg->seq_len is ignored.  Each sequence is one ProxyAttn layer
 * of its own (estimate A1-A6 + prefill A7, the paper's method per sequence):
 * its pooling, budgets and selection see only its own tokens.  Empty sequences are skipped.
 * Everything is ordered on `stream`.  bf16 with b = 128: the per-sequence estimates rotate
 * over up to 8 lanes (`stream` plus library helper streams, forked and joined by events, each
 * lane with its own scratch; fewer lanes — down to 2 — when the lanes' scratch would
 * exceed 256 MiB), the sequences' block lists are kept side by side in the workspace, and ONE
 * attention launch covers every sequence (longest first); otherwise one estimate + prefill
 * per sequence on `stream`.  The sequence table travels as kernel parameters (no host copy), so
 * the call is asynchronous.
 * kstar (optional, DEVICE [n_seqs][Hl] int32) receives each sequence's K*_h. */
int proxyattn_varlen_workspace_bytes(const proxyattn_cfg* cfg, int32_t n_seqs,
                                     const int64_t* cu_seqlens, size_t* out_bytes);
int proxyattn_forward_varlen(const proxyattn_cfg* cfg, int32_t n_seqs, const int64_t* cu_seqlens,
                             const void* Q, const void* K, const void* V, void* O,
                             void* workspace, size_t workspace_bytes, int32_t* kstar,
                             void* stream);

/* ------------------------------------------------- seq-avgpool comparator -- */

/* The coarse estimator the paper's granularity argument is measured against (SURVEY §8(f)
 * rank 4; SPEC S:365-373 seq_avgpool_scores; paper §1 / §2.1 "pooling ... along the
 * sequence dimension", Fig. 6b's estimation-latency comparison).  Per LOCAL
 * query head h and block rows m, n (n <= m):
 *   qbar_m = mean of block m's (real) query rows of head h, kbar_n = mean of block n's key
 *   rows of kv(h); S_h[m][n] = log softmax_{n' <= m}(qbar_m . kbar_n' / sqrt(d)) at n,
 *   -inf for n > m.
 * The block sums are rounded once to bf16 (RNE of the exact sum; fp32 with FP32_DEBUG), the
 * dots accumulate in fp32.  No row range (E_CONFIG); head_dim % 32 == 0; any GQA ratio; the
 * shard may split proxy groups (everything is per head).  Workspace:
 * proxyattn_avgpool_workspace_bytes.  S_out: DEVICE float [Hl][M][M]. */
int proxyattn_avgpool_workspace_bytes(const proxyattn_cfg* cfg, size_t* out_bytes);
int proxyattn_avgpool_scores(const proxyattn_cfg* cfg, const void* Q, const void* K,
                             void* workspace, size_t workspace_bytes, float* S_out, void* stream);
/* The comparator's full estimate: the same Alg. 1 budgets as proxyattn_estimate (kstar an
 * input with KSTAR_GIVEN; static_kstar honoured) and the same Eq. 3 row counts / selection
 * rule (diagonal forced, ties to the lower index, ascending lists), but each head ranks the
 * columns of its OWN map S_h.  Outputs as proxyattn_estimate. */
int proxyattn_avgpool_estimate(const proxyattn_cfg* cfg, const void* Q, const void* K,
                               void* workspace, size_t workspace_bytes,
                               int32_t* kstar, float* budget, int32_t* block_cnt, int32_t* block_idx,
                               void* stream);

/* ----------------------------------------------------------------- misc -- */

/* §3.1 cost model: g / (Hq * s^2). */
double proxyattn_cost_ratio(const proxyattn_cfg* cfg);

/* Thread-local message for the last non-zero return code. */
const char* proxyattn_last_error(void);

/* Library build id (compile flags / arch), for logs. */
const char* proxyattn_build_info(void);

/* Diagnostic: one 128x128x128 tcgen05 GEMM tile of each operand mode the attention
 * kernel uses, on bf16 inputs A [128][128], B [128][128]:
 *   C_ss [128][128] = A · B^T  (A, B K-major in shared memory, TMA SWIZZLE_128B)
 *   C_ts [128][128] = A · B    (A staged in TMEM via tcgen05.st, B MN-major in shared memory)
 * fp32 outputs.  Used by the GPU tests to pin the descriptor encodings. */
int proxyattn_debug_umma(const void* A, const void* B, float* C_ss, float* C_ts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PROXYATTN_H */
