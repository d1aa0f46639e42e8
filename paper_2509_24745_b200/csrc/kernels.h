// kernels.h — host-side launchers of the libproxyattn kernels (called by api.cu).
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace pa {

// A1: pooled group sums at sampled positions.  qsum/ksum (fp32) and/or Pq/Pk (element type
// of the build, bf16 RNE or fp32) — any of the four may be null.
// [q_i0, i_end): sampled rows whose Q is pooled; K is pooled for [0, i_end) (row-range
// estimate); defaults: every row.
cudaError_t launch_pool(const Dims& D, const void* Q, const void* K, float* qsum, float* ksum,
                        void* Pq, void* Pk, cudaStream_t st, long long q_i0 = 0, long long i_end = -1);
// A1 (staged path): round complete fp32 sums to the proxy element type.
cudaError_t launch_round_proxies(const Dims& D, const float* qsum, const float* ksum, void* Pq,
                                 void* Pk, cudaStream_t st);
// A2: lse[c][i] over sampled causal keys.  A3: log-domain block max map.
cudaError_t launch_proxy_lse(const Dims& D, const void* Pq, const void* Pk, float* lse,
                             cudaStream_t st);
cudaError_t launch_proxy_maxpool(const Dims& D, const void* Pq, const void* Pk, const float* lse,
                                 float* L, cudaStream_t st);
// A4: Alg. 1 row lse of the last block, block masses, then sort + prefix -> kstar/budget.
cudaError_t launch_budget_lse(const Dims& D, const void* Q, const void* K, float* blse,
                              cudaStream_t st);
cudaError_t launch_budget_mass(const Dims& D, const void* Q, const void* K, const float* blse,
                               float* bmass, cudaStream_t st);
// Static top-K baseline: kstar[h] = min(static_kstar, M) for every local head.
cudaError_t launch_static_budget(const Dims& D, int* kstar, float* budget, cudaStream_t st);
cudaError_t launch_budget_finalize(const Dims& D, const float* bmass, int* kstar, float* budget,
                                   cudaStream_t st);
// A5-A6: per (group, row) ordering, per head compaction.
// per_head: L is [Hl][M][M] (one score map per local head, the seq-avgpool comparator).
cudaError_t launch_select(const Dims& D, const float* L, const int* kstar, int* block_cnt,
                          int* block_idx, cudaStream_t st, bool per_head = false);
// A7/A8 fp32 debug (SIMT) attention; block lists null => dense.
cudaError_t launch_attn_simt(const Dims& D, const void* Q, const void* K, const void* V,
                             const int* block_cnt, const int* block_idx, void* O,
                             cudaStream_t st);
// Varlen (one packed launch over several sequences, token-major, b = 128): sequence s owns the
// tokens [tok0, tok0 + N) of the packed tensors, its block lists start at cnt_off / idx_off
// ([Hl][M] / [Hl][M][M] of its own M), and its work items are [item0, item0 + Hl * M).
struct SeqDesc {
    long long tok0, cnt_off, idx_off;
    int N, M, item0, pad;
};
// Writes n descriptors into device memory from kernel parameters (no pageable host copy, so
// the varlen call stays asynchronous): 64 per launch.
cudaError_t write_seq_descs(SeqDesc* dst, const SeqDesc* host, int n, cudaStream_t st);
// D: the packed layout (seq_len = total tokens); seqs: device array of n_seqs descriptors.
cudaError_t launch_attn_tc8_varlen(const Dims& D, const void* Q, const void* K, const void* V,
                                   const int* block_cnt, const int* block_idx, void* O,
                                   const SeqDesc* seqs, int n_seqs, int n_items, cudaStream_t st);
cudaError_t launch_attn_tc8(const Dims& D, const void* Q, const void* K, const void* V,
                            const int* block_cnt, const int* block_idx, void* O, cudaStream_t st);
// Scheduler state of an attention launch pair (attn_tc8.cu), shared by attn_tc9.cu.
cudaError_t attn_sched_prepare(const Dims& D, const int* block_cnt, size_t n_items, cudaStream_t st,
                               void** sched, int** flagged, const int** kvperm);
// A7 row-pair kernel (d = b = 128, sparse): work units = (head, block-row pair); varlen when
// n_seqs > 0 (sequence s owns units [item0, item0 + attn_tc9_units(Hl, M_s))).
size_t attn_tc9_units(int Hl, int M);
cudaError_t launch_attn_tc9(const Dims& D, const void* Q, const void* K, const void* V, const int* block_cnt,
                            const int* block_idx, void* O, cudaStream_t st, const SeqDesc* seqs = nullptr,
                            int n_seqs = 0, int varlen_items = 0);
// tcgen05 estimation (bf16, d = b = 128, s = 4): A2+A3 and A4 (see score_tc.cu).
bool score_tc_supported(const Dims& D);
size_t score_tc_scratch_bytes(const Dims& D);
// tile rows [tr0, tr1) of 128 sampled rows (tr1 < 0: all); L written for block rows [rb, re)
cudaError_t launch_proxy_tc(const Dims& D, const void* Pq, const void* Pk, float* scratch,
                            float* lse_nat, float* L, cudaStream_t st, int tr0 = 0, int tr1 = -1);
cudaError_t launch_budget_tc(const Dims& D, const void* Q, const void* K, float* scratch,
                             float* bmass, cudaStream_t st);
// Device-side validation of block lists; *bad_out (device int) receives the violation count.
cudaError_t launch_check_lists(const Dims& D, const int* block_cnt, const int* block_idx,
                               int* bad_out, cudaStream_t st);
// Number of non-finite elements (NaN / Inf) of a tensor laid out as `rows` runs of
// `row_elems` contiguous elements, `row_stride` elements apart, added to *bad (device int).
cudaError_t launch_count_nonfinite(const void* p, bool fp32, long long rows, long long row_elems,
                                   long long row_stride, int* bad, cudaStream_t st);
// Seq-avgpool comparator: per-block means of Q (per local head) and of K (per
// local kv head), bf16 RNE of the exact sums (fp32 in FP32_DEBUG) into Qb [Hl][M][d], Kb
// [Hkvl][M][d] and the real row count of each block into cnt [M].
cudaError_t launch_block_pool(const Dims& D, const void* Q, const void* K, void* Qb, void* Kb,
                              cudaStream_t st);
// z[hl][m][n] = Qb_m . Kb_n / (c_m c_n sqrt(d)) for n <= m (-inf above), lse[hl][m] over n <= m
// (natural log); with normalize, z -= lse (log-domain scores, the comparator's map).
cudaError_t launch_avgpool_scores(const Dims& D, const void* Qb, const void* Kb, float* z, float* lse,
                                  bool normalize, cudaStream_t st);
// Diagnostic GEMM tile (see proxyattn_debug_umma).
cudaError_t launch_debug_umma(const void* A, const void* B, float* C_ss, float* C_ts,
                              cudaStream_t st);

}  // namespace pa
