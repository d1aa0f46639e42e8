/*
 * oracle.h — plain fp64 CPU oracle of the ProxyAttn hot path (arXiv 2509.24745).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (libproxyattn, include/proxyattn.h) shares no code, header, helper or constant
 * with this file and never calls it.
 *
 * Citations: P:<line> = PAPER.md line, S:<line> = SPEC.md line (reference text).
 * Step numbers O1..O10 follow SURVEY.md §8(c); readings Z1..Z23 are listed in DESIGN.md.
 *
 * Pins: every function below is pinned by tests/test_oracle_*.py (-m "not gpu")
 * against values the paper / SPEC fix, closed forms, brute force on tiny inputs
 * and invariants.  See DESIGN.md "Oracle pins".
 */
#ifndef PROXYATTN_ORACLE_H
#define PROXYATTN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Configuration (AttnConfig). */
typedef struct {
    int32_t n_q_heads;          /* Hq */
    int32_t n_kv_heads;         /* Hkv */
    int32_t head_dim;           /* d (d_k in P:248) */
    int64_t seq_len;            /* N */
    int32_t block_size;         /* b */
    int32_t stride;             /* s */
    int32_t n_groups;           /* g, number of proxy heads */
    double  gamma;              /* γ of Alg. 1 */
    int32_t min_budget_tokens;  /* P:466 / P:764 (reading Z13/Z14) */
    int32_t round_bf16;         /* 1: pooled proxies are rounded to bf16 (RNE), precision contract c.3 */
    /* method variants (DESIGN.md readings; all 0 = the paper's method as read in Z1-Z23) */
    int32_t force_sink;         /* block 0 always selected and counted (Z16 alternative) */
    int32_t constant_k;         /* Eq. 3 K = K* on every row, capped at m+1 (Z12 alternative) */
    int32_t designated_head;    /* proxy = the group's first q / kv head (Z1 alternative) */
    int32_t static_kstar;       /* > 0: every head uses K* = static_kstar (Fig. 6c static top-K) */
} oracle_cfg;

/* O1: returns 0 when the config satisfies the DS-1 invariants, -1 otherwise.
 * N need not be a multiple of b: M = ceil(N/b), the last block is zero-padded. */
int oracle_validate(const oracle_cfg* c);

/* O3 helper: round a double to the nearest bf16 value, ties to even (plain definition). */
double oracle_rne_bf16(double x);

/* O2: proxy group of query head h (contiguous balanced KV ranges, Z3). */
int oracle_group_of_q(const oracle_cfg* c, int h);

/* O3 (Eq. 2; stride P:269-270): pooled sums at sampled positions p = i*s.
 * Q: [Hq][N][d], K: [Hkv][N][d] (fp32 values, read exactly).
 * Pq, Pk: [g][N/s][d]; sums (rounded to bf16 when round_bf16).  scale_out: the logit scale
 * 1/(|Gq|·|Gk|·sqrt(d)) that turns the sums into Eq. 1's Q^g K^g^T / sqrt(d_k) (Z2, Z5). */
void oracle_pool(const oracle_cfg* c, const float* Q, const float* K,
                 double* Pq, double* Pk, double* scale_out);

/* O4-O6 (Eq. 1): log-domain block scores.
 * lse: [g][N/s] (may be NULL), L: [g][M][M], L[c][m][n] = max over sampled i in block m,
 * j in block n, j<=i of z_ij - lse_i; -inf for n > m (Z6).
 * rows: optional list of block rows to compute (n_rows entries); NULL = all rows.
 * Rows not listed are left untouched. */
void oracle_proxy_scores(const oracle_cfg* c, const double* Pq, const double* Pk, double scale,
                         const int32_t* rows, int n_rows, double* lse, double* L);

/* O7 inner step (Alg. 1 lines 3-4; readings Z9, Z10, Z11, Z17):
 * given block masses a[0..M), returns K* = min{k >= 1 : sum of the k largest normalised
 * masses >= gamma}; gamma >= 1 gives M.  margin (may be NULL) receives the budget margin
 * delta = min(P(K*) - gamma, gamma - P(K*-1)) on the normalised prefix P. */
int oracle_budget_from_mass(const double* a, int M, double gamma, double* margin);

/* O7 (Alg. 1): per query head budgets from its own last-block queries.
 * heads: optional list of query heads (NULL = all).  Outputs indexed by head id:
 * kstar[h], budget[h] = kstar/M, margin[h] (may be NULL), mass: [Hq][M] (may be NULL). */
void oracle_budgets(const oracle_cfg* c, const float* Q, const float* K,
                    const int32_t* heads, int n_heads,
                    int32_t* kstar, double* budget, double* margin, double* mass);

/* O8 (Eq. 3 K = b_i N applied per causal row, Z12; floor Z13/Z14):
 * K_{h,m} = min(m+1, max(ceil(K* (m+1) / M), F, 1)),  F = ceil(min_budget_tokens / b). */
int oracle_row_count(const oracle_cfg* c, int kstar, int m);

/* O9 (Eq. 3; Z15 diagonal forced and counted, Z17 ties to lower index):
 * for every head h and block row m listed: block_cnt[h*M+m], block_idx[(h*M+m)*M + ...]
 * ascending.  cut_margin[h*M+m] (may be NULL) = L[o_k] - L[o_{k+1}] with k = K-1,
 * +inf when k == 0 or k == m.  rows: optional list (NULL = all rows). */
void oracle_select(const oracle_cfg* c, const double* L, const int32_t* kstar,
                   const int32_t* rows, int n_rows,
                   int32_t* block_cnt, int32_t* block_idx, double* cut_margin);

/* O10: block-sparse causal attention in fp64, two-pass softmax.
 * Q: [Hq][N][d], K/V: [Hkv][N][d]; block lists as produced by oracle_select (or injected).
 * items: optional list of (h, m) pairs, 2*n_items ints (NULL = every head and row).
 * O: [Hq][N][d] doubles, only the listed rows are written. */
void oracle_attention(const oracle_cfg* c, const float* Q, const float* K, const float* V,
                      const int32_t* block_cnt, const int32_t* block_idx,
                      const int32_t* items, int n_items, double* O);

/* Dense causal attention = O10 with every causal block selected. */
void oracle_dense(const oracle_cfg* c, const float* Q, const float* K, const float* V,
                  const int32_t* items, int n_items, double* O);

/* §3.1 cost model: g / (Hq * s^2). */
double oracle_cost_ratio(const oracle_cfg* c);

/* O11 — the seq-avgpool comparator (SPEC S:365-373 seq_avgpool_scores;
 * paper §1 / §2.1, "pooling methods along the sequence dimension"): per query head h,
 * qbar_m = mean of block m's real query rows of head h, kbar_n = mean of block n's real key
 * rows of kv(h) (the padded last block averages its real rows only), and
 * S[h][m][n] = z_mn - log sum_{n' <= m} exp(z_mn'),  z_mn = qbar_m . kbar_n / sqrt(d),
 * for n <= m; -inf for n > m.  round_bf16: the block SUMS are rounded to bf16 before the
 * division (the precision contract of the bf16 build, as O3's proxies).
 * Q: [Hq][N][d], K: [Hkv][N][d]; S: [Hq][M][M]. */
void oracle_seq_avgpool_scores(const oracle_cfg* c, const float* Q, const float* K, double* S);

/* O9 over PER-HEAD score maps (the comparator's selection): as oracle_select, but head h
 * ranks row m of its own map S[h] (S: [Hq][M][M]). */
void oracle_select_heads(const oracle_cfg* c, const double* S, const int32_t* kstar,
                         int32_t* block_cnt, int32_t* block_idx, double* cut_margin);

/* Number of OpenMP threads the oracle uses; set_num_threads changes it (n >= 1). */
int oracle_num_threads(void);
void oracle_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
