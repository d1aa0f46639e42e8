/*
 * oracle.c — plain, slow, fp64 CPU oracle of the ProxyAttn hot path (arXiv 2509.24745).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  It follows the paper's algorithm step by
 * step with no blocking, fusion or reordering beyond what the
 * definitions state.  P:<line> = PAPER.md line, S:<line> = SPEC.md line.
 *
 * Parity pins: tests/test_oracle_*.py.  Functions without an independent pin: none
 * (the realistic-input budgets/selections at 32K-256K are data-dependent).
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------- O1 / O2 -- */

int oracle_validate(const oracle_cfg* c) {
    /* DS-1 invariants. */
    if (c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0) return -1;
    if (c->seq_len <= 0 || c->block_size <= 0 || c->stride <= 0 || c->n_groups <= 0) return -1;
    if (c->n_q_heads % c->n_kv_heads != 0) return -1;   /* GQA ratio integral */
    if (c->n_kv_heads % c->n_groups != 0) return -1;    /* groups aligned with the keys */
    if (c->block_size % c->stride != 0) return -1;
    /* N % b != 0 is allowed: the last block is padded */
    if (!(c->gamma > 0.0 && c->gamma <= 1.0)) return -1;
    if (c->min_budget_tokens < 0) return -1;
    return 0;
}

/* M = ceil(N / b) blocks; the last one is zero-padded when b does not divide N and the
 * padded tokens are masked as keys and produce no output. */
static int n_blocks(const oracle_cfg* c) {
    return (int)((c->seq_len + c->block_size - 1) / c->block_size);
}
/* sampled positions p = i*s < N (keep the first token of every stride window) */
static long n_sampled(const oracle_cfg* c) { return (c->seq_len + c->stride - 1) / c->stride; }

/* "the group granularity will be aligned with the keys"; Z3: contiguous ranges. */
static int group_of_kv(const oracle_cfg* c, int kvh) {
    return kvh / (c->n_kv_heads / c->n_groups);
}

int oracle_group_of_q(const oracle_cfg* c, int h) {
    int r = c->n_q_heads / c->n_kv_heads;           /* kv(h) = floor(h / r) */
    return group_of_kv(c, h / r);
}

/* -------------------------------------------------------------------- O3 -- */

double oracle_rne_bf16(double x) {
    /* bf16 = 1 sign bit, 8 exponent bits, 7 stored mantissa bits (8 significant bits).
     * Quantum of x's binade is 2^(e-8) with x = f * 2^e, f in [0.5, 1); below the
     * smallest normal (2^-126) the quantum is fixed at 2^-133.  Round to the nearest
     * multiple of the quantum, ties to even (nearbyint in the default rounding mode). */
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    frexp(x, &e);
    int qexp = e - 8;
    if (qexp < -133) qexp = -133;
    double q = ldexp(1.0, qexp);
    double r = nearbyint(x / q) * q;
    if (fabs(r) > 3.3895313892515355e38) r = copysign(INFINITY, x); /* > max bf16 */
    return r;
}

void oracle_pool(const oracle_cfg* c, const float* Q, const float* K,
                 double* Pq, double* Pk, double* scale_out) {
    const int d = c->head_dim, g = c->n_groups;
    const long N = c->seq_len, Ns = n_sampled(c);
    const int gq = c->n_q_heads / g, gk = c->n_kv_heads / g;   /* |G| for Q and for K (Z2) */

    #pragma omp parallel for schedule(static)
    for (long ci = 0; ci < (long)g * Ns; ++ci) {
        int grp = (int)(ci / Ns);
        long i = ci % Ns;
        long p = i * c->stride;              /* keep the first token of each stride window */
        double* pq = Pq + ci * d;
        double* pk = Pk + ci * d;
        for (int e = 0; e < d; ++e) { pq[e] = 0.0; pk[e] = 0.0; }
        for (int h = 0; h < c->n_q_heads; ++h) {
            if (oracle_group_of_q(c, h) != grp) continue;
            const float* q = Q + ((long)h * N + p) * d;
            for (int e = 0; e < d; ++e) pq[e] += (double)q[e];
            if (c->designated_head) break;     /* the group's first query head only */
        }
        for (int kvh = 0; kvh < c->n_kv_heads; ++kvh) {
            if (group_of_kv(c, kvh) != grp) continue;
            const float* k = K + ((long)kvh * N + p) * d;
            for (int e = 0; e < d; ++e) pk[e] += (double)k[e];
            if (c->designated_head) break;     /* ... and its first kv head */
        }
        if (c->round_bf16) {
            for (int e = 0; e < d; ++e) { pq[e] = oracle_rne_bf16(pq[e]); pk[e] = oracle_rne_bf16(pk[e]); }
        }
    }
    /* Eq. 2 means and Eq. 1's 1/sqrt(d_k): z = (qsum/|Gq|)·(ksum/|Gk|)/sqrt(d). */
    if (scale_out) *scale_out = c->designated_head ? 1.0 / sqrt((double)d)
                                                   : 1.0 / ((double)gq * (double)gk * sqrt((double)d));
}

/* ----------------------------------------------------------------- O4-O6 -- */

void oracle_proxy_scores(const oracle_cfg* c, const double* Pq, const double* Pk, double scale,
                         const int32_t* rows, int n_rows, double* lse, double* L) {
    const int d = c->head_dim, g = c->n_groups, M = n_blocks(c);
    const long Ns = n_sampled(c);
    const int bs = c->block_size / c->stride;     /* sampled rows per block */
    const int nr = rows ? n_rows : M;

    #pragma omp parallel
    {
        double* z = (double*)malloc(sizeof(double) * (size_t)Ns);
        #pragma omp for schedule(dynamic, 1)
        for (long it = 0; it < (long)g * nr; ++it) {
            int grp = (int)(it / nr);
            int m = rows ? rows[it % nr] : (int)(it % nr);
            double* Lrow = L + ((long)grp * M + m) * M;
            for (int n = 0; n < M; ++n) Lrow[n] = -INFINITY;     /* n > m stays -inf */
            for (int ii = 0; ii < bs; ++ii) {
                long i = (long)m * bs + ii;
                if (i >= Ns) break;                        /* padded sampled rows of the last block */
                const double* qi = Pq + ((long)grp * Ns + i) * d;
                /* O4: z_ij for sampled keys j <= i (causal by original positions j*s <= i*s) */
                double mx = -INFINITY;
                for (long j = 0; j <= i; ++j) {
                    const double* kj = Pk + ((long)grp * Ns + j) * d;
                    double dot = 0.0;
                    for (int e = 0; e < d; ++e) dot += qi[e] * kj[e];
                    z[j] = dot * scale;
                    if (z[j] > mx) mx = z[j];
                }
                /* O5: softmax normaliser over the sampled causal keys only. */
                double sum = 0.0;
                for (long j = 0; j <= i; ++j) sum += exp(z[j] - mx);
                double lse_i = mx + log(sum);
                if (lse) lse[(long)grp * Ns + i] = lse_i;
                /* O6: max-pool of log-probabilities over the (b/s)x(b/s) window (Z6). */
                for (long j = 0; j <= i; ++j) {
                    int n = (int)(j / bs);
                    double v = z[j] - lse_i;
                    if (v > Lrow[n]) Lrow[n] = v;
                }
            }
        }
        free(z);
    }
}

/* -------------------------------------------------------------------- O7 -- */

typedef struct { double v; int n; } vi_pair;

static int cmp_desc_then_index(const void* pa, const void* pb) {
    const vi_pair* a = (const vi_pair*)pa;
    const vi_pair* b = (const vi_pair*)pb;
    if (a->v > b->v) return -1;          /* descending value (Z10) */
    if (a->v < b->v) return 1;
    return (a->n < b->n) ? -1 : (a->n > b->n);   /* ties: lower index first (Z17) */
}

int oracle_budget_from_mass(const double* a, int M, double gamma, double* margin) {
    vi_pair* s = (vi_pair*)malloc(sizeof(vi_pair) * (size_t)M);
    for (int n = 0; n < M; ++n) { s[n].v = a[n]; s[n].n = n; }
    /* Alg. 1 line 3: a <- sort(a) / sum(a) */
    qsort(s, (size_t)M, sizeof(vi_pair), cmp_desc_then_index);
    double T = 0.0;
    for (int j = 0; j < M; ++j) T += s[j].v;        /* summed in the sorted order (Z11) */
    int kstar = M;
    double mg = INFINITY;
    if (gamma < 1.0) {
        /* Alg. 1 line 4: min{k | sum_{j<k} a[j] >= gamma}, k counted from 1 (Z9) */
        double P = 0.0, Pprev = 0.0;
        kstar = M;
        for (int k = 1; k <= M; ++k) {
            Pprev = P;
            P += s[k - 1].v / T;
            if (P >= gamma) { kstar = k; break; }
        }
        double up = P - gamma, down = gamma - Pprev;
        mg = up < down ? up : down;
    }
    /* gamma >= 1: the whole prefix is needed, K* = M (Z11); margin infinite (exact case). */
    if (margin) *margin = mg;
    free(s);
    return kstar;
}

void oracle_budgets(const oracle_cfg* c, const float* Q, const float* K,
                    const int32_t* heads, int n_heads,
                    int32_t* kstar, double* budget, double* margin, double* mass) {
    const int d = c->head_dim, M = n_blocks(c), b = c->block_size;
    const long N = c->seq_len;
    const int r = c->n_q_heads / c->n_kv_heads;
    const int nh = heads ? n_heads : c->n_q_heads;
    const double sd = sqrt((double)d);

    #pragma omp parallel
    {
        double* z = (double*)malloc(sizeof(double) * (size_t)N);
        double* a = (double*)malloc(sizeof(double) * (size_t)M);
        #pragma omp for schedule(dynamic, 1)
        for (int hi = 0; hi < nh; ++hi) {
            int h = heads ? heads[hi] : hi;
            int kvh = h / r;
            if (c->static_kstar > 0) {          /* static top-K baseline: Alg. 1 not run */
                int ks = c->static_kstar < M ? c->static_kstar : M;
                kstar[h] = ks;
                if (budget) budget[h] = (double)ks / M;
                if (margin) margin[h] = INFINITY;
                continue;
            }
            for (int n = 0; n < M; ++n) a[n] = 0.0;
            /* Alg. 1 line 1: A^ = softmax(Q_last K^T / sqrt(d_k)), own head, full resolution,
             * causal inside the last block (Z7). */
            for (long t = (long)(M - 1) * b; t < N; ++t) {   /* the last block's query rows */
                const float* q = Q + ((long)h * N + t) * d;
                double mx = -INFINITY;
                for (long k = 0; k <= t; ++k) {
                    const float* kk = K + ((long)kvh * N + k) * d;
                    double dot = 0.0;
                    for (int e = 0; e < d; ++e) dot += (double)q[e] * (double)kk[e];
                    z[k] = dot / sd;
                    if (z[k] > mx) mx = z[k];
                }
                double sum = 0.0;
                for (long k = 0; k <= t; ++k) sum += exp(z[k] - mx);
                /* Alg. 1 line 2: avgpool over the b query rows and the b keys of each block (Z8) */
                for (long k = 0; k <= t; ++k) a[k / b] += (exp(z[k] - mx) / sum) / ((double)b * b);
            }
            if (mass) for (int n = 0; n < M; ++n) mass[(long)h * M + n] = a[n];
            double mg;
            int ks = oracle_budget_from_mass(a, M, c->gamma, &mg);
            kstar[h] = ks;
            if (budget) budget[h] = (double)ks / M;
            if (margin) margin[h] = mg;
        }
        free(z);
        free(a);
    }
}

/* -------------------------------------------------------------------- O8 -- */

int oracle_row_count(const oracle_cfg* c, int kstar, int m) {
    const long M = n_blocks(c);
    const long b = c->block_size;
    long F = (c->min_budget_tokens + b - 1) / b;                 /* ceil(tokens / b) */
    long K = c->constant_k ? (long)kstar                          /* K = b_i M on every row */
                           : ((long)kstar * (m + 1) + M - 1) / M;   /* ceil(b_i (m+1)), Z12 */
    if (K < F) K = F;
    if (K < 1) K = 1;
    if (K > m + 1) K = m + 1;                                    /* capped at the causal row */
    return (int)K;
}

/* -------------------------------------------------------------------- O9 -- */

void oracle_select(const oracle_cfg* c, const double* L, const int32_t* kstar,
                   const int32_t* rows, int n_rows,
                   int32_t* block_cnt, int32_t* block_idx, double* cut_margin) {
    const int M = n_blocks(c), g = c->n_groups;
    const int nr = rows ? n_rows : M;

    #pragma omp parallel
    {
        vi_pair* s = (vi_pair*)malloc(sizeof(vi_pair) * (size_t)M);
        unsigned char* sel = (unsigned char*)malloc((size_t)M);
        #pragma omp for schedule(dynamic, 1)
        for (long it = 0; it < (long)g * nr; ++it) {
            int grp = (int)(it / nr);
            int m = rows ? rows[it % nr] : (int)(it % nr);
            const double* Lrow = L + ((long)grp * M + m) * M;
            /* Eq. 3 TopK over the shared score row; the diagonal is forced first (Z15),
             * the other columns 0..m-1 ordered by (score desc, index asc) (Z17). */
            for (int n = 0; n < m; ++n) { s[n].v = Lrow[n]; s[n].n = n; }
            if (c->force_sink && m > 0) s[0].v = INFINITY;   /* sink block first (forced, counted) */
            qsort(s, (size_t)m, sizeof(vi_pair), cmp_desc_then_index);
            for (int h = 0; h < c->n_q_heads; ++h) {
                if (oracle_group_of_q(c, h) != grp) continue;
                int K = oracle_row_count(c, kstar[h], m);
                int k = K - 1;                 /* non-diagonal blocks kept */
                memset(sel, 0, (size_t)M);
                sel[m] = 1;
                for (int j = 0; j < k; ++j) sel[s[j].n] = 1;
                long off = (long)h * M + m;
                int w = 0;
                for (int n = 0; n <= m; ++n) if (sel[n]) block_idx[off * M + w++] = n;   /* ascending */
                block_cnt[off] = w;
                if (cut_margin) {
                    cut_margin[off] = (k == 0 || k == m) ? INFINITY : (s[k - 1].v - s[k].v);
                }
            }
        }
        free(s);
        free(sel);
    }
}

/* ------------------------------------------------------------------- O10 -- */

static void attend_rows(const oracle_cfg* c, const float* Q, const float* K, const float* V,
                        int h, int m, const int32_t* list, int cnt, double* O, double* z) {
    const int d = c->head_dim, b = c->block_size;
    const long N = c->seq_len;
    const int kvh = h / (c->n_q_heads / c->n_kv_heads);
    const double sd = sqrt((double)d);
    for (long t = (long)m * b; t < (long)(m + 1) * b && t < N; ++t) {
        const float* q = Q + ((long)h * N + t) * d;
        /* pass 1: logits over the selected blocks' keys with k <= t, and their max */
        long nk = 0;
        double mx = -INFINITY;
        for (int u = 0; u < cnt; ++u) {
            long n = list[u];
            for (long k = n * b; k < (n + 1) * b && k <= t; ++k) {
                const float* kk = K + ((long)kvh * N + k) * d;
                double dot = 0.0;
                for (int e = 0; e < d; ++e) dot += (double)q[e] * (double)kk[e];
                z[nk] = dot / sd;
                if (z[nk] > mx) mx = z[nk];
                ++nk;
            }
        }
        /* pass 2: normalised weights times V */
        double* o = O + ((long)h * N + t) * d;
        for (int e = 0; e < d; ++e) o[e] = 0.0;
        double sum = 0.0;
        nk = 0;
        for (int u = 0; u < cnt; ++u) {
            long n = list[u];
            for (long k = n * b; k < (n + 1) * b && k <= t; ++k) {
                double p = exp(z[nk++] - mx);
                sum += p;
                const float* v = V + ((long)kvh * N + k) * d;
                for (int e = 0; e < d; ++e) o[e] += p * (double)v[e];
            }
        }
        for (int e = 0; e < d; ++e) o[e] /= sum;
    }
}

void oracle_attention(const oracle_cfg* c, const float* Q, const float* K, const float* V,
                      const int32_t* block_cnt, const int32_t* block_idx,
                      const int32_t* items, int n_items, double* O) {
    const int M = n_blocks(c);
    const long total = items ? n_items : (long)c->n_q_heads * M;
    #pragma omp parallel
    {
        double* z = (double*)malloc(sizeof(double) * (size_t)c->seq_len);
        #pragma omp for schedule(dynamic, 1)
        for (long it = 0; it < total; ++it) {
            int h = items ? items[2 * it] : (int)(it / M);
            int m = items ? items[2 * it + 1] : (int)(it % M);
            long off = (long)h * M + m;
            attend_rows(c, Q, K, V, h, m, block_idx + off * M, block_cnt[off], O, z);
        }
        free(z);
    }
}

void oracle_dense(const oracle_cfg* c, const float* Q, const float* K, const float* V,
                  const int32_t* items, int n_items, double* O) {
    const int M = n_blocks(c);
    const long total = items ? n_items : (long)c->n_q_heads * M;
    #pragma omp parallel
    {
        double* z = (double*)malloc(sizeof(double) * (size_t)c->seq_len);
        int32_t* all = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
        for (int n = 0; n < M; ++n) all[n] = n;
        #pragma omp for schedule(dynamic, 1)
        for (long it = 0; it < total; ++it) {
            int h = items ? items[2 * it] : (int)(it / M);
            int m = items ? items[2 * it + 1] : (int)(it % M);
            attend_rows(c, Q, K, V, h, m, all, m + 1, O, z);    /* every causal block 0..m */
        }
        free(all);
        free(z);
    }
}

/* ------------------------------------------------------------------- O11 -- */

/* "q̄_m = mean of b query rows; k̄_n = mean of b key rows; score(m,n) = softmax
 * over valid n of q̄_m·k̄_n/√d_k".  Block sums in fp64 (rounded to bf16 when round_bf16),
 * divided by the block's real row count; softmax over n <= m, stored as log-probabilities. */
void oracle_seq_avgpool_scores(const oracle_cfg* c, const float* Q, const float* K, double* S) {
    const int d = c->head_dim, M = n_blocks(c), b = c->block_size;
    const long N = c->seq_len;
    const int r = c->n_q_heads / c->n_kv_heads;
    double* qbar = (double*)malloc(sizeof(double) * (size_t)c->n_q_heads * M * d);
    double* kbar = (double*)malloc(sizeof(double) * (size_t)c->n_kv_heads * M * d);
    /* block means: sum the block's real rows, round the sum (bf16 contract), divide */
    for (int role = 0; role < 2; ++role) {
        const int H = role == 0 ? c->n_q_heads : c->n_kv_heads;
        const float* X = role == 0 ? Q : K;
        double* out = role == 0 ? qbar : kbar;
        for (int h = 0; h < H; ++h) {
            for (int m = 0; m < M; ++m) {
                double* o = out + ((long)h * M + m) * d;
                long t0 = (long)m * b, t1 = t0 + b < N ? t0 + b : N;
                for (int e = 0; e < d; ++e) o[e] = 0.0;
                for (long t = t0; t < t1; ++t)
                    for (int e = 0; e < d; ++e) o[e] += (double)X[((long)h * N + t) * d + e];
                for (int e = 0; e < d; ++e) {
                    if (c->round_bf16) o[e] = oracle_rne_bf16(o[e]);
                    o[e] /= (double)(t1 - t0);
                }
            }
        }
    }
    #pragma omp parallel for schedule(dynamic, 1)
    for (long hm = 0; hm < (long)c->n_q_heads * M; ++hm) {
        int h = (int)(hm / M), m = (int)(hm % M);
        const double* q = qbar + ((long)h * M + m) * d;
        double* row = S + ((long)h * M + m) * M;
        double mx = -INFINITY;
        for (int n = 0; n < M; ++n) {
            if (n > m) { row[n] = -INFINITY; continue; }
            const double* k = kbar + ((long)(h / r) * M + n) * d;
            double dot = 0.0;
            for (int e = 0; e < d; ++e) dot += q[e] * k[e];
            row[n] = dot / sqrt((double)d);
            if (row[n] > mx) mx = row[n];
        }
        double sum = 0.0;
        for (int n = 0; n <= m; ++n) sum += exp(row[n] - mx);
        double lse = mx + log(sum);
        for (int n = 0; n <= m; ++n) row[n] -= lse;
    }
    free(qbar);
    free(kbar);
}

void oracle_select_heads(const oracle_cfg* c, const double* S, const int32_t* kstar,
                         int32_t* block_cnt, int32_t* block_idx, double* cut_margin) {
    const int M = n_blocks(c);
    #pragma omp parallel
    {
        vi_pair* s = (vi_pair*)malloc(sizeof(vi_pair) * (size_t)M);
        unsigned char* sel = (unsigned char*)malloc((size_t)M);
        #pragma omp for schedule(dynamic, 1)
        for (long hm = 0; hm < (long)c->n_q_heads * M; ++hm) {
            int h = (int)(hm / M), m = (int)(hm % M);
            const double* row = S + ((long)h * M + m) * M;
            /* the same Eq. 3 rule as O9: diagonal forced first (Z15), (score desc, index asc) */
            for (int n = 0; n < m; ++n) { s[n].v = row[n]; s[n].n = n; }
            if (c->force_sink && m > 0) s[0].v = INFINITY;
            qsort(s, (size_t)m, sizeof(vi_pair), cmp_desc_then_index);
            int K = oracle_row_count(c, kstar[h], m);
            int k = K - 1;
            memset(sel, 0, (size_t)M);
            sel[m] = 1;
            for (int j = 0; j < k; ++j) sel[s[j].n] = 1;
            int w = 0;
            for (int n = 0; n <= m; ++n) if (sel[n]) block_idx[hm * M + w++] = n;
            block_cnt[hm] = w;
            if (cut_margin) cut_margin[hm] = (k == 0 || k == m) ? INFINITY : (s[k - 1].v - s[k].v);
        }
        free(s);
        free(sel);
    }
}

/* ------------------------------------------------------------- cost model -- */

double oracle_cost_ratio(const oracle_cfg* c) {
    return (double)c->n_groups / ((double)c->n_q_heads * c->stride * c->stride);
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n >= 1) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
