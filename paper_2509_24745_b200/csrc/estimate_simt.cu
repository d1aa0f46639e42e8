// estimate_simt.cu — A1 pooling, SIMT (FFMA) A2-A4 estimation kernels, A4 budget finalize
// and A5-A6 selection.
//
// A1  Eq. 2, GQA alignment, stride
// A2  Eq. 1 softmax normaliser over the sampled causal keys (Z4)
// A3  Eq. 1 max-pool to (N/b)x(N/b), stored as log-probabilities (Z6)
// A4  Alg. 1 with readings Z7-Z11
// A5  Eq. 3 row counts (Z12-Z14), A6 Eq. 3 top-k (Z15, Z17)
//
// The SIMT estimation kernels (warp per logit row) serve the FP32_DEBUG build (1e-4
// contract) and small configs; the bf16 build uses the tcgen05 kernels of
// estimate_tc.cu for A2-A4 when the shapes allow.
#include <cfloat>
#include <climits>
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace pa {
namespace {

template <typename T>
__device__ __forceinline__ void load_row(const T* p, int lane, float (&x)[4], int dv) {
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = (j < dv) ? to_f32(p[lane * dv + j]) : 0.f;
}

// ------------------------------------------------------------------------ A1 --
// One warp per (local group c, sampled row i).  Lane owns d/32 contiguous elements.
template <typename T>
__global__ void pool_kernel(Dims D, const T* __restrict__ Q, const T* __restrict__ K,
                            float* __restrict__ qsum, float* __restrict__ ksum,
                            T* __restrict__ Pq, T* __restrict__ Pk, long long q_i0, long long i_end) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<long long>(D.gl) * D.Ns) return;
    const int c = static_cast<int>(w / D.Ns);
    const long long i = w % D.Ns;
    if (i >= i_end) return;                       // row-range estimate: rows past the range
    const bool do_q = i >= q_i0;                  // ... and keys only before it
    const long long p = i * D.s;  // first token of each stride window
    const int grp = D.gb + c;
    const int dv = D.d >> 5;
    // group's query heads / kv heads inside the shard (designated head: only the first)
    const int gqe = has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD) ? 1 : D.gq;
    const int gke = has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD) ? 1 : D.gk;
    const int h0 = max(grp * D.gq, D.qb), h1 = min(grp * D.gq + gqe, D.qe);
    const int k0 = max(grp * D.gk, D.kvb), k1 = min(grp * D.gk + gke, D.kvb + D.Hkvl);
    // fp64 accumulation: the sum of <= 64 bf16 (or fp32) values is then exact, so the proxy
    // rounding below is one RNE of the exact sum, as in the oracle (precision contract c.3).
    double aq[4] = {0., 0., 0., 0.}, ak[4] = {0., 0., 0., 0.};
    for (int h = h0; h < (do_q ? h1 : h0); ++h) {  // fixed ascending order
        float x[4];
        load_row(Q + q_off(D, h - D.qb, p), lane, x, dv);
#pragma unroll
        for (int j = 0; j < 4; ++j) aq[j] += x[j];
    }
    for (int k = k0; k < k1; ++k) {
        float x[4];
        load_row(K + kv_off(D, k - D.kvb, p), lane, x, dv);
#pragma unroll
        for (int j = 0; j < 4; ++j) ak[j] += x[j];
    }
    const long long o = w * D.d + lane * dv;
    for (int j = 0; j < dv; ++j) {
        if (qsum && do_q) qsum[o + j] = static_cast<float>(aq[j]);
        if (ksum) ksum[o + j] = static_cast<float>(ak[j]);
        if (Pq && do_q) Pq[o + j] = from_f64<T>(aq[j]);
        if (Pk) Pk[o + j] = from_f64<T>(ak[j]);
    }
}

// bf16 build: 16-byte loads (8 elements per thread, d/8 threads per sampled row), heads
// summed in ascending order in fp64 (exact), 4 rows in flight per thread.
__global__ void pool_bf16_kernel(Dims D, const __nv_bfloat16* __restrict__ Q,
                                 const __nv_bfloat16* __restrict__ K, float* __restrict__ qsum,
                                 float* __restrict__ ksum, __nv_bfloat16* __restrict__ Pq,
                                 __nv_bfloat16* __restrict__ Pk, long long q_i0, long long i_end) {
    const int tpr = D.d >> 3;
    const long long gt = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    const long long row = gt / tpr;
    const int part = static_cast<int>(gt % tpr);
    if (row >= static_cast<long long>(D.gl) * D.Ns) return;
    const int c = static_cast<int>(row / D.Ns);
    const long long i = row % D.Ns;
    if (i >= i_end) return;                       // row-range estimate: rows past the range
    const bool do_q = i >= q_i0;                  // ... and keys only before it
    const long long p = i * D.s;
    const int grp = D.gb + c;
    // group's query heads / kv heads inside the shard (designated head: only the first)
    const int gqe = has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD) ? 1 : D.gq;
    const int gke = has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD) ? 1 : D.gk;
    const int h0 = max(grp * D.gq, D.qb), h1 = do_q ? min(grp * D.gq + gqe, D.qe) : h0;
    const int k0 = max(grp * D.gk, D.kvb), k1 = min(grp * D.gk + gke, D.kvb + D.Hkvl);
    auto accumulate = [&](const __nv_bfloat16* base, int a, int b, int head0, long long hs, long long ts,
                          double (&acc)[8]) {
        for (int h = a; h < b; h += 4) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (h + k < b)
                    v[k] = __ldg(reinterpret_cast<const uint4*>(
                        base + static_cast<long long>(h + k - head0) * hs + p * ts + part * 8));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (h + k >= b) break;
                const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&v[k]);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 f = __bfloat1622float2(e[q]);
                    acc[2 * q] += f.x;
                    acc[2 * q + 1] += f.y;
                }
            }
        }
    };
    double aq[8] = {0, 0, 0, 0, 0, 0, 0, 0}, ak[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    accumulate(Q, h0, h1, D.qb, D.q_hs, D.q_ts, aq);
    accumulate(K, k0, k1, D.kvb, D.kv_hs, D.kv_ts, ak);
    const long long o = row * D.d + part * 8;
    if (qsum) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (do_q) qsum[o + q] = static_cast<float>(aq[q]);
            ksum[o + q] = static_cast<float>(ak[q]);
        }
    }
    if (Pq) {
        uint4 oq, ok;
        uint32_t* wq = reinterpret_cast<uint32_t*>(&oq);
        uint32_t* wk = reinterpret_cast<uint32_t*>(&ok);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162 bq(__double2bfloat16(aq[2 * q]), __double2bfloat16(aq[2 * q + 1]));
            const __nv_bfloat162 bk(__double2bfloat16(ak[2 * q]), __double2bfloat16(ak[2 * q + 1]));
            wq[q] = *reinterpret_cast<const uint32_t*>(&bq);
            wk[q] = *reinterpret_cast<const uint32_t*>(&bk);
        }
        if (do_q) *reinterpret_cast<uint4*>(Pq + o) = oq;
        *reinterpret_cast<uint4*>(Pk + o) = ok;
    }
}

template <typename T>
__global__ void round_kernel(long long n, const float* __restrict__ qs, const float* __restrict__ ks,
                             T* __restrict__ Pq, T* __restrict__ Pk) {
    long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) {
        Pq[i] = from_f32<T>(qs[i]);
        Pk[i] = from_f32<T>(ks[i]);
    }
}

// ------------------------------------------------------------------------ A2 --
// One warp per (c, sampled row i): lse_i = log sum_{j<=i} exp(z_ij).
template <typename T>
__global__ void proxy_lse_simt(Dims D, const T* __restrict__ Pq, const T* __restrict__ Pk,
                               float scale, float* __restrict__ lse) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<long long>(D.gl) * D.Ns) return;
    const int c = static_cast<int>(w / D.Ns);
    const long long i = w % D.Ns;
    const int dv = D.d >> 5;
    float q[4];
    load_row(Pq + w * D.d, lane, q, dv);
    const T* kb = Pk + static_cast<long long>(c) * D.Ns * D.d;
    float mx = -INFINITY, sum = 0.f;
    for (long long j = 0; j <= i; ++j) {
        float k[4];
        load_row(kb + j * D.d, lane, k, dv);
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) part = fmaf(q[e], k[e], part);
        const float z = warp_sum(part) * scale;
        if (z > mx) {
            sum = sum * expf(mx - z) + 1.f;
            mx = z;
        } else {
            sum += expf(z - mx);
        }
    }
    if (lane == 0) lse[w] = mx + logf(sum);
}

// ------------------------------------------------------------------------ A3 --
// One warp per (c, m, n): L[c][m][n] = max_{i in m, j in n, j<=i} z_ij - lse_i; -inf for n > m.
template <typename T>
__global__ void proxy_maxpool_simt(Dims D, const T* __restrict__ Pq, const T* __restrict__ Pk,
                                   float scale, const float* __restrict__ lse,
                                   float* __restrict__ L) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const long long cells = static_cast<long long>(D.gl) * D.M * D.M;
    if (w >= cells) return;
    const int c = static_cast<int>(w / (static_cast<long long>(D.M) * D.M));
    const int m = static_cast<int>((w / D.M) % D.M);
    const int n = static_cast<int>(w % D.M);
    if (n > m) {
        if (lane == 0) L[w] = -INFINITY;
        return;
    }
    const int dv = D.d >> 5;
    const T* qb = Pq + static_cast<long long>(c) * D.Ns * D.d;
    const T* kb = Pk + static_cast<long long>(c) * D.Ns * D.d;
    float best = -INFINITY;
    for (int ii = 0; ii < D.bs; ++ii) {
        const long long i = static_cast<long long>(m) * D.bs + ii;
        if (i >= D.Ns) break;                     // padded sampled rows of a partial last block
        float q[4];
        load_row(qb + i * D.d, lane, q, dv);
        const float li = lse[static_cast<long long>(c) * D.Ns + i];
        for (int jj = 0; jj < D.bs; ++jj) {
            const long long j = static_cast<long long>(n) * D.bs + jj;
            if (j > i) break;
            float k[4];
            load_row(kb + j * D.d, lane, k, dv);
            float part = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) part = fmaf(q[e], k[e], part);
            best = fmaxf(best, warp_sum(part) * scale - li);
        }
    }
    if (lane == 0) L[w] = best;
}

// ------------------------------------------------------------------------ A4 --
// One warp per (local head, last-block row t): lse_t over keys k <= t (own head, full res).
template <typename T>
__global__ void budget_lse_simt(Dims D, const T* __restrict__ Q, const T* __restrict__ K,
                                float* __restrict__ blse) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<long long>(D.Hl) * D.b) return;
    const int hl = static_cast<int>(w / D.b);
    const long long t = static_cast<long long>(D.M - 1) * D.b + (w % D.b);   // last block's rows
    if (t >= D.N) {                               // padded row of a partial last block
        if (lane == 0) blse[w] = INFINITY;        // contributes exp(-inf) = 0 to the masses
        return;
    }
    const int dv = D.d >> 5;
    const float sc = rsqrtf(static_cast<float>(D.d));
    float q[4];
    load_row(Q + q_off(D, hl, t), lane, q, dv);
    const T* kb = K + kv_off(D, hl / D.r, 0);
    float mx = -INFINITY, sum = 0.f;
    for (long long k = 0; k <= t; ++k) {
        float kv[4];
        load_row(kb + k * D.kv_ts, lane, kv, dv);
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) part = fmaf(q[e], kv[e], part);
        const float z = warp_sum(part) * sc;
        if (z > mx) {
            sum = sum * expf(mx - z) + 1.f;
            mx = z;
        } else {
            sum += expf(z - mx);
        }
    }
    if (lane == 0) blse[w] = mx + logf(sum);
}

// One warp per (local head, key block n): a[n] = (1/b^2) sum_t sum_{k in n, k<=t} softmax.
template <typename T>
__global__ void budget_mass_simt(Dims D, const T* __restrict__ Q, const T* __restrict__ K,
                                 const float* __restrict__ blse, float* __restrict__ bmass) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<long long>(D.Hl) * D.M) return;
    const int hl = static_cast<int>(w / D.M);
    const int n = static_cast<int>(w % D.M);
    const int dv = D.d >> 5;
    const float sc = rsqrtf(static_cast<float>(D.d));
    const T* kb = K + kv_off(D, hl / D.r, 0);
    float acc = 0.f;
    for (int tt = 0; tt < D.b; ++tt) {
        const long long t = static_cast<long long>(D.M - 1) * D.b + tt;
        if (t >= D.N) break;
        float q[4];
        load_row(Q + q_off(D, hl, t), lane, q, dv);
        const float lt = blse[static_cast<long long>(hl) * D.b + tt];
        for (int kk = 0; kk < D.b; ++kk) {
            const long long k = static_cast<long long>(n) * D.b + kk;
            if (k > t) break;
            float kv[4];
            load_row(kb + k * D.kv_ts, lane, kv, dv);
            float part = 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) part = fmaf(q[e], kv[e], part);
            acc += expf(warp_sum(part) * sc - lt);
        }
    }
    if (lane == 0) bmass[w] = acc / (static_cast<float>(D.b) * D.b);
}

// Bitonic sort of (key, id) pairs in shared memory, order: key descending, id ascending.
// Each pair is ONE 64-bit word: the high half is the key's bits mapped to an unsigned
// integer of the same order (sign set: all bits flipped; else the sign bit set), the low
// half ~id, so (key desc, id asc) is plain unsigned descending order and a compare-exchange
// is one 64-bit compare plus two selects.  A stage with stride <= 16 only pairs elements
// inside the 64-element segments a warp's 32 threads own (pair t: lo = 2t - t mod stride),
// so consecutive such stages need only a __syncwarp; cross-warp stages (stride >= 32) and
// the end of every merge size keep the block barrier.
__device__ __forceinline__ unsigned long long sort_word(float key, int id) {
    uint32_t u = __float_as_uint(key);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return (static_cast<unsigned long long>(u) << 32) | static_cast<uint32_t>(~static_cast<uint32_t>(id));
}
__device__ __forceinline__ int word_id(unsigned long long w) {
    return static_cast<int>(~static_cast<uint32_t>(w));
}
__device__ __forceinline__ float word_key(unsigned long long w) {
    const uint32_t u = static_cast<uint32_t>(w >> 32);
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}
__device__ void bitonic_sort(unsigned long long* v, int P) {
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                const int lo = 2 * t - (t & (stride - 1));
                const int hi = lo + stride;
                const unsigned long long a = v[lo], b = v[hi];
                const unsigned long long mx = a > b ? a : b, mn = a > b ? b : a;
                const bool desc = ((lo & size) == 0);   // this half of the merge runs descending
                v[lo] = desc ? mx : mn;
                v[hi] = desc ? mn : mx;
            }
            if (stride > 16) __syncthreads();
            else __syncwarp();
        }
        __syncthreads();
    }
}

__host__ __device__ __forceinline__ int next_pow2(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

// Alg. 1 lines 3-4: one CTA per local head.
__global__ void budget_finalize_kernel(Dims D, const float* __restrict__ bmass,
                                       int* __restrict__ kstar, float* __restrict__ budget) {
    extern __shared__ unsigned char sm[];
    const int P = next_pow2(D.M);
    unsigned long long* v = reinterpret_cast<unsigned long long*>(sm);
    float* key = reinterpret_cast<float*>(v + P);   // the masses in descending order
    const int hl = blockIdx.x;
    for (int n = threadIdx.x; n < P; n += blockDim.x)
        v[n] = sort_word((n < D.M) ? bmass[static_cast<long long>(hl) * D.M + n] : -1.f, n);  // pads last
    __syncthreads();
    bitonic_sort(v, P);
    for (int j = threadIdx.x; j < D.M; j += blockDim.x) key[j] = word_key(v[j]);
    __syncthreads();
    // Alg. 1 lines 3-4 in parallel: contiguous chunks of the descending order per thread,
    // a deterministic block scan of the chunk sums (T = total), then the first prefix
    // k with P(k) >= gamma * T (a min-reduction over the threads' candidates).
    __shared__ float warp_sums[32];
    __shared__ int kmin;
    const int nthr = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int per = (D.M + nthr - 1) / nthr;
    const int j0 = min(tid * per, D.M), j1 = min(j0 + per, D.M);
    float local = 0.f;
    for (int j = j0; j < j1; ++j) local += key[j];
    float incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sums[wid] = incl;
    if (tid == 0) kmin = D.M;
    __syncthreads();
    if (wid == 0) {
        float w = lane < (nthr >> 5) ? warp_sums[lane] : 0.f;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += v;
        }
        warp_sums[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    const float T = warp_sums[(nthr >> 5) - 1];
    float run = incl - local + (wid > 0 ? warp_sums[wid - 1] : 0.f);  // exclusive prefix
    if (D.gamma < 1.f) {
        const float target = D.gamma * T;
        for (int j = j0; j < j1; ++j) {
            run += key[j];
            if (run >= target) {
                atomicMin(&kmin, j + 1);  // integer min: order-independent
                break;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const int ks = D.gamma < 1.f ? kmin : D.M;
        kstar[hl] = ks;
        budget[hl] = static_cast<float>(ks) / D.M;
    }
}

// ------------------------------------------------------------------- A5-A6 --
// One CTA per (local group c, block row m).  Sorts columns 0..m-1 of the shared score row
// by (L desc, index asc) once, then each head of the group keeps the first K_{h,m}-1 of
// that order plus the diagonal, emitted ascending (nested prefixes).
// per_head (the seq-avgpool comparator): L holds one score map per LOCAL head, c = local head.
__global__ void select_kernel(Dims D, const float* __restrict__ L, const int* __restrict__ kstar,
                              int* __restrict__ block_cnt, int* __restrict__ block_idx, int per_head) {
    extern __shared__ unsigned char sm[];
    const int nr = D.re - D.rb;                  // block rows [rb, re) (all by default)
    const int c = blockIdx.x / nr;
    const int m = D.re - 1 - (blockIdx.x % nr);  // long rows first
    const int P = next_pow2(max(m, 1));
    unsigned long long* v = reinterpret_cast<unsigned long long*>(sm);
    int* rank = reinterpret_cast<int*>(v + next_pow2(D.M));
    const float* row = L + (static_cast<long long>(c) * D.M + m) * D.M;
    const bool sink = has_flag(D, PROXYATTN_FLAG_FORCE_SINK);
    for (int n = threadIdx.x; n < P; n += blockDim.x)   // forced sink first; pads (id INT_MAX) last
        v[n] = (n < m) ? sort_word((sink && n == 0) ? INFINITY : row[n], n) : sort_word(-INFINITY, INT_MAX);
    __syncthreads();
    if (m > 1) bitonic_sort(v, P);
    for (int p = threadIdx.x; p < m; p += blockDim.x) rank[word_id(v[p])] = p;
    __syncthreads();

    const int grp = D.gb + c;
    const int h0 = per_head ? D.qb + c : max(grp * D.gq, D.qb);
    const int h1 = per_head ? h0 + 1 : min((grp + 1) * D.gq, D.qe);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // One warp per head: ballot compaction of {n <= m : n == m or rank[n] < K - 1}.
    for (int h = h0 + wid; h < h1; h += nw) {
        const int hl = h - D.qb;
        const int K = row_count(D, kstar[hl], m);
        const int keep = K - 1;  // non-diagonal blocks kept (diagonal forced, Z15)
        int* out = block_idx + (static_cast<long long>(hl) * D.M + m) * D.M;
        int base = 0;
        for (int n0 = 0; n0 <= m; n0 += 32) {
            const int n = n0 + lane;
            const bool f = (n <= m) && (n == m || rank[n] < keep);
            const unsigned bal = __ballot_sync(0xffffffffu, f);
            if (f) out[base + __popc(bal & ((1u << lane) - 1u))] = n;
            base += __popc(bal);
        }
        if (lane == 0) block_cnt[static_cast<long long>(hl) * D.M + m] = K;
    }
}

// Device-side list validation (PROXYATTN_FLAG_CHECK): counts rows whose list is empty,
// not strictly ascending, out of range, acausal or missing... (S:319 contract).
__global__ void check_lists_kernel(Dims D, const int* __restrict__ cnt, const int* __restrict__ idx,
                                   int* bad) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<long long>(D.Hl) * D.M) return;
    const int m = static_cast<int>(i % D.M);
    const int k = cnt[i];
    bool ok = (k >= 1 && k <= m + 1);
    const int* l = idx + i * D.M;
    for (int u = 0; ok && u < k; ++u) {
        const int n = l[u];
        if (n < 0 || n > m || (u > 0 && n <= l[u - 1])) ok = false;
    }
    if (!ok) atomicAdd(bad, 1);
}

inline unsigned blocks_for(long long threads, int bs) {
    return static_cast<unsigned>((threads + bs - 1) / bs);
}

}  // namespace

cudaError_t launch_pool(const Dims& D, const void* Q, const void* K, float* qsum, float* ksum,
                        void* Pq, void* Pk, cudaStream_t st, long long q_i0, long long i_end) {
    if (i_end < 0) i_end = D.Ns;
    const long long thr = static_cast<long long>(D.gl) * D.Ns * 32;
    if (D.fp32)
        pool_kernel<float><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const float*>(Q), static_cast<const float*>(K), qsum, ksum,
            static_cast<float*>(Pq), static_cast<float*>(Pk), q_i0, i_end);
    else if (D.d % 8 == 0 && (qsum == nullptr) == (ksum == nullptr) && (Pq == nullptr) == (Pk == nullptr)) {
        const long long t2 = static_cast<long long>(D.gl) * D.Ns * (D.d / 8);
        pool_bf16_kernel<<<blocks_for(t2, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(K), qsum,
            ksum, static_cast<__nv_bfloat16*>(Pq), static_cast<__nv_bfloat16*>(Pk), q_i0, i_end);
    } else
        pool_kernel<__nv_bfloat16><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(K), qsum,
            ksum, static_cast<__nv_bfloat16*>(Pq), static_cast<__nv_bfloat16*>(Pk), q_i0, i_end);
    return cudaGetLastError();
}

cudaError_t launch_round_proxies(const Dims& D, const float* qsum, const float* ksum, void* Pq,
                                 void* Pk, cudaStream_t st) {
    const long long n = static_cast<long long>(D.gl) * D.Ns * D.d;
    if (D.fp32)
        round_kernel<float><<<blocks_for(n, 256), 256, 0, st>>>(n, qsum, ksum,
                                                               static_cast<float*>(Pq),
                                                               static_cast<float*>(Pk));
    else
        round_kernel<__nv_bfloat16><<<blocks_for(n, 256), 256, 0, st>>>(
            n, qsum, ksum, static_cast<__nv_bfloat16*>(Pq), static_cast<__nv_bfloat16*>(Pk));
    return cudaGetLastError();
}

static float proxy_scale(const Dims& D) {
    // Eq. 2 means folded into the logit scale: 1/(|Gq| |Gk| sqrt(d)) (Z2, Z5); a designated
    // head is used as is: 1/sqrt(d)
    if (has_flag(D, PROXYATTN_FLAG_DESIGNATED_HEAD)) return rsqrtf(static_cast<float>(D.d));
    return 1.0f / (static_cast<float>(D.gq) * static_cast<float>(D.gk) *
                   sqrtf(static_cast<float>(D.d)));
}

__global__ void static_budget_kernel(int Hl, int M, int ks, int* kstar, float* budget) {
    const int h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h < Hl) {
        const int k = ks < M ? ks : M;
        kstar[h] = k;
        budget[h] = static_cast<float>(k) / M;
    }
}

cudaError_t launch_static_budget(const Dims& D, int* kstar, float* budget, cudaStream_t st) {
    static_budget_kernel<<<(D.Hl + 127) / 128, 128, 0, st>>>(D.Hl, D.M, D.static_kstar, kstar, budget);
    return cudaGetLastError();
}

cudaError_t launch_proxy_lse(const Dims& D, const void* Pq, const void* Pk, float* lse,
                             cudaStream_t st) {
    const long long thr = static_cast<long long>(D.gl) * D.Ns * 32;
    const float sc = proxy_scale(D);
    if (D.fp32)
        proxy_lse_simt<float><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const float*>(Pq), static_cast<const float*>(Pk), sc, lse);
    else
        proxy_lse_simt<__nv_bfloat16><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Pq), static_cast<const __nv_bfloat16*>(Pk), sc,
            lse);
    return cudaGetLastError();
}

cudaError_t launch_proxy_maxpool(const Dims& D, const void* Pq, const void* Pk, const float* lse,
                                 float* L, cudaStream_t st) {
    const long long thr = static_cast<long long>(D.gl) * D.M * D.M * 32;
    const float sc = proxy_scale(D);
    if (D.fp32)
        proxy_maxpool_simt<float><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const float*>(Pq), static_cast<const float*>(Pk), sc, lse, L);
    else
        proxy_maxpool_simt<__nv_bfloat16><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Pq), static_cast<const __nv_bfloat16*>(Pk), sc,
            lse, L);
    return cudaGetLastError();
}

cudaError_t launch_budget_lse(const Dims& D, const void* Q, const void* K, float* blse,
                              cudaStream_t st) {
    const long long thr = static_cast<long long>(D.Hl) * D.b * 32;
    if (D.fp32)
        budget_lse_simt<float><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const float*>(Q), static_cast<const float*>(K), blse);
    else
        budget_lse_simt<__nv_bfloat16><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(K), blse);
    return cudaGetLastError();
}

cudaError_t launch_budget_mass(const Dims& D, const void* Q, const void* K, const float* blse,
                               float* bmass, cudaStream_t st) {
    const long long thr = static_cast<long long>(D.Hl) * D.M * 32;
    if (D.fp32)
        budget_mass_simt<float><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const float*>(Q), static_cast<const float*>(K), blse, bmass);
    else
        budget_mass_simt<__nv_bfloat16><<<blocks_for(thr, 256), 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Q), static_cast<const __nv_bfloat16*>(K), blse,
            bmass);
    return cudaGetLastError();
}

cudaError_t launch_budget_finalize(const Dims& D, const float* bmass, int* kstar, float* budget,
                                   cudaStream_t st) {
    const int P = next_pow2(D.M);
    const size_t sm = static_cast<size_t>(P) * 12;   // 64-bit sort words + the sorted masses
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(budget_finalize_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    budget_finalize_kernel<<<D.Hl, 512, sm, st>>>(D, bmass, kstar, budget);
    return cudaGetLastError();
}

cudaError_t launch_select(const Dims& D, const float* L, const int* kstar, int* block_cnt,
                          int* block_idx, cudaStream_t st, bool per_head) {
    const int P = next_pow2(D.M);
    const size_t sm = static_cast<size_t>(P) * 4 * 3;
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    select_kernel<<<(per_head ? D.Hl : D.gl) * (D.re - D.rb), 512, sm, st>>>(D, L, kstar, block_cnt, block_idx,
                                                                           per_head ? 1 : 0);
    return cudaGetLastError();
}

// ------------------------------------------------------------ CHECK_FINITE --
// S:37 ("all values finite"), S:49 / S:319 ("non-finite input -> validation error"): counts
// the elements whose exponent field is all ones (NaN or +-Inf).  Element e of run r lives at
// p[r * row_stride + e].  Grid-stride, 8 bf16 / 4 fp32 per 16-byte load when aligned.
template <bool kF32>
__global__ void count_nonfinite_kernel(const void* __restrict__ p, long long rows, long long row_elems,
                                       long long row_stride, int* __restrict__ bad) {
    constexpr int kVec = kF32 ? 4 : 8;
    const bool vec = (row_elems % kVec == 0) && (row_stride % kVec == 0) &&
                     (reinterpret_cast<uintptr_t>(p) % 16 == 0);
    const long long per_row = vec ? row_elems / kVec : row_elems;
    const long long total = rows * per_row;
    int n = 0;
    for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const long long r = i / per_row, c = i % per_row;
        if (vec) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(p) + (r * row_stride) / kVec + c);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (kF32) n += (w[k] & 0x7f800000u) == 0x7f800000u;
                else n += ((w[k] & 0x7f80u) == 0x7f80u) + ((w[k] & 0x7f800000u) == 0x7f800000u);
            }
        } else if (kF32) {
            const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(p) + r * row_stride + c);
            n += (w & 0x7f800000u) == 0x7f800000u;
        } else {
            const unsigned short w = __ldg(reinterpret_cast<const unsigned short*>(p) + r * row_stride + c);
            n += (w & 0x7f80u) == 0x7f80u;
        }
    }
    n = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(bad, n);
}

cudaError_t launch_check_lists(const Dims& D, const int* block_cnt, const int* block_idx,
                               int* bad_out, cudaStream_t st) {
    const long long n = static_cast<long long>(D.Hl) * D.M;
    check_lists_kernel<<<blocks_for(n, 256), 256, 0, st>>>(D, block_cnt, block_idx, bad_out);
    return cudaGetLastError();
}

cudaError_t launch_count_nonfinite(const void* p, bool fp32, long long rows, long long row_elems,
                                   long long row_stride, int* bad, cudaStream_t st) {
    if (rows <= 0 || row_elems <= 0) return cudaSuccess;
    const long long n = rows * row_elems;
    const unsigned grid = static_cast<unsigned>(std::min<long long>((n + 2047) / 2048, 148 * 16));
    if (fp32) count_nonfinite_kernel<true><<<grid, 256, 0, st>>>(p, rows, row_elems, row_stride, bad);
    else count_nonfinite_kernel<false><<<grid, 256, 0, st>>>(p, rows, row_elems, row_stride, bad);
    return cudaGetLastError();
}

}  // namespace pa
