// avgpool.cu — the sequence-avgpool comparator (SPEC S:365-373
// seq_avgpool_scores): the coarse estimator the paper's granularity argument is measured
// against ("pooling methods along the sequence dimension for approximation", §2.1; the
// "few high-scoring positions ... overlooked" of §1).  Per query head h and block row m:
//   q̄_m = mean of block m's query rows of head h, k̄_n = mean of block n's key rows of kv(h),
//   score(m, n) = softmax over n <= m of q̄_m·k̄_n / sqrt(d).
// The same budgets (Alg. 1) and Eq. 3 selection then run on these per-head maps
// (proxyattn_avgpool_estimate), so the two estimators differ only in the score map.
//
// Kernels: block_pool_kernel reads Q and K once (HBM-bound: every token, unlike A1's strided
// proxies) and writes the block sums rounded once to bf16 (fp64 accumulation, as A1);
// avgpool_scores_kernel is a register-blocked FFMA2 tile (64 rows x 64 columns per CTA,
// d staged through shared memory in 32-element chunks) with an online (max, sum) per row.
#include <cuda_bf16.h>

#include <cfloat>

#include "common.cuh"
#include "kernels.h"
#include "sm100.cuh"

namespace pa {
namespace {

// One CTA (128 threads) per (pooled head, block): thread t owns 8 contiguous dimensions
// (d / 8 threads per row) of row group t / (d / 8); the row groups' fp64 partial sums are
// added in a fixed order through shared memory (deterministic).
template <typename T>
__global__ void block_pool_kernel(Dims D, const T* __restrict__ X, long long hs, long long ts, int n_heads,
                                  T* __restrict__ out) {
    __shared__ double part[16][128];
    const int head = blockIdx.x / D.M;
    const int m = blockIdx.x % D.M;
    if (head >= n_heads) return;
    const int tpr = D.d / 8;                        // threads per row
    const int groups = 128 / tpr;                   // rows in flight
    const int part_id = threadIdx.x % tpr, grp = threadIdx.x / tpr;
    const long long t0 = static_cast<long long>(m) * D.b;
    const long long t1 = t0 + D.b < D.N ? t0 + D.b : D.N;   // real rows of the (padded) last block
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (long long t = t0 + grp; t < t1; t += groups) {
        const T* row = X + static_cast<long long>(head) * hs + t * ts + part_id * 8;
        if constexpr (sizeof(T) == 2) {   // one 16-byte load of 8 bf16
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(row));
            const __nv_bfloat162* e2 = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 f = __bfloat1622float2(e2[q]);
                acc[2 * q] += f.x;
                acc[2 * q + 1] += f.y;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] += static_cast<double>(row[e]);
        }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) part[grp][part_id * 8 + e] = acc[e];
    __syncthreads();
    for (int e = threadIdx.x; e < D.d; e += blockDim.x) {
        double s = 0.0;
        for (int g = 0; g < groups; ++g) s += part[g][e];   // fixed order
        out[(static_cast<long long>(head) * D.M + m) * D.d + e] = from_f64<T>(s);
    }
}

constexpr int kTile = 64;      // rows and columns of a score tile
constexpr int kDc = 32;        // d chunk staged in shared memory

// CTA = (local head hl, 64-row tile).  Thread (ty, tx) of 16 x 16 owns rows ty + 16 i and
// columns tx + 16 j (i, j < 4), so a warp's column reads hit 16 distinct banks.
template <typename T>
__global__ void __launch_bounds__(256) avgpool_scores_kernel(Dims D, const T* __restrict__ Qb,
                                                              const T* __restrict__ Kb, float* __restrict__ z,
                                                              float* __restrict__ lse, int normalize) {
    __shared__ float qs[kTile][kDc + 1];
    __shared__ float ks[kTile][kDc + 1];
    const int n_mt = (D.M + kTile - 1) / kTile;
    const int hl = blockIdx.x / n_mt;
    const int mt = n_mt - 1 - blockIdx.x % n_mt;     // long rows first
    const int kvl = hl / D.r;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const float rsd = rsqrtf(static_cast<float>(D.d));
    const int last_cnt = static_cast<int>(D.N - static_cast<long long>(D.M - 1) * D.b);
    auto inv_cnt = [&](int blk) { return blk == D.M - 1 ? 1.f / last_cnt : 1.f / D.b; };
    float rmax[4], rsum[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) rmax[i] = -INFINITY, rsum[i] = 0.f;
    const T* qbase = Qb + (static_cast<long long>(hl) * D.M + mt * kTile) * D.d;
    for (int nt = 0; nt <= mt; ++nt) {
        const T* kbase = Kb + (static_cast<long long>(kvl) * D.M + nt * kTile) * D.d;
        uint64_t acc[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0ull;
        for (int d0 = 0; d0 < D.d; d0 += kDc) {
            __syncthreads();
            for (int e = threadIdx.x; e < kTile * kDc; e += blockDim.x) {
                const int rr = e / kDc, cc = e % kDc;
                const bool qv = mt * kTile + rr < D.M, kv = nt * kTile + rr < D.M;
                qs[rr][cc] = qv ? to_f32(qbase[static_cast<long long>(rr) * D.d + d0 + cc]) : 0.f;
                ks[rr][cc] = kv ? to_f32(kbase[static_cast<long long>(rr) * D.d + d0 + cc]) : 0.f;
            }
            __syncthreads();
#pragma unroll 8
            for (int k = 0; k < kDc; ++k) {
                const uint64_t k01 = f2_pack(ks[tx][k], ks[tx + 16][k]);
                const uint64_t k23 = f2_pack(ks[tx + 32][k], ks[tx + 48][k]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float q = qs[ty + 16 * i][k];
                    const uint64_t q2 = f2_pack(q, q);
                    acc[i][0] = f2_fma(q2, k01, acc[i][0]);
                    acc[i][1] = f2_fma(q2, k23, acc[i][1]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = mt * kTile + ty + 16 * i;
            if (m >= D.M) continue;
            float v[4];
            f2_unpack(acc[i][0], v[0], v[1]);
            f2_unpack(acc[i][1], v[2], v[3]);
            const float sm = inv_cnt(m) * rsd;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = nt * kTile + tx + 16 * j;
                if (n >= D.M) continue;
                float* dst = z + (static_cast<long long>(hl) * D.M + m) * D.M + n;
                if (n > m) {
                    *dst = -INFINITY;
                    continue;
                }
                const float x = v[j] * (sm * inv_cnt(n));
                *dst = x;
                const float nm = fmaxf(rmax[i], x);
                rsum[i] = rsum[i] * __expf(rmax[i] - nm) + __expf(x - nm);
                rmax[i] = nm;
            }
        }
    }
    // the 16 column threads of a row: (max, sum) combine, fixed xor order
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const float om = __shfl_xor_sync(0xffffffffu, rmax[i], o);
            const float os = __shfl_xor_sync(0xffffffffu, rsum[i], o);
            const float nm = fmaxf(rmax[i], om);
            rsum[i] = (rmax[i] == -INFINITY ? 0.f : rsum[i] * __expf(rmax[i] - nm)) +
                      (om == -INFINITY ? 0.f : os * __expf(om - nm));
            rmax[i] = nm;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = mt * kTile + ty + 16 * i;
        if (m >= D.M) continue;
        const float l = rmax[i] + logf(rsum[i]);
        if (tx == 0 && lse) lse[static_cast<long long>(hl) * D.M + m] = l;
        if (normalize) {
            float* row = z + (static_cast<long long>(hl) * D.M + m) * D.M;
            for (int n = tx; n <= m; n += 16) row[n] -= l;   // own writes above: same thread
        }
    }
}

}  // namespace

cudaError_t launch_block_pool(const Dims& D, const void* Q, const void* K, void* Qb, void* Kb,
                              cudaStream_t st) {
    if (D.d % 8 || D.d > 128) return cudaErrorInvalidValue;
    if (D.fp32) {
        block_pool_kernel<float><<<D.Hl * D.M, 128, 0, st>>>(D, static_cast<const float*>(Q), D.q_hs, D.q_ts, D.Hl,
                                                            static_cast<float*>(Qb));
        block_pool_kernel<float><<<D.Hkvl * D.M, 128, 0, st>>>(D, static_cast<const float*>(K), D.kv_hs, D.kv_ts,
                                                              D.Hkvl, static_cast<float*>(Kb));
    } else {
        block_pool_kernel<__nv_bfloat16><<<D.Hl * D.M, 128, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Q), D.q_hs, D.q_ts, D.Hl, static_cast<__nv_bfloat16*>(Qb));
        block_pool_kernel<__nv_bfloat16><<<D.Hkvl * D.M, 128, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(K), D.kv_hs, D.kv_ts, D.Hkvl, static_cast<__nv_bfloat16*>(Kb));
    }
    return cudaGetLastError();
}

cudaError_t launch_avgpool_scores(const Dims& D, const void* Qb, const void* Kb, float* z, float* lse,
                                  bool normalize, cudaStream_t st) {
    if (D.d % kDc) return cudaErrorInvalidValue;
    const unsigned grid = static_cast<unsigned>(D.Hl) * ((D.M + kTile - 1) / kTile);
    if (D.fp32)
        avgpool_scores_kernel<float><<<grid, 256, 0, st>>>(D, static_cast<const float*>(Qb),
                                                          static_cast<const float*>(Kb), z, lse, normalize);
    else
        avgpool_scores_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
            D, static_cast<const __nv_bfloat16*>(Qb), static_cast<const __nv_bfloat16*>(Kb), z, lse, normalize);
    return cudaGetLastError();
}

}  // namespace pa
