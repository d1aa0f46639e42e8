// common.cuh — derived configuration shared by the host API and the kernels of libproxyattn.
#pragma once

// A7 at d = b = 128 runs the row-pair kernel (attn_tc9.cu); 0 selects attn_tc8 everywhere
// (a build define for A/B timing, not a runtime switch)
#ifndef PA_ATTN_V9
#define PA_ATTN_V9 1
#endif
// ... and for the dense A8 (diagonal-first walk over both rows of a pair): 109.4-110.7 vs
// 111.4-111.5 ms for attn_tc8 at 128K, no exact re-runs (profiles/r03_dense_v9_ab.jsonl)
#ifndef PA_ATTN_V9_DENSE
#define PA_ATTN_V9_DENSE 1
#endif
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <set>
#include <utility>

#include "../../include/proxyattn.h"

namespace pa {

// Everything a kernel needs, derived once on the host from proxyattn_cfg (O1 of SURVEY §8c).
struct Dims {
    int Hq, Hkv, d, b, s, g;
    int r;        // Hq / Hkv (GQA ratio)
    int M;        // N / b block rows
    int bs;       // b / s sampled rows per block
    int qb, qe;   // local query-head shard [qb, qe)
    int Hl;       // qe - qb
    int kvb;      // first local kv head = qb / r
    int Hkvl;     // Hl / r
    int gb, gl;   // first touched group, number of touched groups
    int gq, gk;   // query heads / kv heads per group (|G| of Eq. 2 for Q and K, Z2)
    int F;        // ceil(min_budget_tokens / b), per-row floor (Z14)
    long long N, Ns;
    float gamma;
    uint32_t flags;
    bool fp32;    // FP32_DEBUG
    int static_kstar;   // > 0: static top-K baseline (Alg. 1 skipped)
    int rb, re;         // prefill block-row range [rb, re)
    // Q/O and K/V element strides (local head, token): head-major (d, N d) by default,
    // token-major (token stride, d) with PROXYATTN_FLAG_TOKEN_MAJOR
    bool tok;
    long long q_hs, q_ts, kv_hs, kv_ts;
};

// Element offset of (local query head hl, token t) in Q / O, and of (local kv head, t) in K / V.
__host__ __device__ __forceinline__ long long q_off(const Dims& D, int hl, long long t) {
    return static_cast<long long>(hl) * D.q_hs + t * D.q_ts;
}
__host__ __device__ __forceinline__ long long kv_off(const Dims& D, int kvl, long long t) {
    return static_cast<long long>(kvl) * D.kv_hs + t * D.kv_ts;
}

__host__ __device__ __forceinline__ bool has_flag(const Dims& D, uint32_t f) { return (D.flags & f) != 0; }

// Query-head h (global) -> proxy group (groups aligned with the keys, Z3).
__host__ __device__ __forceinline__ int group_of_q(const Dims& D, int h) {
    return (h / D.r) / (D.Hkv / D.g);
}

// Eq. 3 row count under reading Z12: K_{h,m} = min(m+1, max(ceil(K* (m+1)/M), F, 1)).
__host__ __device__ __forceinline__ int row_count(const Dims& D, int kstar, int m) {
    long long k = (D.flags & PROXYATTN_FLAG_CONSTANT_K)
                      ? (long long)kstar                                  // Z12 alternative
                      : ((long long)kstar * (m + 1) + D.M - 1) / D.M;
    if (k < D.F) k = D.F;
    if (k < 1) k = 1;
    if (k > m + 1) k = m + 1;
    return static_cast<int>(k);
}

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

template <typename T>
__device__ __forceinline__ T from_f64(double x);
template <>
__device__ __forceinline__ float from_f64<float>(double x) { return static_cast<float>(x); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f64<__nv_bfloat16>(double x) { return __double2bfloat16(x); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: set it once per
// (kernel, device) pair, thread-safely (one process may drive several GPUs).
inline cudaError_t ensure_smem_attr(const void* fn, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({fn, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({fn, dev});
    return e;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// Workspace carve-up of proxyattn_estimate (all offsets 256-B aligned).
struct Workspace {
    size_t pq, pk, lse, L, blse, bmass, scratch, scratch_b, total;
};
size_t score_tc_scratch_bytes(const Dims& D);
size_t score_tc_budget_scratch_bytes(const Dims& D);
bool score_tc_supported(const Dims& D);
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
inline Workspace workspace_layout(const Dims& D) {
    Workspace w{};
    const size_t el = D.fp32 ? 4 : 2;
    size_t off = 0;
    w.pq = off;    off = align256(off + (size_t)D.gl * D.Ns * D.d * el);
    w.pk = off;    off = align256(off + (size_t)D.gl * D.Ns * D.d * el);
    w.lse = off;   off = align256(off + (size_t)D.gl * D.Ns * 4);
    w.L = off;     off = align256(off + (size_t)D.gl * D.M * D.M * 4);
    w.blse = off;  off = align256(off + (size_t)D.Hl * D.b * 4);
    w.bmass = off; off = align256(off + (size_t)D.Hl * D.M * 4);
    w.scratch = off; off = align256(off + (score_tc_supported(D) ? score_tc_scratch_bytes(D) : 0));
    // Alg. 1's partials get their own region: the budget pass runs concurrently with A1-A3
    w.scratch_b = off; off = align256(off + (score_tc_supported(D) ? score_tc_budget_scratch_bytes(D) : 0));
    w.total = off;
    return w;
}

}  // namespace pa
