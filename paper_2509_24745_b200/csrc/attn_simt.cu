// attn_simt.cu — FP32_DEBUG block-sparse / dense causal attention (A7/A8):
// one warp per query row, fp32 online softmax (FFMA + expf).  This is the 1e-4 parity
// build of the north star, not the bf16 product kernel (attn_tc.cu).
#include "common.cuh"
#include "kernels.h"

namespace pa {
namespace {

__global__ void attn_simt_kernel(Dims D, const float* __restrict__ Q, const float* __restrict__ K,
                                 const float* __restrict__ V, const int* __restrict__ block_cnt,
                                 const int* __restrict__ block_idx, float* __restrict__ O) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= static_cast<long long>(D.Hl) * D.N) return;
    const int hl = static_cast<int>(w / D.N);
    const long long t = w % D.N;
    const int m = static_cast<int>(t / D.b);
    if (m < D.rb || m >= D.re) return;                      // outside the requested row range
    const int dv = D.d >> 5;
    const float sc = rsqrtf(static_cast<float>(D.d));
    const long long kvoff = kv_off(D, hl / D.r, 0);
    const long long qoff = q_off(D, hl, t);
    float q[4], o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = (j < dv) ? Q[qoff + lane * dv + j] : 0.f;
    const bool dense = (block_cnt == nullptr);
    const long long row = static_cast<long long>(hl) * D.M + m;
    const int cnt = dense ? m + 1 : block_cnt[row];
    const int* list = dense ? nullptr : block_idx + row * D.M;
    float mx = -INFINITY, l = 0.f;
    for (int u = 0; u < cnt; ++u) {
        const long long n = dense ? u : list[u];
        const long long kend = min((n + 1) * D.b, t + 1);  // causal mask inside the diagonal block
        for (long long k = n * D.b; k < kend; ++k) {
            const float* kr = K + kvoff + k * D.kv_ts + lane * dv;
            const float* vr = V + kvoff + k * D.kv_ts + lane * dv;
            float part = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) part = fmaf(q[j], (j < dv) ? kr[j] : 0.f, part);
            const float z = warp_sum(part) * sc;
            if (z > mx) {
                const float corr = expf(mx - z);
                l = l * corr + 1.f;
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = o[j] * corr + ((j < dv) ? vr[j] : 0.f);
                mx = z;
            } else {
                const float p = expf(z - mx);
                l += p;
#pragma unroll
                for (int j = 0; j < 4; ++j) o[j] = fmaf(p, (j < dv) ? vr[j] : 0.f, o[j]);
            }
        }
    }
    const float inv = 1.f / l;
    for (int j = 0; j < dv; ++j) O[qoff + lane * dv + j] = o[j] * inv;
}

}  // namespace

cudaError_t launch_attn_simt(const Dims& D, const void* Q, const void* K, const void* V,
                             const int* block_cnt, const int* block_idx, void* O,
                             cudaStream_t st) {
    const long long thr = static_cast<long long>(D.Hl) * D.N * 32;
    const unsigned grid = static_cast<unsigned>((thr + 255) / 256);
    attn_simt_kernel<<<grid, 256, 0, st>>>(D, static_cast<const float*>(Q),
                                           static_cast<const float*>(K),
                                           static_cast<const float*>(V), block_cnt, block_idx,
                                           static_cast<float*>(O));
    return cudaGetLastError();
}

}  // namespace pa
