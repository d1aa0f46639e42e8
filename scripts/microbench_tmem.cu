// Microbenchmark of the attention softmax's inner loop on sm_100a WITHOUT barriers or MMAs:
// W warps (W/4 per SMSP, warp w reads TMEM lanes 32*(w%4)..+31) each loop over "blocks" of
// 128 fp32 S columns in 32-column chunks exactly as attn_tc8's block_exps does (tcgen05.ld
// x32 double-buffered, FFMA2 scale-and-shift, ex2, FADD2 row sum, F2FP pack, tcgen05.st x16
// into a P region), and report clk per block per SM (one block = 128 lanes x 128 columns,
// i.e. the S tile of one (head, row, block) unit; 1024 clk = the tensor time of that unit).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2509_24745_b200/csrc \
//        -o /tmp/mbt scripts/microbench_tmem.cu && /tmp/mbt
// Modes: 0 full loop; 1 without MUFU (P = x); 2 without the TMEM loads (registers reused);
// 3 TMEM loads only (x32, wait per chunk); 4 TMEM stores only; 5 full loop, loads not
// double-buffered; 6 full loop, 1/4 of the exp2s on the FMA-pipe cubic; 7 full loop with the
// bf16 RNE pack on the integer pipe instead of F2FP; 8 no pack; 9 truncating PRMT pack;
// 10 round-half-up integer pack (IADD + PRMT).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace pa;

constexpr int kBlocks = 2048;   // blocks per warp-group pass

template <int kMode>
__global__ void __launch_bounds__(256, 1) k(float* out, long long* cyc, float sc) {
    __shared__ uint32_t tbase_s;
    const int warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    if (warp == 0) tmem_alloc(&tbase_s, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = tbase_s;
    const int quarter = warp & 3;
    const int grp = warp >> 2;                 // warp group: its own S region (up to 2)
    const uint32_t lane_off = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t tS = tbase + lane_off + 128 + (grp & 1) * 128;
    const uint32_t tP = tbase + lane_off + 384 + (grp & 1) * 64;
    const uint64_t sc2 = f2_pack(sc, sc);
    float acc = 0.f;
    uint32_t xb[2][32];
#pragma unroll
    for (int e = 0; e < 32; ++e) xb[0][e] = xb[1][e] = __float_as_uint(0.001f * e);
    __syncthreads();
    const long long t0 = clock64();
    for (int blk = 0; blk < kBlocks; ++blk) {
        uint64_t ls[4] = {0ull, 0ull, 0ull, 0ull};
        const uint64_t nm2 = f2_pack(-1.f - 1e-6f * blk, -1.f - 1e-6f * blk);   // loop-variant
        if (kMode == 3) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                tmem_ld32(tS + 32 * c, xb[c & 1]);
                tmem_ld_wait_regs(xb[c & 1]);
                acc += __uint_as_float(xb[c & 1][c]);
            }
            continue;
        }
        if (kMode == 4) {
            uint32_t pk[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) pk[e] = xb[0][e] + blk;
#pragma unroll
            for (int c = 0; c < 4; ++c) tmem_st16(tP + 16 * c, pk);
            tmem_st_wait();
            continue;
        }
        if (kMode != 2 && kMode != 5) tmem_ld32(tS, xb[0]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (kMode == 5) {
                tmem_ld32(tS + 32 * c, xb[c & 1]);
                tmem_ld_wait_regs(xb[c & 1]);
            } else if (kMode != 2) {
                tmem_ld_wait_regs(xb[c & 1]);
                if (c + 1 < 4) tmem_ld32(tS + 32 * (c + 1), xb[(c + 1) & 1]);
            }
            uint32_t pk[16];
#pragma unroll
            for (int p = 0; p < 16; ++p) {
                const uint64_t x2 = f2_fma(f2_pack(__uint_as_float(xb[c & 1][2 * p]), __uint_as_float(xb[c & 1][2 * p + 1])),
                                           sc2, nm2);
                float p0, p1;
                if (kMode == 6 && (p & 7) < 2) {
                    ex2_poly2(x2, p0, p1);
                } else {
                    float x0, x1;
                    f2_unpack(x2, x0, x1);
                    if (kMode == 1) {
                        p0 = x0;
                        p1 = x1;
                    } else {
                        p0 = ex2(x0);
                        p1 = ex2(x1);
                    }
                }
                ls[p & 3] = f2_add(ls[p & 3], f2_pack(p0, p1));
                if (kMode == 7) {          // RNE to bf16 on the integer pipe
                    const uint32_t u0 = __float_as_uint(p0), u1 = __float_as_uint(p1);
                    const uint32_t r0 = u0 + 0x7fffu + ((u0 >> 16) & 1u);
                    const uint32_t r1 = u1 + 0x7fffu + ((u1 >> 16) & 1u);
                    pk[p] = __byte_perm(r0, r1, 0x7632);
                } else if (kMode == 8) {   // no pack at all (upper bound)
                    pk[p] = __float_as_uint(p0) ^ __float_as_uint(p1);
                } else if (kMode == 10) {  // round half up (differs from RNE on exact ties only)
                    pk[p] = __byte_perm(__float_as_uint(p0) + 0x8000u, __float_as_uint(p1) + 0x8000u, 0x7632);
                } else if (kMode == 9) {   // truncation: one PRMT
                    pk[p] = __byte_perm(__float_as_uint(p0), __float_as_uint(p1), 0x7632);
                } else {
                    pk[p] = pack_bf16(p0, p1);
                }
            }
            tmem_st16(tP + 16 * c, pk);
            if (c & 1) tmem_st_wait();
        }
        const uint64_t t = f2_add(f2_add(ls[0], ls[1]), f2_add(ls[2], ls[3]));
        float a, b;
        f2_unpack(t, a, b);
        acc += a + b;
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tbase, 512);
    (void)nw;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, sizeof(float) * sms * 512);
    cudaMalloc(&cyc, sizeof(long long) * sms);
    const char* names[] = {"full loop", "no MUFU", "no TMEM ld", "TMEM ld only", "TMEM st only",
                           "full, ld not overlapped", "full, 1/4 poly exp2",
                           "full, ALU RNE pack", "full, no pack", "full, PRMT trunc pack",
                           "full, half-up pack"};
    for (int warps : {4, 8}) {
        for (int mode = 0; mode < 11; ++mode) {
            auto run = [&]() {
                switch (mode) {
                    case 0: k<0><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 1: k<1><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 2: k<2><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 3: k<3><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 4: k<4><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 5: k<5><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 6: k<6><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 7: k<7><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 8: k<8><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 9: k<9><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                    case 10: k<10><<<sms, warps * 32>>>(out, cyc, 0.1f); break;
                }
            };
            run();
            cudaDeviceSynchronize();
            run();
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
            long long c0 = 0;
            cudaMemcpy(&c0, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
            // each warp group (4 warps = 128 lanes) processes kBlocks blocks
            const double blocks_per_sm = static_cast<double>(kBlocks) * (warps / 4);
            printf("warps %2d  %-26s  %8.1f clk per 128x128 block per SM\n", warps, names[mode],
                   c0 / blocks_per_sm);
        }
    }
    return 0;
}
