// api.cu — the extern "C" boundary of libproxyattn (include/proxyattn.h): validation,
// workspace carve-up and kernel launches.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdarg>
#include <initializer_list>
#include <map>
#include <tuple>
#include <mutex>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "../../include/proxyattn.h"
#include "common.cuh"
#include "kernels.h"

// A7 kernel choice: the row-pair attn_tc9 at d = b = 128 (PA_ATTN_V9, common.cuh), else attn_tc8
static bool use_v9(int d, int b) { return PA_ATTN_V9 && b == 128 && d == 128; }


namespace {

thread_local std::string g_err;

// NVTX range per method stage: host-side ranges around each stage's launches, so
// a profiler attributes kernels to A1-A8 (nvtx3 is header-only and costs nothing when no
// tool is attached).
struct Nvtx {
    explicit Nvtx(const char* name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(PROXYATTN_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define PA_CUDA(expr, where)                      \
    do {                                          \
        cudaError_t _e = (expr);                  \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

constexpr int kMaxBlocks = 16384;

// O1: validate the config and derive every size the kernels need.
int derive(const proxyattn_cfg* c, pa::Dims& D, bool limit_m = true) {
    if (!c) return fail(PROXYATTN_E_CONFIG, "cfg is NULL");
    if (c->n_q_heads <= 0 || c->n_kv_heads <= 0 || c->head_dim <= 0 || c->seq_len <= 0 ||
        c->block_size <= 0 || c->stride <= 0 || c->n_groups <= 0)
        return fail(PROXYATTN_E_CONFIG, "non-positive dimension");
    if (c->n_q_heads % c->n_kv_heads)
        return fail(PROXYATTN_E_CONFIG, "n_q_heads %% n_kv_heads != 0 (S:30)");
    if (c->n_kv_heads % c->n_groups)
        return fail(PROXYATTN_E_CONFIG, "n_kv_heads %% n_groups != 0 (S:31)");
    if (c->block_size % c->stride)
        return fail(PROXYATTN_E_CONFIG, "block_size %% stride != 0 (S:32)");
    if (!(c->gamma > 0.f && c->gamma <= 1.f))
        return fail(PROXYATTN_E_CONFIG, "gamma must be in (0, 1] (S:33)");
    if (c->min_budget_tokens < 0) return fail(PROXYATTN_E_CONFIG, "min_budget_tokens < 0");
    D.fp32 = (c->flags & PROXYATTN_FLAG_FP32_DEBUG) != 0;
    if (D.fp32) {
        if (c->head_dim % 32 || c->head_dim > 128)
            return fail(PROXYATTN_E_UNSUPPORTED, "FP32_DEBUG needs head_dim %% 32 == 0 and <= 128");
    } else {
        if (c->head_dim != 64 && c->head_dim != 128)
            return fail(PROXYATTN_E_UNSUPPORTED, "bf16 build needs head_dim 64 or 128");
        if (c->block_size != 64 && c->block_size != 128)
            return fail(PROXYATTN_E_UNSUPPORTED, "bf16 build needs block_size 64 or 128");
    }
    // A4/A6 sort one head's / one row's M block scores in shared memory (next_pow2(M) x 12 B
    // <= 227 KB): M <= 16384, i.e. N <= 2M tokens at b = 128, 1M at b = 64
    if (limit_m && (c->seq_len + c->block_size - 1) / c->block_size > kMaxBlocks)
        return fail(PROXYATTN_E_UNSUPPORTED, "seq_len / block_size > %d blocks", kMaxBlocks);
    D.Hq = c->n_q_heads;
    D.Hkv = c->n_kv_heads;
    D.d = c->head_dim;
    D.b = c->block_size;
    D.s = c->stride;
    D.g = c->n_groups;
    D.r = D.Hq / D.Hkv;
    D.N = c->seq_len;
    D.M = static_cast<int>((D.N + D.b - 1) / D.b);   // last block zero-padded when b does not divide N
    D.Ns = (D.N + D.s - 1) / D.s;                    // sampled positions i*s < N
    D.bs = D.b / D.s;
    D.gamma = c->gamma;
    D.flags = c->flags;
    if (c->static_kstar < 0) return fail(PROXYATTN_E_CONFIG, "static_kstar < 0");
    D.static_kstar = c->static_kstar;
    D.rb = c->row_begin;
    D.re = c->row_end == 0 ? D.M : c->row_end;
    if (D.rb < 0 || D.re > D.M || D.rb >= D.re)
        return fail(PROXYATTN_E_CONFIG, "bad row range [%d, %d) of %d block rows", D.rb, D.re, D.M);
    D.F = (c->min_budget_tokens + D.b - 1) / D.b;
    D.gq = D.Hq / D.g;
    D.gk = D.Hkv / D.g;
    D.qb = c->q_head_begin;
    D.qe = c->q_head_end == 0 ? D.Hq : c->q_head_end;
    if (D.qb < 0 || D.qe > D.Hq || D.qb >= D.qe)
        return fail(PROXYATTN_E_CONFIG, "bad shard [%d, %d)", D.qb, D.qe);
    if (D.qb % D.r || D.qe % D.r)
        return fail(PROXYATTN_E_CONFIG, "shard must align to kv heads (r = %d)", D.r);
    D.Hl = D.qe - D.qb;
    D.kvb = D.qb / D.r;
    D.Hkvl = D.Hl / D.r;
    D.gb = pa::group_of_q(D, D.qb);
    D.gl = pa::group_of_q(D, D.qe - 1) - D.gb + 1;
    D.tok = (c->flags & PROXYATTN_FLAG_TOKEN_MAJOR) != 0;
    if (D.tok) {
        D.q_ts = c->q_token_stride ? c->q_token_stride : static_cast<long long>(D.Hl) * D.d;
        D.kv_ts = c->kv_token_stride ? c->kv_token_stride : static_cast<long long>(D.Hkvl) * D.d;
        if (D.q_ts < static_cast<long long>(D.Hl) * D.d || D.kv_ts < static_cast<long long>(D.Hkvl) * D.d)
            return fail(PROXYATTN_E_CONFIG, "token stride smaller than the local heads (%lld / %lld)",
                        D.q_ts, D.kv_ts);
        if (D.q_ts % 8 || D.kv_ts % 8)
            return fail(PROXYATTN_E_CONFIG, "token strides must be multiples of 8 elements (16-byte rows)");
        D.q_hs = D.kv_hs = D.d;
    } else {
        if (c->q_token_stride || c->kv_token_stride)
            return fail(PROXYATTN_E_CONFIG, "token strides need PROXYATTN_FLAG_TOKEN_MAJOR");
        D.q_ts = D.kv_ts = D.d;
        D.q_hs = D.kv_hs = D.N * D.d;
    }
    return PROXYATTN_OK;
}

}  // namespace

namespace {

bool groups_complete(const pa::Dims& D) { return D.qb % D.gq == 0 && D.qe % D.gq == 0; }

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

template <typename T>
T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

int run_proxy_from_pooled(const pa::Dims& D, void* Pq, void* Pk, void* ws, const pa::Workspace& W,
                          float* L, cudaStream_t st, int tr0 = 0, int tr1 = -1) {
    float* lse = at<float>(ws, W.lse);
    if (pa::score_tc_supported(D)) {
        PA_CUDA(pa::launch_proxy_tc(D, Pq, Pk, at<float>(ws, W.scratch), lse, L, st, tr0, tr1), "proxy_tc");
        return PROXYATTN_OK;
    }
    PA_CUDA(pa::launch_proxy_lse(D, Pq, Pk, lse, st), "proxy_lse");
    PA_CUDA(pa::launch_proxy_maxpool(D, Pq, Pk, lse, L, st), "proxy_maxpool");
    return PROXYATTN_OK;
}

int run_budgets(const pa::Dims& D, const void* Q, const void* K, void* ws, const pa::Workspace& W,
                int32_t* kstar, float* budget, cudaStream_t st) {
    float* blse = at<float>(ws, W.blse);
    float* bmass = at<float>(ws, W.bmass);
    if (D.static_kstar > 0) {   // static top-K baseline (Fig. 6c): Alg. 1 is not run
        PA_CUDA(pa::launch_static_budget(D, kstar, budget, st), "static_budget");
        return PROXYATTN_OK;
    }
    if (pa::score_tc_supported(D)) {
        PA_CUDA(pa::launch_budget_tc(D, Q, K, at<float>(ws, W.scratch_b), bmass, st), "budget_tc");
    } else {
        PA_CUDA(pa::launch_budget_lse(D, Q, K, blse, st), "budget_lse");
        PA_CUDA(pa::launch_budget_mass(D, Q, K, blse, bmass, st), "budget_mass");
    }
    PA_CUDA(pa::launch_budget_finalize(D, bmass, kstar, budget, st), "budget_finalize");
    return PROXYATTN_OK;
}

// Library-owned helper streams (non-blocking), one set per (device, CALLER stream): work a
// call forks onto them is joined back to the caller's stream by events, so a graph captured
// on one caller stream never pulls in work of another thread using another stream.  Kinds:
// 0 = Alg. 1 of proxyattn_estimate (concurrent with A1-A3), 1 / 2 = the host path's upload /
// download streams, 3 = the second estimate stream of the packed varlen path.
int helper_stream(cudaStream_t caller, int kind, cudaStream_t* out) {
    static std::mutex mu;
    static std::map<std::tuple<int, cudaStream_t, int>, cudaStream_t> streams;
    int dev = 0;
    PA_CUDA(cudaGetDevice(&dev), "get device");
    std::lock_guard<std::mutex> lock(mu);
    cudaStream_t& s = streams[{dev, caller, kind}];
    if (!s) PA_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream create");
    *out = s;
    return PROXYATTN_OK;
}

// fork / join events of the calling thread on the current device (reused: record -> wait
// pairs are ordered on the host, and nothing is created or destroyed inside a capture)
struct AuxEvents {
    cudaEvent_t fork = nullptr, join = nullptr;
};
int estimate_events(AuxEvents* out) {
    thread_local std::map<int, AuxEvents> per_dev;
    int dev = 0;
    PA_CUDA(cudaGetDevice(&dev), "get device");
    AuxEvents& e = per_dev[dev];
    if (!e.fork) {
        PA_CUDA(cudaEventCreateWithFlags(&e.fork, cudaEventDisableTiming), "event create");
        PA_CUDA(cudaEventCreateWithFlags(&e.join, cudaEventDisableTiming), "event create");
    }
    *out = e;
    return PROXYATTN_OK;
}

// CHECK_FINITE ("all values finite"; "non-finite input -> validation error"):
// counts NaN / Inf elements of the listed tensors on the device, synchronises the stream and
// returns E_NONFINITE when any is found.  `q_role` tensors use the Q / O layout, the others K / V.
int check_finite(const pa::Dims& D, cudaStream_t st, std::initializer_list<std::pair<const void*, bool>> ts) {
    if (!(D.flags & PROXYATTN_FLAG_CHECK_FINITE)) return PROXYATTN_OK;
    int* bad = nullptr;
    PA_CUDA(cudaMallocAsync(&bad, sizeof(int), st), "check alloc");
    PA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st), "check memset");
    for (const auto& t : ts) {
        if (!t.first) continue;
        const bool q = t.second;
        const long long heads = q ? D.Hl : D.Hkvl;
        cudaError_t e = D.tok ? pa::launch_count_nonfinite(t.first, D.fp32, D.N, heads * D.d, q ? D.q_ts : D.kv_ts,
                                                           bad, st)
                              : pa::launch_count_nonfinite(t.first, D.fp32, 1, heads * D.N * D.d, 0, bad, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(bad, st);
            return cuda_fail(e, "count_nonfinite");
        }
    }
    int hbad = 0;
    PA_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "check copy");
    PA_CUDA(cudaFreeAsync(bad, st), "check free");
    PA_CUDA(cudaStreamSynchronize(st), "check sync");
    if (hbad) return fail(PROXYATTN_E_NONFINITE, "%d non-finite input elements (S:49, S:319)", hbad);
    return PROXYATTN_OK;
}

}  // namespace

extern "C" {

int proxyattn_workspace_bytes(const proxyattn_cfg* cfg, size_t* out) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!out) return fail(PROXYATTN_E_CONFIG, "out is NULL");
    *out = pa::workspace_layout(D).total;
    return PROXYATTN_OK;
}

int proxyattn_pool(const proxyattn_cfg* cfg, const void* Q, const void* K, float* qsum,
                   float* ksum, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!Q || !K || !qsum || !ksum) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    if ((rc = check_finite(D, S(stream), {{Q, true}, {K, false}}))) return rc;
    PA_CUDA(pa::launch_pool(D, Q, K, qsum, ksum, nullptr, nullptr, S(stream)), "pool");
    return PROXYATTN_OK;
}

int proxyattn_proxy_scores(const proxyattn_cfg* cfg, const float* qsum, const float* ksum,
                           void* ws, size_t ws_bytes, float* L, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    const pa::Workspace W = pa::workspace_layout(D);
    if (!ws || ws_bytes < W.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", W.total);
    if (!qsum || !ksum || !L) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    void* Pq = at<char>(ws, W.pq);
    void* Pk = at<char>(ws, W.pk);
    PA_CUDA(pa::launch_round_proxies(D, qsum, ksum, Pq, Pk, S(stream)), "round_proxies");
    return run_proxy_from_pooled(D, Pq, Pk, ws, W, L, S(stream));
}

int proxyattn_budgets(const proxyattn_cfg* cfg, const void* Q, const void* K, void* ws,
                      size_t ws_bytes, int32_t* kstar, float* budget, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    const pa::Workspace W = pa::workspace_layout(D);
    if (!ws || ws_bytes < W.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", W.total);
    if (!Q || !K || !kstar || !budget) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    if ((rc = check_finite(D, S(stream), {{Q, true}, {K, false}}))) return rc;
    return run_budgets(D, Q, K, ws, W, kstar, budget, S(stream));
}

int proxyattn_select(const proxyattn_cfg* cfg, const float* L, const int32_t* kstar,
                     int32_t* block_cnt, int32_t* block_idx, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!L || !kstar || !block_cnt || !block_idx) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    PA_CUDA(pa::launch_select(D, L, kstar, block_cnt, block_idx, S(stream)), "select");
    return PROXYATTN_OK;
}

int proxyattn_estimate(const proxyattn_cfg* cfg, const void* Q, const void* K, void* ws,
                       size_t ws_bytes, int32_t* kstar, float* budget, int32_t* block_cnt,
                       int32_t* block_idx, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!groups_complete(D))
        return fail(PROXYATTN_E_CONFIG,
                    "shard [%d, %d) splits a proxy group of %d query heads: use proxyattn_pool + "
                    "all-reduce + proxyattn_proxy_scores",
                    D.qb, D.qe, D.gq);
    const pa::Workspace W = pa::workspace_layout(D);
    if (!ws || ws_bytes < W.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", W.total);
    const bool scores_only = (D.flags & PROXYATTN_FLAG_SCORES_ONLY) != 0;
    if (!Q || !K || !kstar || !budget || (!scores_only && (!block_cnt || !block_idx)))
        return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    cudaStream_t st = S(stream);
    if ((rc = check_finite(D, st, {{Q, true}, {K, false}}))) return rc;
    void* Pq = at<char>(ws, W.pq);
    void* Pk = at<char>(ws, W.pk);
    float* L = at<float>(ws, W.L);
    // Row-range estimate (rows [rb, re), zig-zag row sharding): the lists of those rows need
    // the proxies of their sampled rows and of every key before them, the lse / max-pool of
    // the 128-row proxy tiles covering them, and Alg. 1 (per head, replicated unless
    // KSTAR_GIVEN).  The tcgen05 path restricts every stage; the fp32 SIMT path pools all.
    int tr0 = 0, tr1 = -1;
    long long q_i0 = 0, i_end = -1;
    if ((D.rb != 0 || D.re != D.M) && pa::score_tc_supported(D)) {
        i_end = std::min<long long>(D.Ns, static_cast<long long>(D.re) * D.bs);
        tr0 = static_cast<int>((static_cast<long long>(D.rb) * D.bs) / 128);
        tr1 = static_cast<int>((i_end + 127) / 128);
        q_i0 = static_cast<long long>(tr0) * 128;
    }
    // Alg. 1 (A4) depends on Q and K only: fork it onto the auxiliary stream so it overlaps
    // A1-A3 (their kernels are MUFU- / latency-bound with tails; the pool is HBM-bound),
    // join before A5-A6.  Separate scratch regions (W.scratch vs W.scratch_b).
    const bool alg1 = !(D.flags & PROXYATTN_FLAG_KSTAR_GIVEN);
    cudaStream_t aux = nullptr;
    if (alg1 && pa::score_tc_supported(D) && D.static_kstar == 0) {
        if ((rc = helper_stream(st, 0, &aux))) return rc;
    }
    AuxEvents ev{};
    if (aux) {
        if ((rc = estimate_events(&ev))) return rc;
        PA_CUDA(cudaEventRecord(ev.fork, st), "record");
        PA_CUDA(cudaStreamWaitEvent(aux, ev.fork, 0), "wait");
        Nvtx r("A4 Alg. 1 budgets");
        rc = run_budgets(D, Q, K, ws, W, kstar, budget, aux);
        if (rc) return rc;
        PA_CUDA(cudaEventRecord(ev.join, aux), "record");
    }
    {
        Nvtx r("A1 pool + stride");
        PA_CUDA(pa::launch_pool(D, Q, K, nullptr, nullptr, Pq, Pk, st, q_i0, i_end), "pool");
    }
    {
        Nvtx r("A2-A3 proxy scores");
        rc = run_proxy_from_pooled(D, Pq, Pk, ws, W, L, st, tr0, tr1);
        if (rc) return rc;
    }
    if (aux) {
        PA_CUDA(cudaStreamWaitEvent(st, ev.join, 0), "wait");
    } else if (alg1) {
        Nvtx r("A4 Alg. 1 budgets");
        rc = run_budgets(D, Q, K, ws, W, kstar, budget, st);
        if (rc) return rc;
    }
    if (scores_only) return PROXYATTN_OK;   // L stays in the workspace (proxyattn_select_ws)
    Nvtx r("A5-A6 select");
    PA_CUDA(pa::launch_select(D, L, kstar, block_cnt, block_idx, st), "select");
    return PROXYATTN_OK;
}

int proxyattn_select_ws(const proxyattn_cfg* cfg, const void* ws, size_t ws_bytes, const int32_t* kstar,
                        int32_t* block_cnt, int32_t* block_idx, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    const pa::Workspace W = pa::workspace_layout(D);
    if (!ws || ws_bytes < W.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", W.total);
    if (!kstar || !block_cnt || !block_idx) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    Nvtx r("A5-A6 select");
    const float* L = reinterpret_cast<const float*>(static_cast<const char*>(ws) + W.L);
    PA_CUDA(pa::launch_select(D, L, kstar, block_cnt, block_idx, S(stream)), "select");
    return PROXYATTN_OK;
}

static int attention(const proxyattn_cfg* cfg, const void* Q, const void* K, const void* V,
                     const int32_t* block_cnt, const int32_t* block_idx, void* O, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!Q || !K || !V || !O) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    cudaStream_t st = S(stream);
    if (block_cnt && (D.flags & PROXYATTN_FLAG_CHECK)) {
        int* bad = nullptr;
        PA_CUDA(cudaMallocAsync(&bad, sizeof(int), st), "check alloc");
        PA_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), st), "check memset");
        PA_CUDA(pa::launch_check_lists(D, block_cnt, block_idx, bad, st), "check_lists");
        int hbad = 0;
        PA_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st), "check copy");
        PA_CUDA(cudaFreeAsync(bad, st), "check free");
        PA_CUDA(cudaStreamSynchronize(st), "check sync");
        if (hbad) return fail(PROXYATTN_E_SHAPE, "%d block rows violate the list contract (S:319)", hbad);
    }
    if ((rc = check_finite(D, st, {{Q, true}, {K, false}, {V, false}}))) return rc;
    Nvtx r(block_cnt ? "A7 block-sparse attention" : "A8 dense attention");
    if (D.fp32)
        PA_CUDA(pa::launch_attn_simt(D, Q, K, V, block_cnt, block_idx, O, st), "attn_simt");
#if PA_ATTN_V9
    else if ((block_cnt || PA_ATTN_V9_DENSE) && use_v9(D.d, D.b))   // the row-pair kernel
        PA_CUDA(pa::launch_attn_tc9(D, Q, K, V, block_cnt, block_idx, O, st), "attn_tc9");
#endif
    else   // block-sparse (A7) or, with no lists, every causal block (A8): the same kernel
        PA_CUDA(pa::launch_attn_tc8(D, Q, K, V, block_cnt, block_idx, O, st), "attn_tc8");
    return PROXYATTN_OK;
}

int proxyattn_prefill(const proxyattn_cfg* cfg, const void* Q, const void* K, const void* V,
                      const int32_t* block_cnt, const int32_t* block_idx, void* O, void* stream) {
    if (!block_cnt || !block_idx) return fail(PROXYATTN_E_SHAPE, "NULL block lists");
    return attention(cfg, Q, K, V, block_cnt, block_idx, O, stream);
}

int proxyattn_dense_prefill(const proxyattn_cfg* cfg, const void* Q, const void* K, const void* V,
                            void* O, void* stream) {
    return attention(cfg, Q, K, V, nullptr, nullptr, O, stream);
}

// Bytes spanned by Q (= O) and by K (= V) in the configured layout.
static size_t q_bytes(const pa::Dims& D) {
    const size_t el = D.fp32 ? 4 : 2;
    return (D.tok ? (size_t)D.N * D.q_ts : (size_t)D.Hl * D.N * D.d) * el;
}
static size_t kv_bytes(const pa::Dims& D) {
    const size_t el = D.fp32 ? 4 : 2;
    return (D.tok ? (size_t)D.N * D.kv_ts : (size_t)D.Hkvl * D.N * D.d) * el;
}

// Device workspace of the host path: Q, K, V, O, per-head outputs, then the estimate scratch.
struct HostLayout {
    size_t q, k, v, o, kstar, budget, cnt, idx, ws, total;
};
static HostLayout host_layout(const pa::Dims& D) {
    HostLayout h{};
    size_t off = 0;
    h.q = off;      off = pa::align256(off + q_bytes(D));
    h.k = off;      off = pa::align256(off + kv_bytes(D));
    h.v = off;      off = pa::align256(off + kv_bytes(D));
    h.o = off;      off = pa::align256(off + q_bytes(D));
    h.kstar = off;  off = pa::align256(off + (size_t)D.Hl * 4);
    h.budget = off; off = pa::align256(off + (size_t)D.Hl * 4);
    h.cnt = off;    off = pa::align256(off + (size_t)D.Hl * D.M * 4);
    h.idx = off;    off = pa::align256(off + (size_t)D.Hl * D.M * D.M * 4);
    h.ws = off;     off = pa::align256(off + pa::workspace_layout(D).total);
    h.total = off;
    return h;
}

int proxyattn_forward_host_workspace_bytes(const proxyattn_cfg* cfg, size_t* out) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!out) return fail(PROXYATTN_E_CONFIG, "out is NULL");
    *out = host_layout(D).total;
    return PROXYATTN_OK;
}

int proxyattn_forward_host(const proxyattn_cfg* cfg, const void* Qh, const void* Kh, const void* Vh,
                           void* Oh, int32_t* kstar_h, void* dws, size_t dws_bytes, void* stream) {
    pa::Dims D;
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (!groups_complete(D))
        return fail(PROXYATTN_E_CONFIG, "forward_host needs every proxy group of the shard to be local");
    if (D.rb != 0 || D.re != D.M) return fail(PROXYATTN_E_CONFIG, "forward_host takes no row range");
    const HostLayout H = host_layout(D);
    if (!dws || dws_bytes < H.total) return fail(PROXYATTN_E_WORKSPACE, "device workspace needs %zu bytes", H.total);
    if (!Qh || !Kh || !Vh || !Oh) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    if (D.flags & PROXYATTN_FLAG_CHECK_FINITE)
        return fail(PROXYATTN_E_CONFIG, "forward_host: validate the inputs with a device call (CHECK_FINITE)");
    cudaStream_t st = S(stream);
    const size_t el = D.fp32 ? 4 : 2;
    const size_t kb = kv_bytes(D);
    // Pipeline over query-block-row chunks, LAST rows first.  The block lists of rows [r0, r1)
    // need only their own queries, the keys before them and K* (Alg. 1: the last block's
    // queries), so: K up, then the last row chunk of Q (Alg. 1 and that chunk's estimate can
    // start), then V, then the remaining Q chunks in reverse order; each chunk's row-range
    // estimate (K* given) and attention run as soon as it has landed, and its O goes down on
    // a third stream.  The heaviest rows (the longest causal lists) thus compute while the rest
    // of Q is still crossing PCIe.  Chunk edges sit on 128-row proxy tiles (and on the block-row
    // pairs of both attention kernels), so every chunk's lists and outputs equal the one-shot
    // call's bit for bit.
    const int align = std::max(2, 128 / D.bs);
    const int units = (D.M + align - 1) / align;
    // 16 row chunks (128K: 1 / 4 / 8 / 16 / 24 chunks -> 63.5 / 41.2 / 37.3 / 35.8 / 35.8 ms)
    const int n_ch = std::max(1, std::min(16, units));
    std::vector<std::pair<int, int>> ch;                  // [r0, r1) block rows, last rows first
    for (int k = 0; k < n_ch; ++k) {
        const int c = n_ch - 1 - k;
        const int r0 = std::min(D.M, align * static_cast<int>((static_cast<long long>(units) * c) / n_ch));
        const int r1 = std::min(D.M, align * static_cast<int>((static_cast<long long>(units) * (c + 1)) / n_ch));
        if (r1 > r0) ch.emplace_back(r0, r1);
    }
    cudaStream_t up = nullptr, down = nullptr;
    if ((rc = helper_stream(st, 1, &up)) || (rc = helper_stream(st, 2, &down))) return rc;
    const int nc = static_cast<int>(ch.size());
    // Every exit path goes through the guard: on an error it drains the helper streams and the
    // caller's stream (no async copy into the caller's host buffers is left in flight), and it
    // always destroys the per-call events.
    struct Guard {
        std::vector<cudaEvent_t> ev;
        cudaStream_t st, up, down;
        bool ok;
        ~Guard() {
            if (!ok) {
                cudaStreamSynchronize(up);
                cudaStreamSynchronize(down);
                cudaStreamSynchronize(st);
            }
            for (auto& e : ev)
                if (e) cudaEventDestroy(e);
        }
    } guard{std::vector<cudaEvent_t>(2 * nc + 3, nullptr), st, up, down, false};
    std::vector<cudaEvent_t>& ev = guard.ev;
    for (auto& e : ev) PA_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event create");
    cudaEvent_t ev_k = ev[0], ev_v = ev[1], ev_done = ev[2];
    // token range [t0, t1) of Q / O between host and device, in the configured layout
    auto copy_rows = [&](void* dst, const void* src, int r0, int r1, cudaMemcpyKind kind, cudaStream_t s) -> int {
        const long long t0 = static_cast<long long>(r0) * D.b, t1 = std::min<long long>(static_cast<long long>(r1) * D.b, D.N);
        if (t1 <= t0) return PROXYATTN_OK;
        if (D.tok) {   // [N][token stride]: one contiguous range
            const size_t off = static_cast<size_t>(t0) * D.q_ts * el, n = static_cast<size_t>(t1 - t0) * D.q_ts * el;
            PA_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, static_cast<const char*>(src) + off, n, kind, s),
                    "copy rows");
        } else {       // [Hl][N][d]: one strided block per head
            const size_t pitch = static_cast<size_t>(D.N) * D.d * el, off = static_cast<size_t>(t0) * D.d * el;
            PA_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + off, pitch, static_cast<const char*>(src) + off, pitch,
                                      static_cast<size_t>(t1 - t0) * D.d * el, D.Hl, kind, s), "copy rows");
        }
        return PROXYATTN_OK;
    };
    // uploads: K, Q chunk 0 (the last rows), V, the other Q chunks
    PA_CUDA(cudaEventRecord(ev[0], st), "record");                 // after the caller's prior work
    PA_CUDA(cudaStreamWaitEvent(up, ev[0], 0), "wait");
    PA_CUDA(cudaMemcpyAsync(at<char>(dws, H.k), Kh, kb, cudaMemcpyHostToDevice, up), "H2D K");
    PA_CUDA(cudaEventRecord(ev_k, up), "record");
    for (int c = 0; c < nc; ++c) {
        if ((rc = copy_rows(at<char>(dws, H.q), Qh, ch[c].first, ch[c].second, cudaMemcpyHostToDevice, up))) return rc;
        PA_CUDA(cudaEventRecord(ev[3 + c], up), "record");
        if (c == 0) {
            PA_CUDA(cudaMemcpyAsync(at<char>(dws, H.v), Vh, kb, cudaMemcpyHostToDevice, up), "H2D V");
            PA_CUDA(cudaEventRecord(ev_v, up), "record");
        }
    }
    // compute: Alg. 1 once, then per chunk estimate (K* given) + attention; O chunks down
    proxyattn_cfg cc = *cfg;
    for (int c = 0; c < nc; ++c) {
        PA_CUDA(cudaStreamWaitEvent(st, c == 0 ? ev_k : ev[3 + c], 0), "wait");
        if (c == 0) {
            PA_CUDA(cudaStreamWaitEvent(st, ev[3], 0), "wait");   // the last rows' Q
            rc = proxyattn_budgets(cfg, at<char>(dws, H.q), at<char>(dws, H.k), at<char>(dws, H.ws), dws_bytes - H.ws,
                                   at<int32_t>(dws, H.kstar), at<float>(dws, H.budget), stream);
            if (rc) return rc;
        }
        cc.row_begin = ch[c].first;
        cc.row_end = ch[c].second;
        cc.flags = cfg->flags | PROXYATTN_FLAG_KSTAR_GIVEN;
        rc = proxyattn_estimate(&cc, at<char>(dws, H.q), at<char>(dws, H.k), at<char>(dws, H.ws), dws_bytes - H.ws,
                                at<int32_t>(dws, H.kstar), at<float>(dws, H.budget), at<int32_t>(dws, H.cnt),
                                at<int32_t>(dws, H.idx), stream);
        if (rc) return rc;
        if (c == 0) PA_CUDA(cudaStreamWaitEvent(st, ev_v, 0), "wait");
        cc.flags = cfg->flags;
        rc = proxyattn_prefill(&cc, at<char>(dws, H.q), at<char>(dws, H.k), at<char>(dws, H.v),
                               at<int32_t>(dws, H.cnt), at<int32_t>(dws, H.idx), at<char>(dws, H.o), stream);
        if (rc) return rc;
        PA_CUDA(cudaEventRecord(ev[3 + nc + c], st), "record");
        PA_CUDA(cudaStreamWaitEvent(down, ev[3 + nc + c], 0), "wait");
        if ((rc = copy_rows(Oh, at<char>(dws, H.o), ch[c].first, ch[c].second, cudaMemcpyDeviceToHost, down))) return rc;
    }
    PA_CUDA(cudaEventRecord(ev_done, down), "record");
    PA_CUDA(cudaStreamWaitEvent(st, ev_done, 0), "wait");
    if (kstar_h)
        PA_CUDA(cudaMemcpyAsync(kstar_h, at<char>(dws, H.kstar), (size_t)D.Hl * 4, cudaMemcpyDeviceToHost, st),
                "D2H kstar");
    PA_CUDA(cudaStreamSynchronize(st), "forward_host sync");
    guard.ok = true;
    return PROXYATTN_OK;
}

// ------------------------------------------------------------------ varlen --
// One ProxyAttn layer per packed sequence.  The estimate runs per sequence (the cfg with
// seq_len = its length, pointers advanced by cu_seqlens[i] tokens, scratch reused in stream
// order).  bf16 with b = 128: every sequence's block lists are kept (packed, each with its own
// M) and ONE persistent attention launch covers all sequences (work items of the longest
// sequences first); otherwise one prefill per sequence.
constexpr int kMaxLanes = 8;   // packed varlen: concurrent per-sequence estimates
struct VarlenLayout {
    size_t cnt, idx, descs, total;
    int lanes;                                   // estimate lanes (streams), each with its own
    size_t lane_kstar[kMaxLanes], lane_budget[kMaxLanes], lane_ws[kMaxLanes];   // staging / scratch
    bool packed;
};
static bool varlen_packed(const pa::Dims& D) {
    return !D.fp32 && D.b == 128;
}
static int varlen_layout(const proxyattn_cfg* cfg, int32_t n, const int64_t* cu, VarlenLayout& L,
                         int64_t& max_len) {
    if (!cfg || !(cfg->flags & PROXYATTN_FLAG_TOKEN_MAJOR))
        return fail(PROXYATTN_E_CONFIG, "varlen needs PROXYATTN_FLAG_TOKEN_MAJOR (packed [tokens][heads][d])");
    if (n < 0 || !cu || cu[0] != 0) return fail(PROXYATTN_E_CONFIG, "cu_seqlens must start at 0");
    if (cfg->row_begin != 0 || cfg->row_end != 0) return fail(PROXYATTN_E_CONFIG, "varlen takes no row range");
    max_len = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (cu[i + 1] < cu[i]) return fail(PROXYATTN_E_CONFIG, "cu_seqlens must be non-decreasing");
        max_len = cu[i + 1] - cu[i] > max_len ? cu[i + 1] - cu[i] : max_len;
    }
    proxyattn_cfg c = *cfg;
    c.seq_len = max_len > 0 ? max_len : 1;
    pa::Dims D;
    int rc = derive(&c, D);
    if (rc) return rc;
    L.packed = varlen_packed(D);
    size_t n_cnt = (size_t)D.Hl * D.M, n_idx = (size_t)D.Hl * D.M * D.M;
    if (L.packed) {
        n_cnt = n_idx = 0;
        for (int32_t i = 0; i < n; ++i) {
            const size_t Mi = (size_t)((cu[i + 1] - cu[i] + D.b - 1) / D.b);
            n_cnt += (size_t)D.Hl * Mi;
            n_idx += (size_t)D.Hl * Mi * Mi;
        }
    }
    size_t off = 0;
    L.cnt = off;    off = pa::align256(off + n_cnt * 4);
    L.idx = off;    off = pa::align256(off + n_idx * 4);
    L.descs = off;  off = pa::align256(off + (L.packed ? (size_t)n * sizeof(pa::SeqDesc) : 0));
    // packed: up to kMaxLanes sequences' estimates in flight on their own streams (short
    // sequences' estimates are a few small, latency-bound launches each: concurrency fills the
    // GPU), as many lanes as non-empty sequences, capped so the lanes' scratch stays <= 256 MiB
    // (long sequences' estimates fill the GPU on their own: two lanes, as before)
    int nonempty = 0;
    for (int32_t i = 0; i < n; ++i) nonempty += cu[i + 1] > cu[i];
    const size_t scratch = pa::workspace_layout(D).total;
    L.lanes = 1;
    if (L.packed) {
        const size_t cap = std::max<size_t>(2, (size_t(256) << 20) / std::max<size_t>(scratch, 1));
        L.lanes = static_cast<int>(std::min<size_t>({static_cast<size_t>(kMaxLanes), cap,
                                                     static_cast<size_t>(std::max(nonempty, 1))}));
    }
    for (int k = 0; k < L.lanes; ++k) {
        L.lane_kstar[k] = off;  off = pa::align256(off + (size_t)D.Hl * 4);
        L.lane_budget[k] = off; off = pa::align256(off + (size_t)D.Hl * 4);
        L.lane_ws[k] = off;     off = pa::align256(off + scratch);
    }
    L.total = off;
    return PROXYATTN_OK;
}

int proxyattn_varlen_workspace_bytes(const proxyattn_cfg* cfg, int32_t n_seqs, const int64_t* cu,
                                     size_t* out) {
    VarlenLayout L;
    int64_t mx = 0;
    int rc = varlen_layout(cfg, n_seqs, cu, L, mx);
    if (rc) return rc;
    if (!out) return fail(PROXYATTN_E_CONFIG, "out is NULL");
    *out = L.total;
    return PROXYATTN_OK;
}

int proxyattn_forward_varlen(const proxyattn_cfg* cfg, int32_t n_seqs, const int64_t* cu,
                             const void* Q, const void* K, const void* V, void* O, void* ws,
                             size_t ws_bytes, int32_t* kstar, void* stream) {
    VarlenLayout L;
    int64_t mx = 0;
    int rc = varlen_layout(cfg, n_seqs, cu, L, mx);
    if (rc) return rc;
    if (!ws || ws_bytes < L.total) return fail(PROXYATTN_E_WORKSPACE, "varlen workspace needs %zu bytes", L.total);
    if (!Q || !K || !V || !O) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    proxyattn_cfg c = *cfg;
    c.seq_len = 1;
    pa::Dims D0;
    if ((rc = derive(&c, D0))) return rc;
    const size_t el = D0.fp32 ? 4 : 2;
    c.q_token_stride = D0.q_ts;      // pin the strides: the defaults depend on nothing per sequence,
    c.kv_token_stride = D0.kv_ts;    // but make it explicit
    cudaStream_t st = S(stream);
    std::vector<pa::SeqDesc> descs;
    std::vector<size_t> cnt_off(n_seqs, 0), idx_off(n_seqs, 0);
    if (L.packed) {
        // list offsets in sequence order; work items longest sequence first (heavy rows early)
        size_t oc = 0, oi = 0;
        for (int32_t i = 0; i < n_seqs; ++i) {
            const size_t Mi = (size_t)((cu[i + 1] - cu[i] + D0.b - 1) / D0.b);
            cnt_off[i] = oc;
            idx_off[i] = oi;
            oc += (size_t)D0.Hl * Mi;
            oi += (size_t)D0.Hl * Mi * Mi;
        }
        std::vector<int32_t> order;
        for (int32_t i = 0; i < n_seqs; ++i)
            if (cu[i + 1] > cu[i]) order.push_back(i);
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t x, int32_t y) { return cu[x + 1] - cu[x] > cu[y + 1] - cu[y]; });
        long long item0 = 0;
        for (int32_t i : order) {
            pa::SeqDesc sd{};
            sd.tok0 = cu[i];
            sd.cnt_off = (long long)cnt_off[i];
            sd.idx_off = (long long)idx_off[i];
            sd.N = static_cast<int>(cu[i + 1] - cu[i]);
            sd.M = static_cast<int>((sd.N + D0.b - 1) / D0.b);
            sd.item0 = static_cast<int>(item0);
            item0 += use_v9(D0.d, D0.b) ? (long long)pa::attn_tc9_units(D0.Hl, sd.M)
                                                 : (long long)D0.Hl * sd.M;
            descs.push_back(sd);
        }
        if (item0 > INT32_MAX || cu[n_seqs] > INT32_MAX)
            return fail(PROXYATTN_E_UNSUPPORTED, "varlen batch too large for one launch");
        if (!descs.empty())   // through kernel parameters: no pageable copy, the call stays async
            PA_CUDA(pa::write_seq_descs(at<pa::SeqDesc>(ws, L.descs), descs.data(),
                                        static_cast<int>(descs.size()), st), "varlen descriptors");
    }
    // packed: consecutive sequences' estimates rotate over L.lanes streams (`stream` and helper
    // streams, each lane with its own scratch) so the short, latency-bound estimates overlap
    // Every exit joins the forked lanes back into `stream` (an error path included: no helper
    // stream is left running work the caller cannot order against) and destroys the events.
    struct Lanes {
        cudaStream_t st[kMaxLanes] = {};
        cudaEvent_t fork = nullptr, join[kMaxLanes] = {};
        int n = 1;
        ~Lanes() {
            for (int k = 1; k < n; ++k) {
                if (st[k] && join[k] && cudaEventRecord(join[k], st[k]) == cudaSuccess)
                    cudaStreamWaitEvent(st[0], join[k], 0);
                if (join[k]) cudaEventDestroy(join[k]);   // released once the recorded work completes
            }
            if (fork) cudaEventDestroy(fork);
        }
    } lanes_g;
    cudaStream_t* lane_st = lanes_g.st;
    lane_st[0] = st;
    const int lanes = (L.packed && !descs.empty()) ? L.lanes : 1;
    if (lanes > 1) {
        PA_CUDA(cudaEventCreateWithFlags(&lanes_g.fork, cudaEventDisableTiming), "event create");
        PA_CUDA(cudaEventRecord(lanes_g.fork, st), "record");
        for (int k = 1; k < lanes; ++k) {
            if ((rc = helper_stream(st, 2 + k, &lane_st[k]))) return rc;   // kinds 3 ..
            PA_CUDA(cudaEventCreateWithFlags(&lanes_g.join[k], cudaEventDisableTiming), "event create");
            lanes_g.n = k + 1;
            PA_CUDA(cudaStreamWaitEvent(lane_st[k], lanes_g.fork, 0), "wait");
        }
    }
    int n_done = 0;
    for (int32_t i = 0; i < n_seqs; ++i) {
        const int64_t n = cu[i + 1] - cu[i];
        if (n == 0) continue;
        c.seq_len = n;
        const size_t qo = (size_t)cu[i] * D0.q_ts * el, ko = (size_t)cu[i] * D0.kv_ts * el;
        const int lane = n_done++ % lanes;
        cudaStream_t si = lane_st[lane];
        int32_t* ks = at<int32_t>(ws, L.lane_kstar[lane]);
        float* bu = at<float>(ws, L.lane_budget[lane]);
        const size_t wo = L.lane_ws[lane];
        int32_t* cnt = at<int32_t>(ws, L.cnt) + cnt_off[i];
        int32_t* idx = at<int32_t>(ws, L.idx) + idx_off[i];
        rc = proxyattn_estimate(&c, static_cast<const char*>(Q) + qo, static_cast<const char*>(K) + ko,
                                at<char>(ws, wo), ws_bytes - wo, ks, bu, cnt, idx, si);
        if (rc) return rc;
        if (!L.packed) {
            rc = proxyattn_prefill(&c, static_cast<const char*>(Q) + qo, static_cast<const char*>(K) + ko,
                                   static_cast<const char*>(V) + ko, cnt, idx, static_cast<char*>(O) + qo,
                                   stream);
            if (rc) return rc;
        }
        if (kstar)
            PA_CUDA(cudaMemcpyAsync(kstar + (size_t)i * D0.Hl, ks, (size_t)D0.Hl * 4,
                                    cudaMemcpyDeviceToDevice, si), "varlen kstar");
    }
    for (int k = 1; k < lanes; ++k) {   // join the lanes (the guard then only destroys events)
        PA_CUDA(cudaEventRecord(lanes_g.join[k], lane_st[k]), "record");
        PA_CUDA(cudaStreamWaitEvent(st, lanes_g.join[k], 0), "wait");
    }
    lanes_g.n = 1;
    for (int k = 1; k < lanes; ++k) {
        cudaEventDestroy(lanes_g.join[k]);
        lanes_g.join[k] = nullptr;
    }
    if (L.packed && !descs.empty()) {
        c.seq_len = cu[n_seqs];   // the packed tensors: TMA maps over every token
        pa::Dims D;               // (each sequence's M was checked by varlen_layout; the packed
        if ((rc = derive(&c, D, false))) return rc;   // total may exceed one sequence's limit)
        const bool v9 = use_v9(D.d, D.b);
        const int n_items = descs.back().item0 + (v9 ? static_cast<int>(pa::attn_tc9_units(D.Hl, descs.back().M))
                                                      : D.Hl * descs.back().M);
        if (v9)
            PA_CUDA(pa::launch_attn_tc9(D, Q, K, V, at<int32_t>(ws, L.cnt), at<int32_t>(ws, L.idx), O, st,
                                        at<pa::SeqDesc>(ws, L.descs), static_cast<int>(descs.size()), n_items),
                    "attn_tc9 varlen");
        else
            PA_CUDA(pa::launch_attn_tc8_varlen(D, Q, K, V, at<int32_t>(ws, L.cnt), at<int32_t>(ws, L.idx), O,
                                               at<pa::SeqDesc>(ws, L.descs), static_cast<int>(descs.size()),
                                               n_items, st),
                    "attn_tc8 varlen");
    }
    return PROXYATTN_OK;
}

// ------------------------------------------------------ seq-avgpool comparator --
// SPEC S:365-373 (seq_avgpool_scores): the per-head sequence-pooled
// estimator; the same Alg. 1 budgets and Eq. 3 selection then run on its score maps.
struct AvgLayout {
    size_t qb, kb, z, lse, ws, total;
};
static AvgLayout avg_layout(const pa::Dims& D) {
    AvgLayout A{};
    const size_t el = D.fp32 ? 4 : 2;
    size_t off = 0;
    A.qb = off;  off = pa::align256(off + (size_t)D.Hl * D.M * D.d * el);
    A.kb = off;  off = pa::align256(off + (size_t)D.Hkvl * D.M * D.d * el);
    A.z = off;   off = pa::align256(off + (size_t)D.Hl * D.M * D.M * 4);
    A.lse = off; off = pa::align256(off + (size_t)D.Hl * D.M * 4);
    A.ws = off;  off = pa::align256(off + pa::workspace_layout(D).total);   // Alg. 1 scratch
    A.total = off;
    return A;
}

static int avg_derive(const proxyattn_cfg* cfg, pa::Dims& D) {
    int rc = derive(cfg, D);
    if (rc) return rc;
    if (D.rb != 0 || D.re != D.M) return fail(PROXYATTN_E_CONFIG, "the avgpool comparator takes no row range");
    if (D.d % 32) return fail(PROXYATTN_E_UNSUPPORTED, "the avgpool comparator needs head_dim %% 32 == 0");
    return PROXYATTN_OK;
}

int proxyattn_avgpool_workspace_bytes(const proxyattn_cfg* cfg, size_t* out) {
    pa::Dims D;
    int rc = avg_derive(cfg, D);
    if (rc) return rc;
    if (!out) return fail(PROXYATTN_E_CONFIG, "out is NULL");
    *out = avg_layout(D).total;
    return PROXYATTN_OK;
}

int proxyattn_avgpool_scores(const proxyattn_cfg* cfg, const void* Q, const void* K, void* ws, size_t ws_bytes,
                             float* S_out, void* stream) {
    pa::Dims D;
    int rc = avg_derive(cfg, D);
    if (rc) return rc;
    const AvgLayout A = avg_layout(D);
    if (!ws || ws_bytes < A.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", A.total);
    if (!Q || !K || !S_out) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    cudaStream_t st = S(stream);
    if ((rc = check_finite(D, st, {{Q, true}, {K, false}}))) return rc;
    PA_CUDA(pa::launch_block_pool(D, Q, K, at<char>(ws, A.qb), at<char>(ws, A.kb), st), "block_pool");
    PA_CUDA(pa::launch_avgpool_scores(D, at<char>(ws, A.qb), at<char>(ws, A.kb), S_out, at<float>(ws, A.lse), true, st),
            "avgpool_scores");
    return PROXYATTN_OK;
}

int proxyattn_avgpool_estimate(const proxyattn_cfg* cfg, const void* Q, const void* K, void* ws, size_t ws_bytes,
                               int32_t* kstar, float* budget, int32_t* block_cnt, int32_t* block_idx, void* stream) {
    pa::Dims D;
    int rc = avg_derive(cfg, D);
    if (rc) return rc;
    const AvgLayout A = avg_layout(D);
    if (!ws || ws_bytes < A.total) return fail(PROXYATTN_E_WORKSPACE, "workspace needs %zu bytes", A.total);
    if (!Q || !K || !kstar || !budget || !block_cnt || !block_idx) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    cudaStream_t st = S(stream);
    if ((rc = check_finite(D, st, {{Q, true}, {K, false}}))) return rc;
    const pa::Workspace W = pa::workspace_layout(D);
    void* wsb = at<char>(ws, A.ws);
    Nvtx r("seq-avgpool comparator estimate");
    const bool alg1 = !(D.flags & PROXYATTN_FLAG_KSTAR_GIVEN);
    // Alg. 1 forked onto the helper stream, as in proxyattn_estimate (it reads only Q and K)
    cudaStream_t aux = nullptr;
    AuxEvents ev{};
    if (alg1) {
        if ((rc = helper_stream(st, 0, &aux)) || (rc = estimate_events(&ev))) return rc;
        PA_CUDA(cudaEventRecord(ev.fork, st), "record");
        PA_CUDA(cudaStreamWaitEvent(aux, ev.fork, 0), "wait");
        if ((rc = run_budgets(D, Q, K, wsb, W, kstar, budget, aux))) return rc;
        PA_CUDA(cudaEventRecord(ev.join, aux), "record");
    }
    PA_CUDA(pa::launch_block_pool(D, Q, K, at<char>(ws, A.qb), at<char>(ws, A.kb), st), "block_pool");
    // raw logits suffice for the selection: z - lse_m has the order of z within a row
    PA_CUDA(pa::launch_avgpool_scores(D, at<char>(ws, A.qb), at<char>(ws, A.kb), at<float>(ws, A.z), nullptr, false,
                                      st), "avgpool_scores");
    if (alg1) PA_CUDA(cudaStreamWaitEvent(st, ev.join, 0), "wait");
    PA_CUDA(pa::launch_select(D, at<float>(ws, A.z), kstar, block_cnt, block_idx, st, true), "select per head");
    return PROXYATTN_OK;
}

double proxyattn_cost_ratio(const proxyattn_cfg* cfg) {
    if (!cfg || cfg->n_q_heads <= 0 || cfg->stride <= 0) return 0.0;
    return static_cast<double>(cfg->n_groups) /
           (static_cast<double>(cfg->n_q_heads) * cfg->stride * cfg->stride);
}

const char* proxyattn_last_error(void) { return g_err.c_str(); }

const char* proxyattn_build_info(void) {
    return "libproxyattn sm_100a (tcgen05/TMEM/TMA attention and estimation)";
}

int proxyattn_debug_umma(const void* A, const void* B, float* C_ss, float* C_ts, void* stream) {
    if (!A || !B || !C_ss || !C_ts) return fail(PROXYATTN_E_SHAPE, "NULL pointer");
    PA_CUDA(pa::launch_debug_umma(A, B, C_ss, C_ts, S(stream)), "debug_umma");
    return PROXYATTN_OK;
}

}  // extern "C"
