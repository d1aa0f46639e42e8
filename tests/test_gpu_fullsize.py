"""Full-size parity on bench.py's workloads (128K Llama-3.1-8B shape = the headline, its
b = 64 variant, the d = 64 Llama-3.2-1B shape, Qwen2.5-7B at 64K with g = 4 and the 2048-token
minimum budget, the 70B shape, gamma = 0.95, the 16K / 32K (BASELINE config B) / 64K / 256K
sweep lines; the same launch configuration bench.py times), checked against the oracle at the
sampling of SURVEY §8(c).5: L rows first, last and 16 random per proxy group; Alg. 1 K* of
EVERY head (margin-gated); the block lists of those rows for every head (margin-gated, near
ties within 1e-4 of the cut); O on those rows for every head with the GPU mask injected.  At
32K (config B) L, the lists and O are checked on EVERY row of every head.  Plus properties at any size."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_24745_b200 as pa
import workloads
from test_gpu_parity import check_masks

pytestmark = pytest.mark.gpu

MARGIN = 1e-4


# bench.py's workloads at full size: (Hq, Hkv, d, N, b, g, min budget, preset[, gamma[, static K*]])
WORKLOADS = {
    "llama3.1-8b-attn-128k": (32, 8, 128, 131072, 128, 1, 0, "llama-128k"),
    "llama3.1-8b-attn-128k-b64": (32, 8, 128, 131072, 64, 1, 0, "llama-128k"),
    "llama3.2-1b-attn-128k": (32, 8, 64, 131072, 128, 1, 0, "llama1b-128k"),
    "qwen2.5-7b-attn-64k": (28, 4, 128, 65536, 128, 4, 2048, "qwen-64k"),
    "llama3.1-8b-attn-256k": (32, 8, 128, 262144, 128, 1, 0, "llama-256k"),   # bench --seq-len 262144
    "llama3.1-70b-attn-128k": (64, 8, 128, 131072, 128, 1, 0, "llama-128k"),
    "llama3.1-8b-attn-128k-g95": (32, 8, 128, 131072, 128, 1, 0, "llama-128k", 0.95),
    "llama3.1-8b-attn-16k": (32, 8, 128, 16384, 128, 1, 0, "llama-16k"),     # bench --seq-len sweep
    "llama3.1-8b-attn-32k": (32, 8, 128, 32768, 128, 1, 0, "llama-32k"),     # BASELINE config B
    "llama3.1-8b-attn-64k": (32, 8, 128, 65536, 128, 1, 0, "llama-64k"),
    "llama3.1-8b-attn-128k-fixed": (32, 8, 128, 131072, 128, 1, 0, "llama-128k", 0.9, 164),   # M-C-fixed
}


@pytest.fixture(scope="module", params=list(WORKLOADS))
def layer(request):
    dev = torch.device("cuda:0")
    Hq, Hkv, d, N, b, g, mb, preset, *rest = WORKLOADS[request.param]
    gamma = rest[0] if rest else 0.9
    sk = rest[1] if len(rest) > 1 else 0                      # static K* (the M-C-fixed line)
    cfg = pa.Config(Hq, Hkv, d, N, b, 4, g, gamma, mb, static_kstar=sk)
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=0, params=workloads.PRESETS[preset],
                                      device=dev)
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
    qsum, ksum = pa.pool(cfg, Q, K)
    L = pa.proxy_scores(cfg, qsum, ksum)
    torch.cuda.synchronize()
    oc = oracle.Cfg(Hq, Hkv, d, N, b, 4, g, gamma, mb, round_bf16=True, static_kstar=sk)
    host = dict(Q=Q.float().cpu().numpy(), K=K.float().cpu().numpy(), V=V.float().cpu().numpy())
    return dict(name=request.param, cfg=cfg, oc=oc, kstar=kstar.cpu().numpy(), budget=budget.cpu().numpy(),
                cnt=cnt.cpu().numpy(), idx=idx, O=O, L=L.cpu().numpy(), **host)


def sample_rows(M, seed=0):
    """the first and the last block row plus 16 random ones (seeded)."""
    rng = np.random.default_rng(seed)
    return sorted({0, M - 1} | {int(x) for x in rng.choice(np.arange(1, M - 1), size=min(16, M - 2), replace=False)})


def test_fullsize_properties(layer):
    cfg, cnt, ks = layer["cfg"], layer["cnt"], layer["kstar"]
    M = cfg.M
    assert np.all((ks >= 1) & (ks <= M))
    np.testing.assert_allclose(layer["budget"], ks / M, rtol=1e-6)
    # A5 closed form (Z12) on every (head, row)
    m = np.arange(M)[None, :]
    F = -(-cfg.min_budget_tokens // cfg.block_size)
    K = np.minimum(m + 1, np.maximum(np.maximum((ks[:, None].astype(np.int64) * (m + 1) + M - 1) // M, F), 1))
    assert np.array_equal(cnt, K)
    # lists: ascending, causal, diagonal last
    idx = layer["idx"]
    H = cfg.n_q_heads
    for h in (0, 7, 19, H - 1):
        for mm in (0, 1, M // 3, M - 1):
            lst = idx[h, mm, :cnt[h, mm]].cpu().numpy()
            assert lst[-1] == mm and np.all(np.diff(lst) > 0) and lst[0] >= 0
    for L in layer["L"]:                                     # every proxy group
        assert np.all(np.isneginf(L[np.triu_indices(M, 1)]))
        assert np.all(np.isfinite(L[np.tril_indices(M)]))
        assert np.all(L[np.tril_indices(M)] <= 1e-6)        # log-probabilities
    assert torch.isfinite(layer["O"]).all()


def test_fullsize_sampled_parity(layer):
    cfg, oc = layer["cfg"], layer["oc"]
    M, G, H, b = cfg.M, cfg.n_groups, cfg.n_q_heads, cfg.block_size
    complete = layer["name"] == "llama3.1-8b-attn-32k"          # config B: every row
    rows = list(range(M)) if complete else sample_rows(M)
    Pq, Pk, scale = oracle.pool(oc, layer["Q"], layer["K"])
    _, Lref = oracle.proxy_scores(oc, Pq, Pk, scale, rows=None if complete else rows)
    del Pq, Pk
    for c in range(G):                                       # stage 2, every group
        for m in rows:
            ref = Lref[c, m, :m + 1]
            got = layer["L"][c, m, :m + 1].astype(np.float64)
            assert np.max(np.abs(got - ref)) <= 1e-4, (c, m)
    # stage 3: Alg. 1 K* of EVERY head (margin-gated, |dK*| <= 1 below the margin)
    ks_ref, _, bmg, _ = oracle.budgets(oc, layer["Q"], layer["K"])
    ks = layer["kstar"]
    ok = bmg > MARGIN
    assert np.array_equal(ks[ok], ks_ref[ok]), (ks, ks_ref)
    assert np.all(np.abs(ks.astype(int) - ks_ref.astype(int)) <= 1)
    print(f"{layer['name']}: K* exact on {int(ok.sum())}/{H} heads with margin > 1e-4")
    # stage 4: lists of the sampled rows for EVERY head (oracle L, GPU budgets injected)
    Lfull = np.full((G, M, M), -np.inf)
    Lfull[:, rows] = Lref[:, rows]
    del Lref
    checked, near = check_masks(oc, Lfull, ks, layer["cnt"], layer["idx"], rows=rows)
    # a guard that the margin gate does not hide a systematic difference (near-tie rows are still
    # validated by the near-tie rule above); with a static K* every head cuts the SAME shared
    # order at the same rank, so one near-tie row counts once per head (2 of 18 rows at 128K)
    assert checked >= (0.85 if cfg.static_kstar else 0.9) * (checked + near)
    del Lfull
    # stage 5: O on the sampled rows for EVERY head, GPU mask injected
    orows = rows                                             # config B: every row
    items = [(h, m) for h in range(H) for m in orows]
    cnt_h = layer["cnt"]
    idx = layer["idx"]
    idx_h = np.zeros((H, M, M), np.int32)
    for h in range(H):
        sel = idx[h, orows].cpu().numpy()
        for k, m in enumerate(orows):
            idx_h[h, m, :cnt_h[h, m]] = sel[k, :cnt_h[h, m]]
    Oref = oracle.attention(oc, layer["Q"], layer["K"], layer["V"], cnt_h, idx_h,
                            items=np.array(items, np.int32).reshape(-1))
    O = layer["O"]
    worst = 0.0
    for h in range(H):
        got = O[h].float().cpu().numpy()
        for m in orows:
            t0, t1 = m * b, min((m + 1) * b, cfg.seq_len)
            err = np.abs(got[t0:t1] - Oref[h, t0:t1])
            assert err.max() <= 2e-2 and err.mean() <= 2e-3, (h, m, err.max(), err.mean())
            worst = max(worst, float(err.max()))
    print(f"{layer['name']}: O on {len(items)} (head, row) items, max |dO| {worst:.2e}")


def test_fullsize_dense_sampled(layer):
    cfg, oc = layer["cfg"], layer["oc"]
    dev = torch.device("cuda:0")
    M = cfg.M
    Q = torch.from_numpy(layer["Q"]).to(dev).bfloat16()
    K = torch.from_numpy(layer["K"]).to(dev).bfloat16()
    V = torch.from_numpy(layer["V"]).to(dev).bfloat16()
    Od = pa.dense_prefill(cfg, Q, K, V)
    items = [(3, M - 1), (20, M // 3)]
    Oref = oracle.dense(oc, layer["Q"], layer["K"], layer["V"],
                        items=np.array(items, np.int32).reshape(-1))
    b = cfg.block_size
    for h, m in items:
        got = Od[h, m * b:(m + 1) * b].float().cpu().numpy()
        err = np.abs(got - Oref[h, m * b:(m + 1) * b])
        assert err.max() <= 2e-2 and err.mean() <= 2e-3, (h, m, err.max(), err.mean())


def test_fullsize_attention_recall_sampled(layer):
    # the share of each sampled query's dense causal softmax mass that its selected blocks
    # hold (fp32 torch reference on the GPU for the sampled rows only) — the quantity gamma
    # targets (§3.2).  Recorded, and bounded from below as a regression guard.
    cfg = layer["cfg"]
    dev = torch.device("cuda:0")
    M, b, d, r = cfg.M, cfg.block_size, cfg.head_dim, cfg.r
    Q = torch.from_numpy(layer["Q"]).to(dev)
    K = torch.from_numpy(layer["K"]).to(dev)
    cnt, idx = layer["cnt"], layer["idx"]
    g = torch.Generator().manual_seed(5)
    recs = []
    for h in range(0, cfg.n_q_heads, 3):
        for t in torch.randint(0, cfg.seq_len, (16,), generator=g).tolist():
            m = t // b
            s = (K[h // r, :t + 1] @ Q[h, t]) / d ** 0.5
            p = torch.softmax(s.double(), 0)
            keep = torch.zeros(t + 1, dtype=torch.bool, device=dev)
            for n in idx[h, m, :cnt[h, m]].tolist():
                keep[n * b:min((n + 1) * b, t + 1)] = True
            recs.append(float(p[keep].sum()))
    mean = float(np.mean(recs))
    print(f"recall mean {mean:.4f} min {min(recs):.4f}")
    assert mean >= 0.7, mean
