"""Full-size parity on bench.py's workloads (128K Llama-3.1-8B shape = the headline, its
b = 64 variant, the d = 64 Llama-3.2-1B shape, Qwen2.5-7B at 64K with g = 4 and the 2048-token
minimum budget, the 70B shape, gamma = 0.95, the 256K sweep line; the same launch configuration bench.py times), checked against the oracle on SAMPLED
outputs the oracle can compute one by one: L rows, Alg. 1 budgets of sampled heads,
selected blocks on sampled rows (margin-gated), and O on sampled (head, row)
items with the GPU mask injected.  Plus properties that hold at any size."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

MARGIN = 1e-4


# bench.py's workloads at full size: (Hq, Hkv, d, N, b, g, min budget, preset[, gamma])
WORKLOADS = {
    "llama3.1-8b-attn-128k": (32, 8, 128, 131072, 128, 1, 0, "llama-128k"),
    "llama3.1-8b-attn-128k-b64": (32, 8, 128, 131072, 64, 1, 0, "llama-128k"),
    "llama3.2-1b-attn-128k": (32, 8, 64, 131072, 128, 1, 0, "llama1b-128k"),
    "qwen2.5-7b-attn-64k": (28, 4, 128, 65536, 128, 4, 2048, "qwen-64k"),
    "llama3.1-8b-attn-256k": (32, 8, 128, 262144, 128, 1, 0, "llama-256k"),   # bench --seq-len 262144
    "llama3.1-70b-attn-128k": (64, 8, 128, 131072, 128, 1, 0, "llama-128k"),
    "llama3.1-8b-attn-128k-g95": (32, 8, 128, 131072, 128, 1, 0, "llama-128k", 0.95),
}


@pytest.fixture(scope="module", params=list(WORKLOADS))
def layer(request):
    dev = torch.device("cuda:0")
    Hq, Hkv, d, N, b, g, mb, preset, *rest = WORKLOADS[request.param]
    gamma = rest[0] if rest else 0.9
    cfg = pa.Config(Hq, Hkv, d, N, b, 4, g, gamma, mb)
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=0, params=workloads.PRESETS[preset],
                                      device=dev)
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
    qsum, ksum = pa.pool(cfg, Q, K)
    L = pa.proxy_scores(cfg, qsum, ksum)
    torch.cuda.synchronize()
    oc = oracle.Cfg(Hq, Hkv, d, N, b, 4, g, gamma, mb, round_bf16=True)
    host = dict(Q=Q.float().cpu().numpy(), K=K.float().cpu().numpy(), V=V.float().cpu().numpy())
    return dict(cfg=cfg, oc=oc, kstar=kstar.cpu().numpy(), budget=budget.cpu().numpy(),
                cnt=cnt.cpu().numpy(), idx=idx, O=O, L=L.cpu().numpy(), **host)


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
    M = cfg.M
    rows = [0, 1, M // 4, M // 2, 3 * M // 4, M - 1]
    Pq, Pk, scale = oracle.pool(oc, layer["Q"], layer["K"])
    _, Lref = oracle.proxy_scores(oc, Pq, Pk, scale, rows=rows)
    G = cfg.n_groups
    for c in range(G):
        for m in rows:
            ref = Lref[c, m, :m + 1]
            got = layer["L"][c, m, :m + 1].astype(np.float64)
            assert np.max(np.abs(got - ref)) <= 1e-4, (c, m)
    # budgets of sampled heads (margin-gated)
    H, b = cfg.n_q_heads, cfg.block_size
    heads = [0, 5, 17, H - 2]
    ks_ref, _, bmg, _ = oracle.budgets(oc, layer["Q"], layer["K"], heads=heads)
    for h in heads:
        if bmg[h] > MARGIN:
            assert layer["kstar"][h] == ks_ref[h], (h, layer["kstar"][h], ks_ref[h])
        else:
            assert abs(int(layer["kstar"][h]) - int(ks_ref[h])) <= 1
    # selection on sampled rows from the oracle's L with the GPU budgets injected
    Lfull = np.full((G, M, M), -np.inf)
    Lfull[:, rows] = Lref[:, rows]
    ocnt, oidx, cmg = oracle.select(oc, Lfull, layer["kstar"], rows=rows)
    checked = 0
    idx = layer["idx"]
    for h in range(cfg.n_q_heads):
        for m in rows:
            assert layer["cnt"][h, m] == ocnt[h, m]
            if cmg[h, m] > MARGIN:
                c = ocnt[h, m]
                assert np.array_equal(idx[h, m, :c].cpu().numpy(), oidx[h, m, :c]), (h, m)
                checked += 1
    assert checked >= 0.9 * cfg.n_q_heads * len(rows)
    # O on sampled (head, row) items with the GPU mask injected
    items = [(0, M - 1), (17, M - 1), (5, M // 2), (H - 2, 1), (11, 0), (24, 3 * M // 4), (H - 1, M - 2)]
    cnt_h = layer["cnt"]
    idx_h = np.zeros((cfg.n_q_heads, M, M), np.int32)
    for h, m in items:
        idx_h[h, m, :cnt_h[h, m]] = idx[h, m, :cnt_h[h, m]].cpu().numpy()
    Oref = oracle.attention(oc, layer["Q"], layer["K"], layer["V"], cnt_h, idx_h,
                            items=np.array(items, np.int32).reshape(-1))
    O = layer["O"]
    for h, m in items:
        got = O[h, m * b:(m + 1) * b].float().cpu().numpy()
        err = np.abs(got - Oref[h, m * b:(m + 1) * b])
        assert err.max() <= 2e-2 and err.mean() <= 2e-3, (h, m, err.max(), err.mean())


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
