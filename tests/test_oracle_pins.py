"""Pins of the fp64 CPU oracle (oracle/) against what the paper and the mathematics fix.

Each test names the passage it pins (P:<line> PAPER.md, S:<line> SPEC.md) and checks the
oracle against a value the paper/SPEC prints, a closed form, an invariant, a special case
that reduces to a textbook routine, or brute force on tiny inputs — chosen so that a
dropped term, wrong sign/index or transposed operand in any oracle step fails one of them.
"""
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import workloads

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))

CFG_A = oracle.Cfg(n_q_heads=8, n_kv_heads=2, head_dim=64, seq_len=1024, block_size=64,
                   stride=4, n_groups=2, gamma=0.9)   # BASELINE.json configs[0]
GAMMAS = [0.5, 0.7, 0.9, 0.95, 1.0]                     # AC4 grid


def rand_qkv(cfg, seed, scale=1.0):
    Q, K, V = workloads.iid(cfg.n_q_heads, cfg.n_kv_heads, cfg.seq_len, cfg.head_dim, seed)
    return (Q * scale).numpy(), (K * scale).numpy(), V.numpy()


# ----------------------------------------------------------------------- brute force --
def bf_probs(q, k):
    """Dense causal softmax probabilities of one head, [N][N] (textbook definition)."""
    d = q.shape[1]
    z = (q.astype(np.float64) @ k.astype(np.float64).T) / math.sqrt(d)
    N = z.shape[0]
    z[np.triu_indices(N, 1)] = -np.inf
    z -= z.max(axis=1, keepdims=True)
    p = np.exp(z)
    return p / p.sum(axis=1, keepdims=True)


def bf_attention(q, k, v, allowed=None):
    """out[t] = sum_s softmax(q_t k_s / sqrt d) v_s over causal s (and allowed[t, s])."""
    d = q.shape[1]
    z = (q.astype(np.float64) @ k.astype(np.float64).T) / math.sqrt(d)
    N = z.shape[0]
    mask = np.tril(np.ones((N, N), bool))
    if allowed is not None:
        mask &= allowed
    z[~mask] = -np.inf
    z -= z.max(axis=1, keepdims=True)
    p = np.exp(z)
    p /= p.sum(axis=1, keepdims=True)
    return p @ v.astype(np.float64)


# ------------------------------------------------------------------------------- O1 --
def test_validate_rejects_invariant_violations():
    assert oracle.validate(CFG_A)
    for bad in [dict(n_q_heads=7), dict(n_groups=3), dict(stride=3), dict(seq_len=0),
                dict(gamma=0.0), dict(gamma=1.5), dict(min_budget_tokens=-1)]:
        assert not oracle.validate(CFG_A.replace(**bad)), bad
    assert oracle.validate(CFG_A.replace(seq_len=1000))        # ragged N: padded last block


# ------------------------------------------------------------------------------- O2 --
def test_groups_llama_qwen_identity():
    # S:121 Llama g=1: all heads in group 0; S:122 Qwen 28/4, g=4: 7 query heads per group
    llama = oracle.Cfg(32, 8, 128, 1024, 128, 4, 1, 0.9)
    assert {oracle.group_of_q(llama, h) for h in range(32)} == {0}
    qwen = oracle.Cfg(28, 4, 128, 1024, 128, 4, 4, 0.9)
    groups = [oracle.group_of_q(qwen, h) for h in range(28)]
    assert groups == [h // 7 for h in range(28)]
    ident = oracle.Cfg(4, 4, 64, 256, 64, 4, 4, 0.9)    # S:123 n_q = n_kv = g
    assert [oracle.group_of_q(ident, h) for h in range(4)] == [0, 1, 2, 3]


# ------------------------------------------------------------------------------- O3 --
def test_rne_bf16_matches_torch_and_ties_to_even():
    rng = np.random.default_rng(0)
    x = (rng.standard_normal(20000) * np.exp(rng.uniform(-30, 30, 20000))).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    got = np.array([oracle.rne_bf16(float(v)) for v in x])
    assert np.array_equal(got, ref)
    # exact ties: 1 + 2^-8 lies halfway between 1 and 1 + 2^-7 -> even mantissa (1.0)
    assert oracle.rne_bf16(1.0 + 2.0 ** -8) == 1.0
    assert oracle.rne_bf16(1.0 + 3 * 2.0 ** -8) == 1.0 + 2 * 2.0 ** -7
    assert oracle.rne_bf16(-(1.0 + 2.0 ** -8)) == -1.0


def test_pool_single_head_group_is_identity_and_stride_keeps_window_heads():
    # S:130 group of one head -> Q^g identical; S:139-141 stride keeps tokens 0, s, 2s, ...
    cfg = oracle.Cfg(2, 2, 8, 8, 4, 4, 2, 0.9)
    Q, K, _ = rand_qkv(cfg, 1)
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    assert Pq.shape == (2, 2, 8)
    for h in range(2):
        assert np.array_equal(Pq[h], Q[h, [0, 4]].astype(np.float64))
        assert np.array_equal(Pk[h], K[h, [0, 4]].astype(np.float64))
    assert scale == pytest.approx(1.0 / math.sqrt(8))
    cfg1 = cfg.replace(stride=1)
    Pq1, _, _ = oracle.pool(cfg1, Q, K)
    assert np.array_equal(Pq1, Q.astype(np.float64))      # stride=1 is the identity


def test_pool_antisymmetric_pair_gives_zero_and_mean_matches_scalar_loop():
    cfg = oracle.Cfg(2, 1, 4, 8, 4, 2, 1, 0.9)
    Q = np.random.default_rng(2).standard_normal((2, 8, 4)).astype(np.float32)
    Q[1] = -Q[0]                                            # S:131 Q2 = -Q1 -> 0
    K = np.random.default_rng(3).standard_normal((1, 8, 4)).astype(np.float32)
    Pq, _, scale = oracle.pool(cfg, Q, K)
    assert np.all(Pq == 0.0)
    # S:132 seeded 4-head group: elementwise mean by a scalar loop (GQA: 4 q / 2 kv heads)
    cfg2 = oracle.Cfg(4, 2, 3, 8, 4, 2, 1, 0.9)
    rng = np.random.default_rng(4)
    Q2 = rng.standard_normal((4, 8, 3)).astype(np.float32)
    K2 = rng.standard_normal((2, 8, 3)).astype(np.float32)
    Pq2, Pk2, sc2 = oracle.pool(cfg2, Q2, K2)
    for i in range(4):
        for e in range(3):
            s = 0.0
            for h in range(4):
                s += float(Q2[h, 2 * i, e])
            assert Pq2[0, i, e] / 4 == pytest.approx(s / 4, abs=1e-12)
            s = 0.0
            for h in range(2):
                s += float(K2[h, 2 * i, e])
            assert Pk2[0, i, e] / 2 == pytest.approx(s / 2, abs=1e-12)
    # Eq. 2 means + Eq. 1 1/sqrt(d_k) fold into 1/(|Gq| |Gk| sqrt d)   (Z2, Z5)
    assert sc2 == pytest.approx(1.0 / (4 * 2 * math.sqrt(3)))


def test_pool_bf16_rounding_of_sums():
    cfg = oracle.Cfg(4, 2, 8, 16, 8, 4, 1, 0.9, round_bf16=True)
    rng = np.random.default_rng(5)
    Q = torch.from_numpy(rng.standard_normal((4, 16, 8)).astype(np.float32)).bfloat16().float().numpy()
    K = torch.from_numpy(rng.standard_normal((2, 16, 8)).astype(np.float32)).bfloat16().float().numpy()
    Pq, Pk, _ = oracle.pool(cfg, Q, K)
    exact = Q[:, ::4].astype(np.float64).sum(0)
    ref = torch.from_numpy(exact).to(torch.bfloat16).double().numpy()   # exact sum -> RNE
    assert np.array_equal(Pq[0], ref)


# ---------------------------------------------------------------------------- O4-O6 --
def test_proxy_scores_degenerate_equals_block_max_of_dense_probs():
    # AC3: stride 1, singleton groups -> exp(L) == block-max of the dense probs
    cfg = oracle.Cfg(3, 3, 8, 64, 16, 1, 3, 0.9)
    Q, K, _ = rand_qkv(cfg, 7, scale=2.0)
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    lse, L = oracle.proxy_scores(cfg, Pq, Pk, scale)
    M, b = cfg.M, cfg.block_size
    for h in range(3):
        P = bf_probs(Q[h], K[h])
        for m in range(M):
            for n in range(M):
                if n > m:
                    assert L[h, m, n] == -np.inf
                else:
                    ref = P[m * b:(m + 1) * b, n * b:(n + 1) * b].max()
                    assert math.exp(L[h, m, n]) == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_proxy_softmax_rows_sum_to_one_over_sampled_keys():
    # S:165 subsample-then-softmax rows sum to 1 (over sampled causal keys only, Z4)
    cfg = CFG_A.replace(seq_len=256)
    Q, K, _ = rand_qkv(cfg, 8)
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    lse, _ = oracle.proxy_scores(cfg, Pq, Pk, scale)
    for c in range(cfg.n_groups):
        z = (Pq[c] @ Pk[c].T) * scale
        for i in range(0, cfg.Ns, 7):
            assert np.exp(z[i, :i + 1] - lse[c, i]).sum() == pytest.approx(1.0, abs=1e-12)


def test_proxy_needle_block_attains_row_max():
    # a key with a large dot product with all queries -> its block column is the
    # row maximum of every block row that can see it.
    cfg = oracle.Cfg(2, 2, 16, 512, 64, 4, 2, 0.9)
    pos = 100 * 4 // 4 * 1   # sampled position (multiple of the stride) inside block 1
    Q, K, _ = workloads.needle(2, 512, 16, pos=pos, boost=12.0, seed=3)
    Q, K = Q.numpy(), K.numpy()
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    _, L = oracle.proxy_scores(cfg, Pq, Pk, scale)
    nb = pos // cfg.block_size
    for c in range(2):
        for m in range(nb + 1, cfg.M):
            assert int(np.argmax(L[c, m, :m + 1])) == nb


def test_proxy_row_subset_matches_full():
    cfg = CFG_A.replace(seq_len=512)
    Q, K, _ = rand_qkv(cfg, 9)
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    _, L = oracle.proxy_scores(cfg, Pq, Pk, scale)
    rows = [0, 3, 7]
    _, Ls = oracle.proxy_scores(cfg, Pq, Pk, scale, rows=rows)
    assert np.array_equal(Ls[:, rows], L[:, rows])


# ------------------------------------------------------------------------------- O7 --
@pytest.mark.parametrize("case", GOLD["budget_from_mass"], ids=lambda c: c["cite"][:12])
def test_budget_from_mass_spec_examples(case):
    k, _ = oracle.budget_from_mass(case["mass"], case["gamma"])
    assert k == case["kstar"]
    assert k / len(case["mass"]) == pytest.approx(case["budget"])


def test_budget_uniform_attention_all_zero_q():
    # all-zero Q -> uniform attention over the causal keys; N/b = 4, gamma = 0.75 -> 3
    # (with the causal last block (Z7) the normalised masses are .283/.283/.283/.151 and the
    # prefix still first crosses 0.75 at k = 3).
    cfg = oracle.Cfg(2, 1, 8, 64, 16, 4, 1, 0.75)
    Q = np.zeros((2, 64, 8), np.float32)
    K = np.random.default_rng(0).standard_normal((1, 64, 8)).astype(np.float32)
    kstar, budget, _, mass = oracle.budgets(cfg, Q, K)
    assert list(kstar) == [3, 3] and budget[0] == 0.75
    b = 16
    exp0 = sum(b / (t + 1) for t in range(48, 64)) / b ** 2      # closed form, full blocks
    exp3 = sum((t - 47) / (t + 1) for t in range(48, 64)) / b ** 2
    assert mass[0, :3] == pytest.approx([exp0] * 3, rel=1e-12)
    assert mass[0, 3] == pytest.approx(exp3, rel=1e-12)


def test_budget_one_hot_and_gamma_one():
    # S:207 one-hot mass on one block -> 1/(N/b); S:216 gamma = 1 -> 1
    cfg = oracle.Cfg(1, 1, 8, 128, 16, 4, 1, 0.95)
    w = np.zeros(8, np.float32)
    w[0] = 1.0
    Q = np.tile(w, (1, 128, 1))
    K = np.zeros((1, 128, 8), np.float32)
    K[0, 16:32] = 60.0 * w            # block 1 dominates every row that sees it
    kstar, budget, _, _ = oracle.budgets(cfg, Q, K)
    assert kstar[0] == 1 and budget[0] == pytest.approx(1 / 8)
    kstar1, budget1, _, _ = oracle.budgets(cfg.replace(gamma=1.0), Q, K)
    assert kstar1[0] == 8 and budget1[0] == 1.0


def test_budget_identical_heads_and_sharper_head():
    # S:214 identical heads -> identical budgets; S:215 sharper (peaked) head -> smaller b_i
    cfg = oracle.Cfg(2, 1, 64, 1024, 64, 4, 1, 0.9)
    Q, K, _ = rand_qkv(cfg.replace(n_q_heads=1), 11)
    Qi = np.concatenate([Q, Q])
    kstar, _, _, _ = oracle.budgets(cfg, Qi, K)
    assert kstar[0] == kstar[1]
    # block-structured logits z(t, k) = beta * a_{block(k)}: flat (beta=0.3) vs peaked (beta=4)
    rng = np.random.default_rng(3)
    w = np.zeros(64, np.float32)
    w[0] = 1.0
    a = rng.standard_normal(cfg.M).astype(np.float32)
    Kb = (np.repeat(a, cfg.block_size)[:, None] * math.sqrt(64) * w)[None].astype(np.float32)
    Qs = np.stack([np.tile(0.3 * w, (1024, 1)), np.tile(4.0 * w, (1024, 1))]).astype(np.float32)
    ks, _, _, _ = oracle.budgets(cfg, Qs, Kb)
    assert ks[1] < ks[0]


def test_budget_shift_invariance():
    # S:221 adding a constant to a head's logits leaves b_i unchanged: adding one vector u
    # to every key shifts row t's logits by q_t.u / sqrt(d), a per-row constant.
    cfg = oracle.Cfg(2, 1, 32, 512, 64, 4, 1, 0.9)
    Q, K, _ = rand_qkv(cfg, 12)
    k0, _, _, m0 = oracle.budgets(cfg, Q, K)
    u = np.random.default_rng(1).standard_normal(32).astype(np.float32)
    k1, _, _, m1 = oracle.budgets(cfg, Q, K + u)
    assert np.array_equal(k0, k1)
    assert np.allclose(m0, m1, rtol=1e-5, atol=1e-12)   # K + u rounds in fp32


def test_budget_brute_force_tiny():
    # brute force: dense probabilities of the last block, block sums, stable sort, cumsum
    cfg = oracle.Cfg(4, 2, 16, 256, 32, 4, 1, 0.8)
    Q, K, _ = rand_qkv(cfg, 13, scale=1.5)
    kstar, _, _, mass = oracle.budgets(cfg, Q, K)
    b, M = cfg.block_size, cfg.M
    for h in range(4):
        P = bf_probs(Q[h], K[h // 2])[-b:]
        a = P.reshape(b, M, b).sum(axis=(0, 2)) / b ** 2
        assert mass[h] == pytest.approx(a, rel=1e-10, abs=1e-18)
        srt = np.sort(a)[::-1]
        cum = np.cumsum(srt / srt.sum())
        ref = int(np.argmax(cum >= cfg.gamma)) + 1
        assert kstar[h] == ref


def test_budget_monotone_in_gamma_ac4():
    # AC4: b_i nondecreasing over the gamma grid for every head on 20 seeds
    cfg = CFG_A.replace(seq_len=256)
    for seed in range(20):
        Q, K, _ = rand_qkv(cfg, 100 + seed)
        prev = None
        for g in GAMMAS:
            ks, _, _, _ = oracle.budgets(cfg.replace(gamma=g), Q, K)
            assert np.all(ks >= 1) and np.all(ks <= cfg.M)
            if prev is not None:
                assert np.all(ks >= prev), (seed, g)
            prev = ks
        assert np.all(prev == cfg.M)         # gamma = 1 -> full budget


# ------------------------------------------------------------------------------- O8 --
@pytest.mark.parametrize("case", GOLD["min_budget_floor_blocks"], ids=lambda c: c["cite"][:6])
def test_min_budget_floor(case):
    b = case["b"]
    cfg = oracle.Cfg(1, 1, 32, b * 64, b, 4 if b % 4 == 0 else 1, 1, 0.9,
                     min_budget_tokens=case["tokens"])
    F = case["blocks"]
    # with kstar = 1 the ratio term is 1 on every row, so the row count is min(m+1, max(F, 1))
    for m in range(64):
        assert oracle.row_count(cfg, 1, m) == min(m + 1, max(F, 1))


@pytest.mark.parametrize("case", GOLD["forced_kstar_sparsity"], ids=lambda c: str(c["M"]))
def test_row_count_forced_kstar_sparsity(case):
    M, F, ks = case["M"], case["F"], case["kstar"]
    cfg = oracle.Cfg(1, 1, 32, 128 * M, 128, 4, 1, 0.9, min_budget_tokens=F * 128)
    total = sum(oracle.row_count(cfg, ks, m) for m in range(M))
    assert 1 - total / (M * (M + 1) / 2) == pytest.approx(case["sparsity"], abs=5e-5)
    assert oracle.row_count(cfg, M, M - 1) == M                # kstar = M -> full last row
    assert all(oracle.row_count(cfg, M, m) == m + 1 for m in range(0, M, 37))


# ------------------------------------------------------------------------------- O9 --
def test_select_full_budget_gives_full_causal_mask():
    # S:261 b_i = 1 -> full causal block mask, sparsity 0
    cfg = CFG_A.replace(seq_len=512)
    Q, K, _ = rand_qkv(cfg, 14)
    est = oracle.estimate(cfg.replace(gamma=1.0), Q, K)
    assert np.all(est["kstar"] == cfg.M)
    for h in range(cfg.n_q_heads):
        for m in range(cfg.M):
            assert est["block_cnt"][h, m] == m + 1
            assert list(est["block_idx"][h, m, :m + 1]) == list(range(m + 1))
    assert oracle.sparsity(cfg, est["block_cnt"]) == 0.0


def test_select_diagonal_only_sparsity_closed_form():
    # S:280 only diagonal blocks: sparsity 1 - 2/(M+1)
    g = GOLD["diagonal_only_sparsity"]
    M = g["M"]
    cfg = oracle.Cfg(2, 1, 8, 64 * M, 64, 4, 1, 0.9)
    L = np.random.default_rng(0).standard_normal((1, M, M))
    cnt, idx, _ = oracle.select(cfg, L, [1, 1])
    assert np.all(cnt == 1)
    assert all(idx[0, m, 0] == m for m in range(M))
    assert oracle.sparsity(cfg, cnt) == pytest.approx(g["value"])


def test_select_brute_force_nested_and_ties():
    cfg = oracle.Cfg(4, 2, 8, 64 * 24, 64, 4, 1, 0.9, min_budget_tokens=128)
    M = cfg.M
    L = np.random.default_rng(1).standard_normal((1, M, M))
    L[0, 5, :5] = 0.25                                        # an all-tie row
    kstar = [2, 9, 17, 24]
    cnt, idx, mg = oracle.select(cfg, L, kstar)
    for h in range(4):
        for m in range(M):
            K = oracle.row_count(cfg, kstar[h], m)
            order = np.argsort(-L[0, m, :m], kind="stable")     # desc, ties -> lower index
            ref = sorted(set(order[:K - 1].tolist()) | {m})
            assert cnt[h, m] == K == len(ref)
            assert list(idx[h, m, :K]) == ref
            if h:                                             # S:263 nested across heads
                assert set(idx[h - 1, m, :cnt[h - 1, m]]) <= set(ref)
    assert list(idx[0, 5, :cnt[0, 5]]) == list(range(cnt[0, 5] - 1)) + [5]


def test_select_all_zero_q_tie_rule():
    # all-zero Q -> every proxy logit ties -> selection = {0..K-2} u {m} (Z17)
    cfg = oracle.Cfg(2, 1, 16, 64 * 12, 64, 4, 1, 0.7)
    Q = np.zeros((2, cfg.seq_len, 16), np.float32)
    K = np.random.default_rng(3).standard_normal((1, cfg.seq_len, 16)).astype(np.float32)
    est = oracle.estimate(cfg, Q, K)
    for h in range(2):
        for m in range(cfg.M):
            c = est["block_cnt"][h, m]
            assert list(est["block_idx"][h, m, :c]) == list(range(c - 1)) + [m]


# ------------------------------------------------------------------------------ O10 --
def test_attention_single_token_is_v_row():
    cfg = oracle.Cfg(2, 1, 8, 1, 1, 1, 1, 0.9)            # S:51 seq_len = 1
    Q, K, V = rand_qkv(cfg, 15)
    O = oracle.dense(cfg, Q, K, V)
    assert np.array_equal(O[:, 0], np.repeat(V[:1, 0].astype(np.float64), 2, axis=0))


def test_attention_two_token_hand_example():
    g = GOLD["two_token_attention"]
    q = np.array(g["q"], np.float32)[None]
    cfg = oracle.Cfg(1, 1, 4, 2, 2, 1, 1, 0.9)
    O = oracle.dense(cfg, q, q, q)
    w = g["row1_weights"]
    assert O[0, 1] == pytest.approx([w[0], w[1], 0, 0], abs=1e-15)
    assert O[0, 0] == pytest.approx([1, 0, 0, 0], abs=1e-15)


def test_attention_dense_matches_textbook_softmax():
    # S:53 brute-force O(N^2) two-pass reference; GQA mapping kv(h) = h // r
    cfg = oracle.Cfg(4, 2, 16, 64, 16, 4, 1, 0.9)
    Q, K, V = rand_qkv(cfg, 16, scale=1.7)
    O = oracle.dense(cfg, Q, K, V)
    for h in range(4):
        assert O[h] == pytest.approx(bf_attention(Q[h], K[h // 2], V[h // 2]), abs=1e-12)


def test_attention_full_mask_equals_dense_and_diag_is_windowed():
    cfg = oracle.Cfg(2, 1, 16, 128, 16, 4, 1, 0.9)
    Q, K, V = rand_qkv(cfg, 17)
    M = cfg.M
    full_cnt = np.tile(np.arange(1, M + 1, dtype=np.int32), (2, 1))
    full_idx = np.tile(np.arange(M, dtype=np.int32), (2, M, 1))
    Of = oracle.attention(cfg, Q, K, V, full_cnt, full_idx)
    Od = oracle.dense(cfg, Q, K, V)
    assert np.max(np.abs(Of - Od)) <= 1e-12                   # AC1
    diag_cnt = np.ones((2, M), np.int32)
    diag_idx = np.tile(np.arange(M, dtype=np.int32)[:, None], (2, 1, M))
    Ow = oracle.attention(cfg, Q, K, V, diag_cnt, diag_idx)
    blk = np.arange(cfg.seq_len) // cfg.block_size
    allowed = blk[:, None] == blk[None, :]                    # S:322 window = own block
    for h in range(2):
        assert Ow[h] == pytest.approx(bf_attention(Q[h], K[0], V[0], allowed), abs=1e-12)


def test_attention_independent_of_block_visit_order():
    # permuting the visitation order changes nothing beyond rounding
    cfg = oracle.Cfg(1, 1, 16, 256, 16, 4, 1, 0.9)
    Q, K, V = rand_qkv(cfg, 18)
    M = cfg.M
    rng = np.random.default_rng(0)
    cnt = np.array([[max(1, m // 2 + 1) for m in range(M)]], np.int32)
    idx = np.zeros((1, M, M), np.int32)
    for m in range(M):
        sel = sorted(set(rng.choice(m + 1, cnt[0, m] - 1, replace=False).tolist() if m else []) | {m})
        while len(sel) < cnt[0, m]:
            sel = sorted(set(sel) | {int(rng.integers(0, m + 1))})
        idx[0, m, :cnt[0, m]] = sel
    O1 = oracle.attention(cfg, Q, K, V, cnt, idx)
    idx2 = idx.copy()
    for m in range(M):
        idx2[0, m, :cnt[0, m]] = idx[0, m, :cnt[0, m]][::-1]
    O2 = oracle.attention(cfg, Q, K, V, cnt, idx2)
    assert np.max(np.abs(O1 - O2)) <= 1e-12


# ---------------------------------------------------------------- whole pipeline --
def test_pipeline_gamma_one_equals_dense_ac2():
    cfg = CFG_A.replace(seq_len=512, gamma=1.0)
    Q, K, V = rand_qkv(cfg, 19)
    est = oracle.pipeline(cfg, Q, K, V)
    assert np.max(np.abs(est["O"] - oracle.dense(cfg, Q, K, V))) <= 1e-12


def test_sparsity_direction_ac8():
    # AC8 / Table 1 (P:429 vs P:431): sparsity(0.90) >= sparsity(0.95) on fixed workloads
    cfg = oracle.Cfg(4, 2, 64, 2048, 64, 4, 1, 0.9)
    Q, K, _, _ = workloads.structured(4, 2, 2048, 64, seed=0, dtype=torch.float32)
    Q, K = Q.numpy(), K.numpy()
    s90 = oracle.sparsity(cfg, oracle.estimate(cfg, Q, K)["block_cnt"])
    s95 = oracle.sparsity(cfg, oracle.estimate(cfg.replace(gamma=0.95), Q, K)["block_cnt"])
    assert s90 >= s95 > 0.0


@pytest.mark.parametrize("case", GOLD["cost_ratio"], ids=lambda c: c["cite"][:5])
def test_cost_ratio_spec_examples(case):
    cfg = oracle.Cfg(case["n"], case["g"], 16, 64, 16, case["s"], case["g"], 0.9)
    assert oracle.cost_ratio(cfg) == pytest.approx(case["value"], rel=1e-12)
    if "approx" in case:
        assert round(oracle.cost_ratio(cfg), 4) == case["approx"]


def test_cost_ratio_counted_macs_ac7():
    # AC7: counted proxy QK^T MACs / dense QK^T MACs within 5 % of g/(n s^2) (Z22)
    for g, n, s in [(1, 32, 4), (4, 28, 4), (2, 16, 2)]:
        N, d = 1024, 64
        Ns = N // s
        proxy = g * d * Ns * (Ns + 1) / 2          # one logit per sampled causal (i, j)
        dense = n * d * N * (N + 1) / 2
        cfg = oracle.Cfg(n, g, d, N, 64, s, g, 0.9)
        assert proxy / dense == pytest.approx(oracle.cost_ratio(cfg), rel=0.05)


def test_block_reduce_sum_example():
    # S:71 N=4, b=2, uniform causal rows: block (1,0) sum = 2/3 + 2/4 (mass identity used by
    # Alg. 1's avgpool through oracle.budgets with all-zero Q)
    cfg = oracle.Cfg(1, 1, 4, 4, 2, 1, 1, 0.9)
    Q = np.zeros((1, 4, 4), np.float32)
    K = np.ones((1, 4, 4), np.float32)
    _, _, _, mass = oracle.budgets(cfg, Q, K)        # last block = rows 2, 3
    assert mass[0, 0] * 4 == pytest.approx(GOLD["block_reduce_sum"]["value"], abs=1e-15)


def test_item_subsets_match_full_rows():
    cfg = oracle.Cfg(4, 2, 16, 512, 64, 4, 1, 0.8)
    Q, K, V = rand_qkv(cfg, 21)
    est = oracle.pipeline(cfg, Q, K, V)
    items = [(3, 7), (0, 0), (2, 4)]
    Os = oracle.attention(cfg, Q, K, V, est["block_cnt"], est["block_idx"], items=items)
    Od = oracle.dense(cfg, Q, K, V, items=np.array(items).reshape(-1))
    Of = oracle.dense(cfg, Q, K, V)
    b = cfg.block_size
    for h, m in items:
        assert np.array_equal(Os[h, m * b:(m + 1) * b], est["O"][h, m * b:(m + 1) * b])
        assert np.array_equal(Od[h, m * b:(m + 1) * b], Of[h, m * b:(m + 1) * b])
    assert np.isnan(Os[1]).all()                      # rows not listed are not written


def test_determinism():
    cfg = CFG_A.replace(seq_len=512)
    Q, K, V = rand_qkv(cfg, 20)
    a = oracle.pipeline(cfg, Q, K, V)
    b = oracle.pipeline(cfg, Q, K, V)
    for k in ("L", "kstar", "block_cnt", "block_idx", "O"):
        assert np.array_equal(a[k], b[k], equal_nan=True)


# ------------------------------------------------------------- method variants --
def test_designated_head_equals_mean_for_singleton_groups_and_first_head_brute_force():
    # Z1 alternative ("a designated head"): with singleton groups it IS the mean
    cfg = oracle.Cfg(4, 4, 8, 256, 32, 4, 4, 0.9, round_bf16=True)
    Q, K, _ = rand_qkv(cfg, 31)
    a = oracle.estimate(cfg, Q, K)
    b = oracle.estimate(cfg.replace(designated_head=True), Q, K)
    assert np.array_equal(a["L"], b["L"]) and np.array_equal(a["block_idx"], b["block_idx"])
    # multi-head group, stride 1: exp(L) = block-max of the FIRST head's dense probabilities
    cfg2 = oracle.Cfg(4, 2, 8, 64, 16, 1, 1, 0.9, designated_head=True)
    Q2, K2, _ = rand_qkv(cfg2, 32, scale=2.0)
    Pq, Pk, scale = oracle.pool(cfg2, Q2, K2)
    assert scale == pytest.approx(1 / math.sqrt(8))
    _, L = oracle.proxy_scores(cfg2, Pq, Pk, scale)
    P = bf_probs(Q2[0], K2[0])
    b_ = cfg2.block_size
    for m in range(cfg2.M):
        for n in range(m + 1):
            ref = P[m * b_:(m + 1) * b_, n * b_:(n + 1) * b_].max()
            assert math.exp(L[0, m, n]) == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_static_topk_budgets_and_brute_force_masks():
    # Fig. 6c static top-K baseline: every head gets the same K*
    cfg = oracle.Cfg(4, 2, 16, 64 * 16, 64, 4, 1, 0.9, static_kstar=5)
    Q, K, _ = rand_qkv(cfg, 33)
    est = oracle.estimate(cfg, Q, K)
    assert np.all(est["kstar"] == 5)
    for h in range(4):
        for m in range(cfg.M):
            Kc = min(m + 1, max(-(-5 * (m + 1) // cfg.M), 1))
            order = np.argsort(-est["L"][0, m, :m], kind="stable")
            ref = sorted(set(order[:Kc - 1].tolist()) | {m})
            assert list(est["block_idx"][h, m, :est["block_cnt"][h, m]]) == ref


@pytest.mark.parametrize("case", GOLD["constant_k_sparsity"], ids=lambda c: str(c["M"]))
def test_constant_k_reading_counts_and_sparsity(case):
    M, ks = case["M"], case["kstar"]
    cfg = oracle.Cfg(1, 1, 32, 128 * M, 128, 4, 1, 0.9, constant_k=True)
    counts = [oracle.row_count(cfg, ks, m) for m in range(M)]
    assert counts == [min(m + 1, ks) for m in range(M)]
    assert 1 - sum(counts) / (M * (M + 1) / 2) == pytest.approx(case["sparsity"], abs=5e-5)


def test_force_sink_selects_block_zero_counted():
    cfg = oracle.Cfg(4, 2, 8, 64 * 20, 64, 4, 1, 0.9, force_sink=True)
    M = cfg.M
    L = np.random.default_rng(5).standard_normal((1, M, M))
    kstar = [1, 4, 9, 20]
    cnt, idx, _ = oracle.select(cfg, L, kstar)
    for h in range(4):
        for m in range(M):
            K = oracle.row_count(cfg, kstar[h], m)
            lst = idx[h, m, :cnt[h, m]].tolist()
            assert cnt[h, m] == K and lst[-1] == m
            others = [n for n in np.argsort(-L[0, m, :m], kind="stable").tolist() if n != 0]
            ref = {m} | ({0} if (K >= 2 and m > 0) else set()) | set(others[:max(K - 2, 0)])
            assert set(lst) == ref, (h, m)


# ------------------------------------------------------------------- ragged N --
def test_ragged_n_dense_and_degenerate_proxy_brute_force():
    # S:81 zero-pad + mask: the block structure must not change the textbook results
    cfg = oracle.Cfg(2, 2, 8, 90, 16, 1, 2, 0.9)          # M = 6, last block has 10 tokens
    assert cfg.M == 6 and cfg.Ns == 90
    Q, K, V = rand_qkv(cfg, 41, scale=2.0)
    O = oracle.dense(cfg, Q, K, V)
    for h in range(2):
        assert O[h] == pytest.approx(bf_attention(Q[h], K[h], V[h]), abs=1e-12)
    Pq, Pk, scale = oracle.pool(cfg, Q, K)
    _, L = oracle.proxy_scores(cfg, Pq, Pk, scale)
    b = cfg.block_size
    for h in range(2):
        P = bf_probs(Q[h], K[h])
        for m in range(cfg.M):
            for n in range(m + 1):
                ref = P[m * b:(m + 1) * b, n * b:(n + 1) * b].max()   # slices clip at N
                assert math.exp(L[h, m, n]) == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_ragged_n_budget_brute_force_uses_partial_last_block():
    cfg = oracle.Cfg(2, 1, 16, 300, 64, 4, 1, 0.8)         # M = 5, last block rows 256..299
    Q, K, _ = rand_qkv(cfg, 42, scale=1.5)
    kstar, _, _, mass = oracle.budgets(cfg, Q, K)
    b, M, N = 64, cfg.M, 300
    for h in range(2):
        P = bf_probs(Q[h], K[0])[(M - 1) * b:N]              # the last block's 44 real rows
        a = np.array([P[:, n * b:(n + 1) * b].sum() for n in range(M)]) / b ** 2
        assert mass[h] == pytest.approx(a, rel=1e-10, abs=1e-18)
        srt = np.sort(a)[::-1]
        ref = int(np.argmax(np.cumsum(srt / srt.sum()) >= cfg.gamma)) + 1
        assert kstar[h] == ref


def test_ragged_n_sampled_rows_and_gamma_one_equals_dense():
    cfg = oracle.Cfg(4, 2, 16, 1000, 64, 4, 1, 1.0)          # Ns = 250, last block: 232 tokens
    Q, K, V = rand_qkv(cfg, 43)
    Pq, _, _ = oracle.pool(cfg, Q, K)
    assert Pq.shape[1] == 250
    assert np.array_equal(Pq[0, 249], Q[:, 996].astype(np.float64).sum(0))
    est = oracle.pipeline(cfg, Q, K, V)
    assert np.max(np.abs(est["O"] - oracle.dense(cfg, Q, K, V))) <= 1e-12


def _attention_recall(oc, Q, K, cnt, idx):
    """Mean over (head, query) of the dense causal softmax mass that falls on the query's
    selected blocks (keys k <= t in them), fp64 brute force."""
    H, N, d = Q.shape
    r, b = oc.n_q_heads // oc.n_kv_heads, oc.block_size
    tot = 0.0
    t = np.arange(N)
    for h in range(H):
        S = (Q[h].astype(np.float64) @ K[h // r].astype(np.float64).T) / math.sqrt(d)
        S[t[:, None] < t[None, :]] = -np.inf
        P = np.exp(S - S.max(axis=1, keepdims=True))
        P /= P.sum(axis=1, keepdims=True)
        keep = np.zeros((N, N), bool)
        for m in range((N + b - 1) // b):
            for n in idx[h, m, :cnt[h, m]]:
                keep[m * b:(m + 1) * b, n * b:(n + 1) * b] = True
        tot += float((P * keep).sum(axis=1).mean())
    return tot / H


def test_recall_under_budget_shared_focus():
    # SPEC AC6 as a pin of the estimate's intent (§3.2: gamma is the attention mass the budget
    # should cover): gamma = 0.95, stride 4, one proxy group, shared-focus multi-temperature
    # inputs -> mean dense-attention recall of the selected blocks above SPEC's hard floor 0.85
    # (measured 0.881 on this generator: Alg. 1 sizes K* on the LAST block's rows, earlier rows
    # get the per-row ratio of Z12 and the proxy ranking, so recall sits a little below gamma;
    # SPEC's 0.90 target is for its own workload); and recall grows with gamma (0.759 at 0.90)
    N, Hq, Hkv, d, b = 2048, 8, 2, 64, 64
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=3)
    Qf, Kf = Q.float().numpy(), K.float().numpy()
    rec = {}
    for gamma in (0.9, 0.95):
        oc = oracle.Cfg(Hq, Hkv, d, N, b, 4, 1, gamma, round_bf16=True)
        est = oracle.estimate(oc, Qf, Kf)
        rec[gamma] = _attention_recall(oc, Qf, Kf, est["block_cnt"], est["block_idx"])
    assert rec[0.95] >= 0.85, rec
    assert rec[0.95] > rec[0.9], rec
