"""GPU parity: the CUDA path (through the C-ABI) against the fp64 CPU oracle on the same
seeded inputs, following the staged protocol of SURVEY.md §8(c).5:

  1. pooled proxies       — exact fp32 sums (bf16 RNE of them is then identical)
  2. L (log-domain map)   — |dL| <= 1e-4 on valid cells, -inf on invalid ones
  3. kstar                — exact for heads whose budget margin > 1e-4
  4. block lists          — exact (ascending) for rows whose cut margin > 1e-4
  5. O with a mask injected — bf16: max-abs <= 2e-2, mean-abs <= 2e-3; fp32 debug: 1e-4
Each stage can take the other side's upstream result so a mismatch localises.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None
GAMMAS = [0.5, 0.7, 0.9, 0.95, 1.0]
MARGIN = 1e-4
BF16_MAX, BF16_MEAN, FP32_TOL = 2e-2, 2e-3, 1e-4


def ocfg_of(cfg: pa.Config) -> oracle.Cfg:
    return oracle.Cfg(cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.seq_len, cfg.block_size,
                      cfg.stride, cfg.n_groups, cfg.gamma, cfg.min_budget_tokens,
                      round_bf16=not cfg.fp32_debug, force_sink=cfg.force_sink,
                      constant_k=cfg.constant_k, designated_head=cfg.designated_head,
                      static_kstar=cfg.static_kstar)


def to_dev(*ts):
    return [t.to(DEV).contiguous() for t in ts]


def np32(t):
    return t.float().cpu().numpy()


def check_masks(ocfg, L_ref, kstar_gpu, cnt, idx, rows=None, per_head=False):
    """Stage 4: oracle selection from the oracle's L (per_head: the comparator's per-head
    maps) with the GPU budgets injected.  Every (head, row) is checked:
    * the counts are equal (A5 is integer arithmetic);
    * rows whose cut margin > 1e-4: the ascending lists are identical;
    * near-tie rows: the GPU list is valid (ascending, in range, diagonal last) and may differ
      from the oracle's only in blocks whose oracle score lies within 1e-4 of the cut (the
      lowest kept non-diagonal score): a block only the GPU kept scores >= cut - 1e-4, a
      block only the oracle kept scores <= cut + 1e-4, and there are as many of each.
    Returns (exact rows, near-tie rows); prints the near-tie fraction."""
    sel = oracle.select_heads if per_head else oracle.select
    if per_head:
        ocnt, oidx, cmg = sel(ocfg, L_ref, kstar_gpu)
    else:
        ocnt, oidx, cmg = sel(ocfg, L_ref, kstar_gpu, rows=rows)
    cnt = cnt.cpu().numpy() if torch.is_tensor(cnt) else np.asarray(cnt)
    idx = idx.cpu().numpy() if torch.is_tensor(idx) else np.asarray(idx)
    rows = range(ocfg.M) if rows is None else rows
    checked = near = 0
    for h in range(ocfg.n_q_heads):
        grp = h if per_head else oracle.group_of_q(ocfg, h)
        for m in rows:
            assert cnt[h, m] == ocnt[h, m], (h, m)
            c = ocnt[h, m]
            got, ref = idx[h, m, :c], oidx[h, m, :c]
            if cmg[h, m] > MARGIN:
                assert np.array_equal(got, ref), (h, m, got, ref)
                checked += 1
                continue
            near += 1
            assert got[-1] == m and np.all(np.diff(got) > 0) and got[0] >= 0, (h, m, got)
            lr = L_ref[grp, m, :m + 1]
            kept = [n for n in ref[:-1] if not (ocfg.force_sink and n == 0)]
            cut = lr[kept].min()
            only_gpu, only_ref = np.setdiff1d(got, ref), np.setdiff1d(ref, got)
            assert len(only_gpu) == len(only_ref), (h, m)
            assert np.all(lr[only_gpu] >= cut - MARGIN) and np.all(lr[only_ref] <= cut + MARGIN), \
                (h, m, cut, lr[only_gpu], lr[only_ref])
    total = checked + near
    if total:
        print(f"selection: {checked} rows exact, {near} near-tie rows ({near / total:.2%}) within 1e-4 of the cut")
    return checked, near


def check_out(O_gpu, O_ref, fp32):
    err = np.abs(np32(O_gpu) - O_ref)
    err = err[~np.isnan(O_ref)]
    if fp32:
        assert err.max() <= FP32_TOL, err.max()
    else:
        assert err.max() <= BF16_MAX and err.mean() <= BF16_MEAN, (err.max(), err.mean())
    return float(err.max()), float(err.mean())


# --------------------------------------------------------------------- tcgen05 --
def test_umma_descriptor_encodings():
    g = torch.Generator(device=DEV).manual_seed(0)
    A = torch.randn(128, 128, generator=g, device=DEV).bfloat16()
    B = torch.randn(128, 128, generator=g, device=DEV).bfloat16()
    Css, Cts = pa.debug_umma(A, B)
    torch.cuda.synchronize()
    ref_ss = A.float() @ B.float().T
    ref_ts = A.float() @ B.float()
    assert torch.allclose(Css, ref_ss, rtol=1e-4, atol=1e-3), (Css - ref_ss).abs().max()
    assert torch.allclose(Cts, ref_ts, rtol=1e-4, atol=1e-3), (Cts - ref_ts).abs().max()


# ----------------------------------------------------------- config A, fp32 --
CFG_A = pa.Config(n_q_heads=8, n_kv_heads=2, head_dim=64, seq_len=1024, block_size=64,
                  stride=4, n_groups=2, gamma=0.9, fp32_debug=True)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("gamma", GAMMAS)
def test_config_a_fp32_staged(seed, gamma):
    cfg = CFG_A.replace(gamma=gamma)
    oc = ocfg_of(cfg)
    Q, K, V = workloads.iid(8, 2, 1024, 64, seed)
    Qf, Kf, Vf = Q.numpy(), K.numpy(), V.numpy()
    Qd, Kd, Vd = to_dev(Q, K, V)
    # stage 1: pooled sums
    qsum, ksum = pa.pool(cfg, Qd, Kd)
    Pq, Pk, scale = oracle.pool(oc, Qf, Kf)
    assert np.allclose(qsum.cpu().numpy(), Pq, rtol=1e-6, atol=1e-6)
    assert np.allclose(ksum.cpu().numpy(), Pk, rtol=1e-6, atol=1e-6)
    # stage 2: L from the GPU's sums
    L = pa.proxy_scores(cfg, qsum, ksum)
    lse, Lref = oracle.proxy_scores(oc, Pq, Pk, scale)
    Lg = L.cpu().numpy().astype(np.float64)
    valid = np.isfinite(Lref)
    assert np.array_equal(np.isfinite(Lg), valid)
    assert np.max(np.abs(Lg[valid] - Lref[valid])) <= 1e-4
    # stage 3: budgets
    kstar, budget = pa.budgets(cfg, Qd, Kd)
    ks_ref, _, bmg, _ = oracle.budgets(oc, Qf, Kf)
    ks = kstar.cpu().numpy()
    ok = bmg > MARGIN
    assert np.array_equal(ks[ok], ks_ref[ok])
    assert np.all(np.abs(ks - ks_ref) <= 1)
    assert np.allclose(budget.cpu().numpy(), ks / oc.M)
    # stage 4: selection from the GPU L must match the oracle's selection on the same L exactly
    cnt, idx = pa.select(cfg, L, kstar)
    ocnt, oidx, _ = oracle.select(oc, Lg, ks)
    c_np, i_np = cnt.cpu().numpy(), idx.cpu().numpy()
    assert np.array_equal(c_np, ocnt)
    for h in range(8):
        for m in range(oc.M):
            assert np.array_equal(i_np[h, m, :ocnt[h, m]], oidx[h, m, :ocnt[h, m]])
    # ... and from the oracle's L, margin-gated
    check_masks(oc, Lref, ks, cnt, idx)
    # stage 5: O with the oracle mask injected, and dense
    O = pa.prefill(cfg, Qd, Kd, Vd, torch.from_numpy(ocnt).to(DEV), torch.from_numpy(oidx.clip(0)).to(DEV))
    check_out(O, oracle.attention(oc, Qf, Kf, Vf, ocnt, oidx), fp32=True)
    if gamma == 1.0:
        Od = pa.dense_prefill(cfg, Qd, Kd, Vd)
        check_out(Od, oracle.dense(oc, Qf, Kf, Vf), fp32=True)
        assert torch.equal(O, Od) or torch.allclose(O, Od, atol=1e-6)   # AC2


def test_config_a_fp32_ragged_n():
    cfg = CFG_A.replace(seq_len=1000)                    # M = 16, last block 40 tokens
    oc = ocfg_of(cfg)
    Q, K, V = workloads.iid(8, 2, 1000, 64, 7)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    est = oracle.estimate(oc, Q.numpy(), K.numpy())
    ks = kstar.cpu().numpy()
    ok = est["budget_margin"] > MARGIN
    assert np.array_equal(ks[ok], est["kstar"][ok])
    check_masks(oc, est["L"], ks, cnt, idx)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    check_out(O, oracle.attention(oc, Q.numpy(), K.numpy(), V.numpy(), cnt.cpu().numpy(),
                                  idx.cpu().numpy()), fp32=True)
    check_out(pa.dense_prefill(cfg, Qd, Kd, Vd), oracle.dense(oc, Q.numpy(), K.numpy(), V.numpy()), fp32=True)


def test_config_a_fp32_end_to_end_matches_staged():
    cfg = CFG_A
    Q, K, V = to_dev(*workloads.iid(8, 2, 1024, 64, 5))
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
    qsum, ksum = pa.pool(cfg, Q, K)
    L = pa.proxy_scores(cfg, qsum, ksum)
    k2, _ = pa.budgets(cfg, Q, K)
    c2, i2 = pa.select(cfg, L, k2)
    assert torch.equal(kstar, k2) and torch.equal(cnt, c2)
    for h in range(8):
        for m in range(cfg.M):
            n = int(cnt[h, m])
            assert torch.equal(idx[h, m, :n], i2[h, m, :n])


# ------------------------------------------------- bf16, structured, small N --
def llama_small(N=2048, gamma=0.9, heads=(8, 2), g=1, min_budget=0, stride=4):
    return pa.Config(n_q_heads=heads[0], n_kv_heads=heads[1], head_dim=128, seq_len=N,
                     block_size=128, stride=stride, n_groups=g, gamma=gamma,
                     min_budget_tokens=min_budget)


@pytest.mark.parametrize("case", [
    dict(N=2048, gamma=0.9, heads=(8, 2), g=1, seed=0),
    dict(N=2048, gamma=0.95, heads=(8, 2), g=2, seed=1),
    dict(N=4096, gamma=0.9, heads=(7, 1), g=1, seed=2, min_budget=512),     # Qwen-like r=7
    dict(N=1152, gamma=0.7, heads=(4, 4), g=2, seed=3),                     # ragged: M=9
    dict(N=1024, gamma=0.9, heads=(8, 2), g=1, seed=4, stride=1),           # b/s = 128
    dict(N=2048, gamma=0.9, heads=(8, 2), g=2, seed=5, stride=2),           # b/s = 64
    dict(N=4096, gamma=0.9, heads=(8, 2), g=1, seed=6, stride=8),           # b/s = 16
    dict(N=2000, gamma=0.9, heads=(8, 2), g=1, seed=7),                     # ragged N
    dict(N=3001, gamma=0.95, heads=(7, 1), g=1, seed=8, min_budget=256),    # ragged, N % s != 0
    dict(N=700, gamma=0.7, heads=(4, 2), g=2, seed=9, stride=2),            # ragged, M = 6
])
def test_bf16_structured_staged(case):
    case = dict(case)
    seed = case.pop("seed")
    cfg = llama_small(**case)
    oc = ocfg_of(cfg)
    Hq, Hkv = cfg.n_q_heads, cfg.n_kv_heads
    Q, K, V, _ = workloads.structured(Hq, Hkv, cfg.seq_len, 128, seed=seed)
    Qf, Kf, Vf = np32(Q), np32(K), np32(V)
    Qd, Kd, Vd = to_dev(Q, K, V)
    # stage 1: fp32 sums are exact (bf16 inputs), so their bf16 RNE equals the oracle's
    qsum, ksum = pa.pool(cfg, Qd, Kd)
    Pq, Pk, scale = oracle.pool(oc.replace(round_bf16=False), Qf, Kf)
    for got, ref in ((qsum, Pq), (ksum, Pk)):                 # fp32 view of the exact sum
        assert np.array_equal(got.cpu().numpy(), ref.astype(np.float32))
    Pq_r, Pk_r, _ = oracle.pool(oc, Qf, Kf)
    # the staged path rounds the fp32 view to bf16 (double rounding only at exact ties)
    assert np.mean(qsum.bfloat16().double().cpu().numpy() == Pq_r) >= 0.9999
    # stage 2
    L = pa.proxy_scores(cfg, qsum, ksum)
    _, Lref = oracle.proxy_scores(oc, Pq_r, Pk_r, scale)
    Lg = L.cpu().numpy().astype(np.float64)
    valid = np.isfinite(Lref)
    assert np.array_equal(np.isfinite(Lg), valid)
    assert np.max(np.abs(Lg[valid] - Lref[valid])) <= 1e-4
    # stage 3
    kstar, _ = pa.budgets(cfg, Qd, Kd)
    ks_ref, _, bmg, _ = oracle.budgets(oc, Qf, Kf)
    ks = kstar.cpu().numpy()
    ok = bmg > MARGIN
    assert np.array_equal(ks[ok], ks_ref[ok]), (ks, ks_ref, bmg)
    # stage 4 (fused estimate)
    k2, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    assert torch.equal(k2, kstar)
    checked, skipped = check_masks(oc, Lref, ks, cnt, idx)
    assert checked > 0.9 * (checked + skipped)
    # stage 5: O with the GPU mask injected into the oracle
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    check_out(O, oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy()), fp32=False)
    Od = pa.dense_prefill(cfg, Qd, Kd, Vd)
    check_out(Od, oracle.dense(oc, Qf, Kf, Vf), fp32=False)


# ------------------------------------------------------------------ edge cases --
def test_single_block_and_gamma_one_equals_dense():
    cfg = llama_small(N=128, gamma=0.9)                       # M = 1: diagonal only
    Q, K, V, _ = workloads.structured(8, 2, 128, 128, seed=4)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    assert torch.all(kstar == 1) and torch.all(cnt == 1) and torch.all(idx[:, 0, 0] == 0)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    check_out(O, oracle.dense(ocfg_of(cfg), np32(Q), np32(K), np32(V)), fp32=False)
    cfg1 = llama_small(N=1024, gamma=1.0)
    Q, K, V, _ = workloads.structured(8, 2, 1024, 128, seed=5)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg1, Qd, Kd)
    assert torch.all(kstar == cfg1.M)
    O = pa.prefill(cfg1, Qd, Kd, Vd, cnt, idx)
    Od = pa.dense_prefill(cfg1, Qd, Kd, Vd)
    # AC2: gamma = 1 -> dense.  The sparse launch (attn_tc8) and the dense baseline
    # (attn_tc) are different kernels (different softmax reference points and P rounding),
    # so they agree within the bf16 output tolerance, not bitwise.
    assert (O.float() - Od.float()).abs().max().item() <= 2e-2
    check_out(O, oracle.dense(ocfg_of(cfg1), np32(Q), np32(K), np32(V)), fp32=False)
    Os = pa.prefill(cfg1, Qd, Kd, Vd, cnt, idx)
    assert torch.equal(O, Os)                                 # deterministic


def test_min_budget_floor_saturates_and_all_zero_q_ties():
    cfg = llama_small(N=1024, gamma=0.5, min_budget=8 * 128)  # F = M -> full mask
    Q, K, V, _ = workloads.structured(8, 2, 1024, 128, seed=6)
    Qd, Kd, _ = to_dev(Q, K, V)
    _, _, cnt, _ = pa.estimate(cfg, Qd, Kd)
    assert torch.equal(cnt.cpu(), torch.arange(1, 9, dtype=torch.int32).repeat(8, 1))
    cfg0 = llama_small(N=2048, gamma=0.7)
    _, K0, _, _ = workloads.structured(8, 2, 2048, 128, seed=16)
    Qz = torch.zeros(8, 2048, 128, dtype=torch.bfloat16, device=DEV)
    kstar, _, cnt, idx = pa.estimate(cfg0, Qz, K0.to(DEV))
    for h in range(8):
        for m in range(cfg0.M):
            c = int(cnt[h, m])
            assert idx[h, m, :c].cpu().tolist() == list(range(c - 1)) + [m]


def test_check_flag_rejects_bad_lists():
    cfg = llama_small(N=512).replace(check=True)
    Q, K, V, _ = workloads.structured(8, 2, 512, 128, seed=7)
    Qd, Kd, Vd = to_dev(Q, K, V)
    cnt = torch.ones(8, 4, dtype=torch.int32, device=DEV)
    idx = torch.zeros(8, 4, 4, dtype=torch.int32, device=DEV)
    idx[:, :, 0] = torch.arange(4, device=DEV, dtype=torch.int32)
    pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)                      # diagonal-only lists: valid
    bad = idx.clone()
    bad[3, 2, 0] = 3                                           # acausal block
    with pytest.raises(pa.ProxyAttnError) as ei:
        pa.prefill(cfg, Qd, Kd, Vd, cnt, bad)
    assert ei.value.code == pa._lib.E_SHAPE
    zero = cnt.clone()
    zero[0, 1] = 0                                             # empty row
    with pytest.raises(pa.ProxyAttnError):
        pa.prefill(cfg, Qd, Kd, Vd, zero, idx)


def test_determinism_bitwise():
    cfg = llama_small(N=2048)
    Q, K, V, _ = workloads.structured(8, 2, 2048, 128, seed=8)
    Qd, Kd, Vd = to_dev(Q, K, V)
    a = pa.estimate(cfg, Qd, Kd)
    Oa = pa.prefill(cfg, Qd, Kd, Vd, a[2], a[3])
    b = pa.estimate(cfg, Qd, Kd)
    Ob = pa.prefill(cfg, Qd, Kd, Vd, b[2], b[3])
    assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2]) and torch.equal(Oa, Ob)


def test_forward_host_matches_device_path():
    cfg = llama_small(N=1024)
    Q, K, V, _ = workloads.structured(8, 2, 1024, 128, seed=9)
    Qh, Kh, Vh = Q.pin_memory(), K.pin_memory(), V.pin_memory()
    Oh = torch.empty_like(Qh).pin_memory()
    ks = torch.empty(8, dtype=torch.int32).pin_memory()
    ws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=DEV)
    pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws, ks)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    torch.cuda.synchronize()
    assert torch.equal(ks, kstar.cpu()) and torch.equal(Oh, O.cpu())


# ------------------------------------------------------------ method variants --
@pytest.mark.parametrize("variant", [dict(designated_head=True), dict(static_kstar=7),
                                     dict(constant_k=True), dict(force_sink=True),
                                     dict(force_sink=True, constant_k=True, n_groups=2)],
                         ids=["designated", "static7", "constantK", "sink", "sink+constK+g2"])
def test_method_variants_match_oracle(variant):
    variant = dict(variant)
    g = variant.pop("n_groups", 1)
    cfg = llama_small(N=2048, gamma=0.9, g=g).replace(**variant)
    oc = ocfg_of(cfg)
    Q, K, V, _ = workloads.structured(8, 2, 2048, 128, seed=11)
    Qf, Kf, Vf = np32(Q), np32(K), np32(V)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    est = oracle.estimate(oc, Qf, Kf)
    ks = kstar.cpu().numpy()
    ok = est["budget_margin"] > MARGIN
    assert np.array_equal(ks[ok], est["kstar"][ok])
    if cfg.static_kstar:
        assert np.all(ks == cfg.static_kstar)
    checked, skipped = check_masks(oc, est["L"], ks, cnt, idx)
    assert checked > 0.9 * (checked + skipped)
    if cfg.force_sink:
        c_np, i_np = cnt.cpu().numpy(), idx.cpu().numpy()
        for h in range(8):
            for m in range(1, cfg.M):
                if c_np[h, m] >= 2:
                    assert i_np[h, m, 0] == 0
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    check_out(O, oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy()), fp32=False)


def test_variant_fp32_debug_designated_config_a():
    cfg = CFG_A.replace(designated_head=True, force_sink=True)
    oc = ocfg_of(cfg)
    Q, K, V = workloads.iid(8, 2, 1024, 64, 3)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    est = oracle.estimate(oc, Q.numpy(), K.numpy())
    ks = kstar.cpu().numpy()
    ok = est["budget_margin"] > MARGIN
    assert np.array_equal(ks[ok], est["kstar"][ok])
    check_masks(oc, est["L"], ks, cnt, idx)


def test_row_range_prefill_matches_full_bitwise():
    # zig-zag row sharding building block: rows [b, e) only, other rows untouched
    from paper_2509_24745_b200 import shard
    cfg = llama_small(N=4096)
    Q, K, V, _ = workloads.structured(8, 2, 4096, 128, seed=12)
    Qd, Kd, Vd = to_dev(Q, K, V)
    _, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    full = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    for world in (2, 3):
        O = torch.zeros_like(full)
        for rank in range(world):
            shard.prefill_rows(cfg, Qd, Kd, Vd, cnt, idx, O,
                               shard.zigzag_rows(cfg.M, world, rank, shard.row_align(cfg)))
        assert torch.equal(O, full)
    # a range aligned to the kernel's block-row pairs: bit for bit; an unaligned one splits a
    # pair (row 5 alone: its own two first blocks set its reference) -> within tolerance
    for b, e, exact in ((4, 12, True), (5, 12, False)):
        part = torch.zeros_like(full)
        pa.prefill(cfg.replace(row_begin=b, row_end=e), Qd, Kd, Vd, cnt, idx, part)
        if exact:
            assert torch.equal(part[:, b * 128:e * 128], full[:, b * 128:e * 128])
        else:
            d = (part[:, b * 128:e * 128].float() - full[:, b * 128:e * 128].float()).abs()
            assert d.max().item() <= 2e-2 and d.mean().item() <= 2e-3
        assert torch.all(part[:, :b * 128] == 0) and torch.all(part[:, e * 128:] == 0)


def test_score_spikes_wide_dynamic_range():
    # Keys whose scores jump far above (and below) the first blocks' maxima: the softmax
    # reference of attn_tc7 is fixed per row (shift invariance of softmax), so
    # these exercise its large-P fast path (+20 in log2 units) and its exact second pass
    # (+80: the reference is replaced by the row's true max).  Head 3 sees the spikes negated.
    cfg = llama_small(N=2048, gamma=1.0, heads=(4, 1))
    g = torch.Generator().manual_seed(21)
    Q = (torch.randn(4, 2048, 128, generator=g) * 0.5 + 0.5)
    Q[3] = -Q[3]
    K = torch.randn(1, 2048, 128, generator=g) * 0.5
    V = torch.randn(1, 2048, 128, generator=g)
    K[0, 7 * 128 + 5] = 2.5                                   # ~ +20 log2 over the reference
    K[0, 9 * 128 + 77] = 10.0                                 # ~ +80: second pass
    K[0, 12 * 128 + 1] = -20.0                                # far below: underflows to 0
    Q, K, V = Q.bfloat16(), K.bfloat16(), V.bfloat16()
    Qd, Kd, Vd = to_dev(Q, K, V)
    _, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    assert torch.all(cnt.cpu() == torch.arange(1, 17, dtype=torch.int32))
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    assert torch.isfinite(O.float()).all()
    ref = oracle.attention(ocfg_of(cfg), np32(Q), np32(K), np32(V), cnt.cpu().numpy(),
                           idx.cpu().numpy())
    check_out(O, ref, fp32=False)
    Od = pa.dense_prefill(cfg, Qd, Kd, Vd)
    check_out(Od, ref, fp32=False)


@pytest.mark.parametrize("N", [4096, 3001])
def test_row_range_estimate_matches_full_bitwise(N):
    # zig-zag row sharding of the estimate: each rank computes the lists of its rows only
    # (proxies of its sampled rows and the keys before them, the covering proxy tiles,
    # selection of its rows), Alg. 1 once per rank; the lists must equal the full estimate's
    from paper_2509_24745_b200 import shard
    cfg = llama_small(N=N)
    Q, K, V, _ = workloads.structured(8, 2, N, 128, seed=13)
    Qd, Kd, _ = to_dev(Q, K, V)
    kstar, budget, cnt, idx = pa.estimate(cfg, Qd, Kd)
    for world in (2, 3):
        for rank in range(world):
            rows = shard.zigzag_rows(cfg.M, world, rank)
            out = (torch.zeros_like(kstar), torch.zeros_like(budget), torch.zeros_like(cnt),
                   torch.full_like(idx, -7))
            k2, b2, c2, i2 = shard.estimate_rows(cfg, Qd, Kd, rows, out=out)
            assert torch.equal(k2, kstar) and torch.equal(b2, budget)
            for b, e in rows:
                assert torch.equal(c2[:, b:e], cnt[:, b:e])
                for h in range(8):
                    for m in range(b, e):
                        c = int(cnt[h, m])
                        assert torch.equal(i2[h, m, :c], idx[h, m, :c])
            covered = torch.zeros(cfg.M, dtype=torch.bool)
            for b, e in rows:
                covered[b:e] = True
            assert torch.all(c2[:, ~covered.to(c2.device)] == 0)   # other rows untouched
