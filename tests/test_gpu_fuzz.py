"""GPU parity on seeded random configurations (bf16 tensor-core path) against the fp64 oracle,
staged as in SURVEY §8(c).5: budgets on margin-qualified heads, block lists on
margin-qualified rows, O with the GPU mask injected, and the dense path.  Each case draws
head_dim and block size from the supported set, a GQA ratio (odd ones included), a
proxy-group count dividing the KV heads, a stride dividing the block, gamma, a minimum
budget, a ragged length spanning several tiles, and i.i.d. or structured inputs — the
combinations the hand-written cases do not enumerate.  The FP32_DEBUG build is fuzzed over
its wider shape set at the 1e-4 tolerance."""
import numpy as np
import pytest

import oracle
import paper_2509_24745_b200 as pa
import workloads
from test_gpu_parity import DEV, MARGIN, check_masks, check_out, ocfg_of, to_dev
from test_gpu_shapes import run_staged

pytestmark = pytest.mark.gpu


def draw(case: int):
    rng = np.random.default_rng(1000 + case)
    d = int(rng.choice([64, 128]))
    b = int(rng.choice([64, 128]))
    Hkv = int(rng.choice([1, 2, 4]))
    r = int(rng.choice([1, 2, 3, 4, 7]))
    g = int(rng.choice([x for x in (1, 2, 4) if Hkv % x == 0]))
    s = int(rng.choice([2, 4, 8]))
    gamma = float(rng.choice([0.6, 0.8, 0.9, 0.95]))
    min_budget = int(rng.choice([0, 0, b, 3 * b]))
    N = int(rng.integers(3 * b, 24 * b)) | 1          # odd: always a partial last block
    structured = bool(rng.integers(0, 2))
    return dict(d=d, b=b, Hq=Hkv * r, Hkv=Hkv, g=g, s=s, gamma=gamma, min_budget=min_budget, N=N,
                structured=structured)


@pytest.mark.parametrize("case", range(64))
def test_random_config_staged(case):
    c = draw(case)
    cfg = pa.Config(c["Hq"], c["Hkv"], c["d"], c["N"], c["b"], c["s"], c["g"], c["gamma"], c["min_budget"])
    if c["structured"]:
        Q, K, V, _ = workloads.structured(c["Hq"], c["Hkv"], c["N"], c["d"], seed=case)
    else:
        Q, K, V = (t.bfloat16() for t in workloads.iid(c["Hq"], c["Hkv"], c["N"], c["d"], seed=case))
    run_staged(cfg, Q, K, V, min_checked=0.75)


def draw_fp32(case: int):
    rng = np.random.default_rng(5000 + case)
    d = int(rng.choice([32, 64, 96, 128]))
    b = int(rng.choice([16, 32, 48, 64, 128]))
    s = int(rng.choice([x for x in (1, 2, 4, 8) if b % x == 0]))
    Hkv = int(rng.choice([1, 2, 4]))
    r = int(rng.choice([1, 2, 3, 4]))
    g = int(rng.choice([x for x in (1, 2, 4) if Hkv % x == 0]))
    gamma = float(rng.choice([0.5, 0.7, 0.9, 0.95, 1.0]))
    min_budget = int(rng.choice([0, 0, b, 2 * b]))
    N = int(rng.integers(2 * b, 20 * b))
    return dict(d=d, b=b, s=s, Hq=Hkv * r, Hkv=Hkv, g=g, gamma=gamma, min_budget=min_budget, N=N)


@pytest.mark.parametrize("case", range(32))
def test_random_config_fp32_debug(case):
    # the FP32_DEBUG build (SIMT kernels, the 1e-4 contract) over its wider shape set:
    # d % 32 == 0, any b divisible by s, ragged N
    c = draw_fp32(case)
    cfg = pa.Config(c["Hq"], c["Hkv"], c["d"], c["N"], c["b"], c["s"], c["g"], c["gamma"], c["min_budget"],
                    fp32_debug=True)
    oc = ocfg_of(cfg)
    Q, K, V = workloads.iid(c["Hq"], c["Hkv"], c["N"], c["d"], seed=case)
    Qf, Kf, Vf = Q.numpy(), K.numpy(), V.numpy()
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    est = oracle.estimate(oc, Qf, Kf)
    ks = kstar.cpu().numpy()
    ok = est["budget_margin"] > MARGIN
    assert np.array_equal(ks[ok], est["kstar"][ok])
    assert np.all(np.abs(ks - est["kstar"]) <= 1)
    checked, skipped = check_masks(oc, est["L"], ks, cnt, idx)
    assert checked >= 0.75 * (checked + skipped)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    check_out(O, oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy()), fp32=True)
    check_out(pa.dense_prefill(cfg, Qd, Kd, Vd), oracle.dense(oc, Qf, Kf, Vf), fp32=True)


@pytest.mark.parametrize("case", range(32))
def test_random_config_layouts_and_shards_bitwise(case):
    # on the bf16 random configurations: token-major views, and the zig-zag row-sharded
    # estimate (K* given, scores only + select) and prefill over 2-4 ranks, must reproduce the
    # head-major one-call results BIT for bit (layout and row ranges change addressing only)
    from paper_2509_24745_b200 import shard
    import torch
    c = draw(case)
    cfg = pa.Config(c["Hq"], c["Hkv"], c["d"], c["N"], c["b"], c["s"], c["g"], c["gamma"], c["min_budget"])
    Q, K, V, _ = workloads.structured(c["Hq"], c["Hkv"], c["N"], c["d"], seed=100 + case)
    Qd, Kd, Vd = to_dev(Q, K, V)
    kstar, budget, cnt, idx = pa.estimate(cfg, Qd, Kd)
    full = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)

    def same_lists(c2, i2, rows=None):
        assert torch.equal(c2 if rows is None else c2[:, rows], cnt if rows is None else cnt[:, rows])
        c_np, a, b_ = cnt.cpu().numpy(), idx.cpu().numpy(), i2.cpu().numpy()
        for h in range(cfg.n_q_heads):
            for m in (range(cfg.M) if rows is None else rows):
                assert np.array_equal(a[h, m, :c_np[h, m]], b_[h, m, :c_np[h, m]]), (h, m)
    tcfg = cfg.replace(token_major=True)
    Qt, Kt, Vt = (x.transpose(0, 1).contiguous() for x in (Qd, Kd, Vd))
    k2, _, c2, i2 = pa.estimate(tcfg, Qt, Kt)
    assert torch.equal(k2, kstar)
    same_lists(c2, i2)
    assert torch.equal(pa.prefill(tcfg, Qt, Kt, Vt, c2, i2).transpose(0, 1), full)
    world = 2 + case % 3
    O = torch.zeros_like(full)
    for rank in range(world):
        rows = shard.zigzag_rows(cfg.M, world, rank, shard.row_align(cfg))
        wss = [pa.alloc_workspace(cfg, DEV), pa.alloc_workspace(cfg, DEV)]
        out = (kstar.clone(), budget.clone(), torch.zeros_like(cnt), torch.zeros_like(idx))
        shard.estimate_rows(cfg, Qd, Kd, rows, out=out, kstar_given=True, scores_only=True,
                            streams=[torch.cuda.Stream(), torch.cuda.Stream()], workspaces=wss)
        torch.cuda.synchronize()
        shard.select_rows(cfg, rows, wss, out[0], (out[2], out[3]))
        torch.cuda.synchronize()
        same_lists(out[2], out[3], [m for b0, e0 in rows for m in range(b0, e0)])
        shard.prefill_rows(cfg, Qd, Kd, Vd, out[2], out[3], O, rows)
    assert torch.equal(O, full)


@pytest.mark.parametrize("case", range(16))
def test_random_varlen_and_host_path_bitwise(case):
    # random packed batches (1-6 sequences, lengths 0-3000 tokens, empty ones included) through
    # proxyattn_forward_varlen == one estimate + prefill per sequence, bit for bit; and the
    # pipelined host path (PROXYATTN_HOST_CHUNKS default) == the device-resident call
    import torch
    rng = np.random.default_rng(9000 + case)
    c = draw(case)
    Hq, Hkv, d, b = c["Hq"], c["Hkv"], c["d"], c["b"]
    lens = [int(x) if rng.random() > 0.15 else 0 for x in rng.integers(1, 3000, int(rng.integers(1, 7)))]
    cu = np.concatenate([[0], np.cumsum(lens)]).tolist()
    if cu[-1] == 0:
        lens[0], cu = 777, [0] + [777] * len(lens)
    seqs = {i: workloads.structured(Hq, Hkv, n, d, seed=200 + case * 8 + i, device=DEV)
            for i, n in enumerate(lens) if n}
    packed = [torch.cat([seqs[i][j].transpose(0, 1) for i in sorted(seqs)], 0).contiguous() for j in range(3)]
    vcfg = pa.Config(Hq, Hkv, d, 1, b, c["s"], c["g"], c["gamma"], c["min_budget"], token_major=True)
    O, kstar = pa.forward_varlen(vcfg, cu, *packed)
    for i, (Q, K, V, _) in seqs.items():
        cfg = pa.Config(Hq, Hkv, d, lens[i], b, c["s"], c["g"], c["gamma"], c["min_budget"])
        k1, _, cnt, idx = pa.estimate(cfg, Q, K)
        O1 = pa.prefill(cfg, Q, K, V, cnt, idx)
        assert torch.equal(kstar[i], k1), i
        assert torch.equal(O[cu[i]:cu[i + 1]], O1.transpose(0, 1)), i
        if i == max(seqs, key=lambda j: lens[j]):          # host path on the longest sequence
            Qh, Kh, Vh = (t.cpu().pin_memory() for t in (Q, K, V))
            Oh = torch.empty_like(Qh).pin_memory()
            ks = torch.empty(Hq, dtype=torch.int32).pin_memory()
            ws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=DEV)
            pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws, ks)
            torch.cuda.synchronize()
            assert torch.equal(ks, k1.cpu()) and torch.equal(Oh, O1.cpu())


@pytest.mark.parametrize("case", range(24))
def test_random_config_method_variants(case):
    # the method variants (designated proxy head, static K*, constant-K reading
    # of Eq. 3, forced sink block), alone and combined, on the random bf16 configurations
    rng = np.random.default_rng(7000 + case)
    c = draw(case + 100)
    M = -(-c["N"] // c["b"])
    v = dict(designated_head=bool(rng.integers(0, 2)), constant_k=bool(rng.integers(0, 2)),
             force_sink=bool(rng.integers(0, 2)))
    if rng.random() < 0.3:
        v["static_kstar"] = int(rng.integers(1, M + 1))
    cfg = pa.Config(c["Hq"], c["Hkv"], c["d"], c["N"], c["b"], c["s"], c["g"], c["gamma"], c["min_budget"], **v)
    Q, K, V, _ = workloads.structured(c["Hq"], c["Hkv"], c["N"], c["d"], seed=300 + case)
    cnt, idx = run_staged(cfg, Q, K, V, min_checked=0.75)
    if cfg.force_sink:
        c_np, i_np = cnt.cpu().numpy(), idx.cpu().numpy()
        assert np.all(i_np[:, 1:, 0][c_np[:, 1:] >= 2] == 0)
