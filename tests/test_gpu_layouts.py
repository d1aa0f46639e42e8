"""GPU: token-major ([N][heads][d], token strides) and packed variable-length inputs
(SURVEY §8(f) rank 1).  The layout changes only addressing (3-D TMA maps, strided SIMT
loads), never arithmetic, so every output must be BIT-identical to the head-major run on
the same values; the varlen path must equal one single-sequence call per sequence, and
one sequence is also checked against the fp64 oracle end to end."""
import numpy as np
import pytest
import torch

import oracle
import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


def tok(t):                       # [H][N][d] -> contiguous [N][H][d]
    return t.transpose(0, 1).contiguous()


def run(cfg, Q, K, V):
    est = pa.estimate(cfg, Q, K)
    O = pa.prefill(cfg, Q, K, V, est[2], est[3])
    Od = pa.dense_prefill(cfg, Q, K, V)
    return est, O, Od


@pytest.mark.parametrize("N,heads,g,seed", [(2048, (8, 2), 1, 0), (2000, (8, 2), 2, 1),
                                            (3001, (7, 1), 1, 2)])
def test_token_major_bitwise_equals_head_major(N, heads, g, seed):
    Hq, Hkv = heads
    cfg = pa.Config(Hq, Hkv, 128, N, 128, 4, g, 0.9)
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, 128, seed=seed, device=DEV)
    (k0, b0, c0, i0), O0, Od0 = run(cfg, Q, K, V)
    tcfg = cfg.replace(token_major=True)
    (k1, b1, c1, i1), O1, Od1 = run(tcfg, tok(Q), tok(K), tok(V))
    assert torch.equal(k0, k1) and torch.equal(b0, b1) and torch.equal(c0, c1)
    for h in range(Hq):
        for m in range(cfg.M):
            c = int(c0[h, m])
            assert torch.equal(i0[h, m, :c], i1[h, m, :c])
    # the default sparse kernel reads both layouts; dense head-major runs attn_tc, so the
    # dense comparison is against the oracle tolerance instead of bitwise
    assert torch.equal(O0, O1.transpose(0, 1))
    assert (Od0.float() - Od1.transpose(0, 1).float()).abs().max().item() <= 2e-2


def test_token_major_head_slices_of_a_packed_activation():
    # a rank's shard = a head slice of the packed [N][H][d] activation: token stride H*d
    N, Hq, Hkv = 2048, 8, 2
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, 128, seed=5, device=DEV)
    Qp, Kp, Vp = tok(Q), tok(K), tok(V)
    full = pa.Config(Hq, Hkv, 128, N, 128, 4, 2, 0.9)
    shard = full.replace(q_head_begin=4, q_head_end=8)         # kv head 1, group 1 (g=2)
    (k0, _, c0, i0), O0, _ = run(shard, Q[4:].contiguous(), K[1:].contiguous(), V[1:].contiguous())
    Qs, Ks, Vs = Qp[:, 4:], Kp[:, 1:], Vp[:, 1:]
    scfg = pa.with_strides(shard, Qs, Ks)
    assert scfg.q_token_stride == Hq * 128 and scfg.kv_token_stride == Hkv * 128
    k1, _, c1, i1 = pa.estimate(scfg, Qs, Ks)
    O1 = pa.prefill(scfg, Qs, Ks, Vs, c1, i1)
    assert O1.stride(0) == Hq * 128
    assert torch.equal(k0, k1) and torch.equal(c0, c1)
    assert torch.equal(O0, O1.transpose(0, 1))


def test_token_major_fp32_debug_bitwise():
    cfg = pa.Config(8, 2, 64, 1024, 64, 4, 2, 0.9, fp32_debug=True)
    Q, K, V = workloads.iid(8, 2, 1024, 64, seed=3)
    Q, K, V = [t.to(DEV) for t in (Q, K, V)]
    (k0, _, c0, _), O0, Od0 = run(cfg, Q, K, V)
    (k1, _, c1, _), O1, Od1 = run(cfg.replace(token_major=True), tok(Q), tok(K), tok(V))
    assert torch.equal(k0, k1) and torch.equal(c0, c1)
    assert torch.equal(O0, O1.transpose(0, 1)) and torch.equal(Od0, Od1.transpose(0, 1))


def test_varlen_equals_one_call_per_sequence_and_the_oracle():
    Hq, Hkv, lens = 8, 2, [1000, 2048, 0, 640]
    seqs = [workloads.structured(Hq, Hkv, n, 128, seed=10 + i, device=DEV) if n else None
            for i, n in enumerate(lens)]
    cu = np.concatenate([[0], np.cumsum(lens)]).tolist()
    packed = [torch.cat([tok(s[j]) for s in seqs if s is not None], 0) for j in range(3)]
    cfg = pa.Config(Hq, Hkv, 128, 1, 128, 4, 1, 0.9, token_major=True)
    O, kstar = pa.forward_varlen(cfg, cu, *packed)
    assert kstar.shape == (len(lens), Hq)
    lists = {}
    for i, n in enumerate(lens):
        if n == 0:
            continue
        Q, K, V, _ = seqs[i]
        c1 = pa.Config(Hq, Hkv, 128, n, 128, 4, 1, 0.9)
        k1, _, cnt, idx = pa.estimate(c1, Q, K)
        O1 = pa.prefill(c1, Q, K, V, cnt, idx)
        lists[i] = (cnt, idx)
        assert torch.equal(kstar[i], k1)
        assert torch.equal(O[cu[i]:cu[i + 1]], tok(O1))
    # against the oracle on the shortest sequence (its own layer): budgets where their
    # margin is clear, and O with the GPU's lists injected (the staged protocol)
    Q, K, V, _ = seqs[3]
    oc = oracle.Cfg(Hq, Hkv, 128, 640, 128, 4, 1, 0.9, round_bf16=True)
    Qf, Kf, Vf = (t.float().cpu().numpy() for t in (Q, K, V))
    ks_ref, _, bmg, _ = oracle.budgets(oc, Qf, Kf)
    ok = bmg > 1e-4
    assert np.array_equal(kstar[3].cpu().numpy()[ok], ks_ref[ok])
    cnt, idx = lists[3]
    ref = oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy())
    err = np.abs(O[cu[3]:cu[4]].transpose(0, 1).float().cpu().numpy() - ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
