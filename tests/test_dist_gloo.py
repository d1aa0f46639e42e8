"""World-size-2 CPU tests (gloo) of the multi-GPU orchestration (paper_2509_24745_b200.shard):
head sharding aligned to KV heads, the all-reduce of Eq. 2's pooled partial sums when a
proxy group spans ranks, and local budgets/selection.  The CUDA ops are
replaced by fp64 oracle ops with the same signatures, so the sharded pipeline must
reproduce the unsharded oracle EXACTLY (the decomposition is exact: sums of bf16 values,
per-head Alg. 1 and Eq. 3)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import workloads
from paper_2509_24745_b200 import Config, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def local_ocfg(cfg: Config) -> oracle.Cfg:
    """Oracle config of the shard's sub-problem (local heads, local groups)."""
    b, e = cfg.local_heads
    Hl = e - b
    r = cfg.r
    gq = cfg.n_q_heads // cfg.n_groups
    gl = max(1, Hl // gq)
    return oracle.Cfg(Hl, Hl // r, cfg.head_dim, cfg.seq_len, cfg.block_size, cfg.stride, gl,
                      cfg.gamma, cfg.min_budget_tokens, round_bf16=True)


def oracle_ops() -> shard.Ops:
    def pool(cfg, Q, K):
        oc = local_ocfg(cfg).replace(round_bf16=False)
        Pq, Pk, _ = oracle.pool(oc, Q.numpy(), K.numpy())
        return torch.from_numpy(Pq), torch.from_numpy(Pk)

    def proxy_scores(cfg, qsum, ksum, ws=None):
        oc = local_ocfg(cfg)
        rne = np.vectorize(oracle.rne_bf16)
        gq, gk = cfg.n_q_heads // cfg.n_groups, cfg.n_kv_heads // cfg.n_groups
        scale = 1.0 / (gq * gk * np.sqrt(cfg.head_dim))       # the GLOBAL group sizes
        _, L = oracle.proxy_scores(oc, rne(qsum.numpy()), rne(ksum.numpy()), scale)
        return torch.from_numpy(L)

    def budgets(cfg, Q, K, ws=None):
        ks, b, _, _ = oracle.budgets(local_ocfg(cfg), Q.numpy(), K.numpy())
        return torch.from_numpy(ks), torch.from_numpy(b)

    def select(cfg, L, kstar):
        cnt, idx, _ = oracle.select(local_ocfg(cfg), L.numpy(), kstar.numpy())
        return torch.from_numpy(cnt), torch.from_numpy(idx)

    def estimate(cfg, Q, K, ws=None, out=None):
        est = oracle.estimate(local_ocfg(cfg), Q.numpy(), K.numpy())
        return (torch.from_numpy(est["kstar"]), torch.from_numpy(est["budget"]),
                torch.from_numpy(est["block_cnt"]), torch.from_numpy(est["block_idx"]))

    return shard.Ops(estimate, pool, proxy_scores, budgets, select)


def _worker(rank, world, port, cfg_kw, seed, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = Config(**cfg_kw)
        Q, K, _, _ = workloads.structured(cfg.n_q_heads, cfg.n_kv_heads, cfg.seq_len,
                                          cfg.head_dim, seed=seed, dtype=torch.bfloat16)
        Q, K = Q.float(), K.float()
        lcfg = shard.shard_config(cfg, world, rank)
        b, e = lcfg.local_heads
        r = cfg.r
        calls = []

        def all_reduce(t):
            calls.append(t.shape)
            dist.all_reduce(t)

        kstar, budget, cnt, idx = shard.estimate_sharded(
            lcfg, Q[b:e].contiguous(), K[b // r:e // r].contiguous(), world, ops=oracle_ops(),
            all_reduce=all_reduce)
        full = [shard.gather_heads(t.contiguous(), world) for t in (kstar, cnt, idx)]
        if rank == 0:
            q.put((len(calls), [f.numpy() for f in full]))
    finally:
        dist.destroy_process_group()


def run_sharded(cfg_kw, seed, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_kw, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


CASES = [
    # Llama-like g = 1: the proxy group spans both ranks -> one all-reduce of (qsum, ksum)
    dict(cfg=dict(n_q_heads=8, n_kv_heads=4, head_dim=32, seq_len=1024, block_size=64,
                  stride=4, n_groups=1, gamma=0.9), n_allreduce=2),
    # Qwen-like g = Hkv: groups inside shards -> no cross-rank traffic
    dict(cfg=dict(n_q_heads=8, n_kv_heads=4, head_dim=32, seq_len=1024, block_size=64,
                  stride=4, n_groups=4, gamma=0.9, min_budget_tokens=128), n_allreduce=0),
    # g = #ranks: exactly one group per rank
    dict(cfg=dict(n_q_heads=8, n_kv_heads=4, head_dim=32, seq_len=512, block_size=64,
                  stride=2, n_groups=2, gamma=0.7), n_allreduce=0),
]


@pytest.mark.parametrize("case", CASES, ids=["g1-allreduce", "g4-local", "g2-local"])
def test_sharded_estimate_equals_unsharded_oracle(case):
    cfg_kw = case["cfg"]
    n_calls, (kstar, cnt, idx) = run_sharded(cfg_kw, seed=3)
    assert n_calls == case["n_allreduce"]
    cfg = Config(**cfg_kw)
    oc = oracle.Cfg(cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim, cfg.seq_len, cfg.block_size,
                    cfg.stride, cfg.n_groups, cfg.gamma, cfg.min_budget_tokens, round_bf16=True)
    Q, K, _, _ = workloads.structured(cfg.n_q_heads, cfg.n_kv_heads, cfg.seq_len, cfg.head_dim,
                                      seed=3, dtype=torch.bfloat16)
    ref = oracle.estimate(oc, Q.float().numpy(), K.float().numpy())
    assert np.array_equal(kstar, ref["kstar"])
    assert np.array_equal(cnt, ref["block_cnt"])
    for h in range(cfg.n_q_heads):
        for m in range(cfg.M):
            c = cnt[h, m]
            assert np.array_equal(idx[h, m, :c], ref["block_idx"][h, m, :c])


def test_head_shard_arithmetic():
    assert shard.head_shard(32, 8, 8, 3) == (12, 16)
    assert shard.head_shard(28, 4, 4, 1) == (7, 14)
    assert shard.head_shard(28, 4, 2, 1) == (14, 28)
    with pytest.raises(ValueError):
        shard.head_shard(28, 4, 8, 0)
    llama = Config(32, 8, 128, 4096)
    assert shard.group_spans_ranks(llama, 2) and not shard.group_spans_ranks(llama, 1)
    qwen = Config(28, 4, 128, 4096, n_groups=4)
    assert not shard.group_spans_ranks(qwen, 4) and not shard.group_spans_ranks(qwen, 2)
    lc = shard.shard_config(llama, 8, 7)
    assert lc.local_heads == (28, 32) and lc.Hl == 4


def test_work_share_sums_to_one():
    cnt = torch.randint(1, 10, (32, 16))
    s = shard.work_share(cnt, 8, 4)
    assert len(s) == 4 and abs(sum(s) - 1) < 1e-12


# ----------------------------------------------------------- zig-zag row sharding --
def test_zigzag_rows_cover_exactly_once_and_balance_linear_rows():
    for align in (1, 2):                 # 2: block size 64 (the kernel's row pairs)
        for M in (16, 1000, 1024, 2048, 7, 2047):
            for P in (1, 2, 4, 8):
                if 2 * P * align > M:
                    continue
                seen = np.zeros(M, int)
                loads = []
                for r in range(P):
                    rr = shard.zigzag_rows(M, P, r, align)
                    assert len(rr) <= 2
                    load = 0
                    for b, e in rr:
                        assert b % align == 0 and (e % align == 0 or e == M)
                        seen[b:e] += 1
                        load += sum(m + 1 for m in range(b, e))       # K_{h,m} ~ (m+1) (Z12)
                    loads.append(load)
                assert np.all(seen == 1)
                if M >= 64:
                    assert max(loads) / (sum(loads) / P) < 1.01 + 0.01 * align, (M, P, align, loads)


def test_zigzag_balance_on_bimodal_budgets_vs_head_sharding():
    # bimodal per-head budgets (the calibrated generator's, recorded in scripts/union_stats.py)
    ks = [3, 5, 84, 340, 3, 3, 121, 143, 3, 3, 3, 4, 3, 3, 178, 208,
          3, 244, 468, 634, 3, 80, 91, 665, 3, 159, 514, 615, 3, 3, 5, 638]
    M = 1024
    m = np.arange(M)
    cnt = torch.tensor(np.minimum(m + 1, np.maximum(-(-np.outer(ks, m + 1) // M), 1)))
    rows = shard.row_work_share(cnt, 8)
    heads = shard.work_share(cnt, 8, 8)
    assert max(rows) * 8 < 1.02          # zig-zag: balanced
    assert max(heads) * 8 > 1.8          # head sharding: the densest kv head dominates


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oc = oracle.Cfg(4, 2, 16, 1024, 64, 4, 1, 0.9, round_bf16=True)
        Q, K, V, _ = workloads.structured(4, 2, 1024, 16, seed=5, dtype=torch.bfloat16)
        Qf, Kf, Vf = Q.float().numpy(), K.float().numpy(), V.float().numpy()
        est = oracle.estimate(oc, Qf, Kf)                    # replicated estimate
        O = torch.zeros(4, 1024, 16, dtype=torch.float64)

        def prefill(cfg, Q_, K_, V_, cnt, idx, O_):          # oracle op, rows [b, e) only
            items = [(h, m) for h in range(4) for m in range(cfg.row_begin, cfg.row_end)]
            Oh = oracle.attention(oc, Qf, Kf, Vf, cnt, idx, items=items)
            for h, m in items:
                O_[h, m * 64:(m + 1) * 64] = torch.from_numpy(Oh[h, m * 64:(m + 1) * 64])

        cfg = Config(4, 2, 16, 1024, 64, 4, 1, 0.9)
        shard.prefill_rows(cfg, None, None, None, est["block_cnt"], est["block_idx"], O,
                           shard.zigzag_rows(oc.M, world, rank), prefill=prefill)
        dist.all_reduce(O)                                    # disjoint rows: sum == gather
        if rank == 0:
            q.put(O.numpy())
    finally:
        dist.destroy_process_group()


def test_zigzag_sharded_attention_equals_unsharded_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    O = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    oc = oracle.Cfg(4, 2, 16, 1024, 64, 4, 1, 0.9, round_bf16=True)
    Q, K, V, _ = workloads.structured(4, 2, 1024, 16, seed=5, dtype=torch.bfloat16)
    ref = oracle.pipeline(oc, Q.float().numpy(), K.float().numpy(), V.float().numpy())["O"]
    assert np.max(np.abs(O - ref)) == 0.0


# ----------------------------------------------- head-sharded Alg. 1 + K* all-gather --
def _alg1_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oc = oracle.Cfg(8, 4, 16, 1024, 64, 4, 1, 0.9, round_bf16=True)
        Q, K, V, _ = workloads.structured(8, 4, 1024, 16, seed=9, dtype=torch.bfloat16)
        Qf, Kf = Q.float().numpy(), K.float().numpy()
        calls = []

        def budgets(cfg, Q_, K_, workspace=None):          # oracle op on the shard's heads
            b, e = cfg.q_head_begin, cfg.q_head_end
            calls.append((b, e))
            assert Q_.shape[0] == e - b and K_.shape[0] == (e - b) // 2
            ks, bu, _, _ = oracle.budgets(oc, Qf, Kf, heads=list(range(b, e)))
            return (torch.tensor(ks[b:e], dtype=torch.int32), torch.tensor(bu[b:e], dtype=torch.float32))

        def all_gather(dst, src):
            parts = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(parts, src)
            dst.copy_(torch.cat(parts))

        cfg = Config(8, 4, 16, 1024, 64, 4, 1, 0.9)
        ks, bu = shard.budgets_sharded(cfg, Q, K, world, rank, budgets=budgets, all_gather=all_gather)
        assert len(calls) == 1 and calls[0] == shard.head_shard(8, 4, world, rank)
        if rank == 0:
            q.put((ks.numpy(), bu.numpy()))
    finally:
        dist.destroy_process_group()


def test_head_sharded_alg1_gathers_the_replicated_kstar():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_alg1_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ks, bu = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    oc = oracle.Cfg(8, 4, 16, 1024, 64, 4, 1, 0.9, round_bf16=True)
    Q, K, V, _ = workloads.structured(8, 4, 1024, 16, seed=9, dtype=torch.bfloat16)
    ref, _, _, _ = oracle.budgets(oc, Q.float().numpy(), K.float().numpy())
    assert np.array_equal(ks, ref)                           # every head, bit for bit
    assert np.allclose(bu, ref / oc.M)


# ---------------------- bench.py's N > 1 estimate: scores | Alg. 1 + all-gather | select --
def _overlap_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oc = oracle.Cfg(8, 4, 16, 2048, 64, 4, 1, 0.9, round_bf16=True)
        Q, K, V, _ = workloads.structured(8, 4, 2048, 16, seed=19, dtype=torch.bfloat16)
        Qf, Kf = Q.float().numpy(), K.float().numpy()
        M = oc.M
        phases = []

        def estimate(cfg, Q_, K_, ws, out):                # SCORES_ONLY: L of the rows -> ws
            assert cfg.scores_only and cfg.kstar_given
            phases.append(("scores", cfg.row_begin, cfg.row_end))
            rows = list(range(cfg.row_begin, cfg.row_end))
            Pq, Pk, sc = oracle.pool(oc, Qf, Kf)
            _, L = oracle.proxy_scores(oc, Pq, Pk, sc, rows=rows)
            ws["L"] = L
            return out

        def select_ws(cfg, ws, kstar, out):
            phases.append(("select", cfg.row_begin, cfg.row_end))
            rows = list(range(cfg.row_begin, cfg.row_end))
            cnt, idx, _ = oracle.select(oc, np.nan_to_num(ws["L"], nan=-np.inf), kstar.numpy(), rows=rows)
            out[0][:, rows] = torch.from_numpy(cnt[:, rows])
            out[1][:, rows] = torch.from_numpy(idx[:, rows])
            return out

        def budgets(cfg, Q_, K_, workspace=None):
            phases.append(("alg1", cfg.q_head_begin, cfg.q_head_end))
            b, e = cfg.q_head_begin, cfg.q_head_end
            ks, bu, _, _ = oracle.budgets(oc, Qf, Kf, heads=list(range(b, e)))
            return torch.tensor(ks[b:e], dtype=torch.int32), torch.tensor(bu[b:e], dtype=torch.float32)

        def all_gather(dst, src):
            phases.append(("all_gather",))
            parts = [torch.empty_like(src) for _ in range(world)]
            dist.all_gather(parts, src)
            dst.copy_(torch.cat(parts))

        cfg = Config(8, 4, 16, 2048, 64, 4, 1, 0.9)
        ranges = shard.zigzag_rows(M, world, rank, shard.row_align(cfg))
        out = (torch.zeros(8, dtype=torch.int32), torch.zeros(8), torch.zeros(8, M, dtype=torch.int32),
               torch.full((8, M, M), -1, dtype=torch.int32))
        wss = [dict() for _ in ranges]
        shard.estimate_rows_overlapped(cfg, Q, K, ranges, world, rank, wss, out, estimate=estimate,
                                       select_ws=select_ws, budgets=budgets, all_gather=all_gather)
        kinds = [p[0] for p in phases]
        # scores of every range precede the selection, which follows the K* exchange
        assert kinds.index("all_gather") < kinds.index("select")
        assert max(i for i, k in enumerate(kinds) if k == "scores") < kinds.index("select")
        q.put((rank, ranges, out[0].numpy(), out[1].numpy(), out[2].numpy(), out[3].numpy()))
    finally:
        dist.destroy_process_group()


def test_overlapped_row_sharded_estimate_equals_unsharded_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    oc = oracle.Cfg(8, 4, 16, 2048, 64, 4, 1, 0.9, round_bf16=True)
    Q, K, _, _ = workloads.structured(8, 4, 2048, 16, seed=19, dtype=torch.bfloat16)
    est = oracle.estimate(oc, Q.float().numpy(), K.float().numpy())
    covered = np.zeros(oc.M, bool)
    for rank, ranges, ks, bu, cnt, idx in res:
        assert np.array_equal(ks, est["kstar"]) and np.allclose(bu, est["kstar"] / oc.M)
        for b, e in ranges:
            assert not covered[b:e].any()
            covered[b:e] = True
            assert np.array_equal(cnt[:, b:e], est["block_cnt"][:, b:e])
            assert np.array_equal(idx[:, b:e], est["block_idx"][:, b:e])
    assert covered.all()
