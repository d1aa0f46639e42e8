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
