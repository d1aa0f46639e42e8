"""Multi-GPU orchestration of one ProxyAttn layer: query heads sharded by KV-head group
(SURVEY.md §8(e)), one process per GPU, torch.distributed (NCCL) for the plumbing.

* Each rank holds a contiguous, KV-aligned shard of query heads [b, e) and the KV heads
  they use; everything after pooling (budgets, selection, attention) is per head and local.
* When every proxy group touched by a shard lies inside it (g >= #ranks, e.g. Qwen g=4 on
  <= 4 GPUs) there is NO cross-GPU traffic.
* When a proxy group spans ranks (Llama g=1), Eq. 2's pooled sums are the one exchange
  step: fp32 partial sums of the local heads are all-reduced (sum), then each rank rounds
  them and computes the group's block scores itself (replicated, ~0.3 ms at 128K).
* all_gather of O is for verification only (not part of the timed step).
* Balanced alternative: zig-zag query-block-row sharding.  Every rank holds
  the whole layer and computes, for all heads, the block lists (estimate_rows: proxies,
  scores and selection of its rows only; Alg. 1 replicated) and the attention of two row
  chunks p and 2P-1-p; since K_{h,m} grows ~linearly in m for every head (reading Z12), the
  pair sums to the same work on every rank regardless of how budgets differ between heads,
  with no cross-GPU traffic at all.  Alg. 1 (per head, needed by every rank) is either
  replicated or sharded by heads with an all-gather of the Hq K* values (budgets_sharded).

The ops are the C-ABI calls of paper_2509_24745_b200 by default; tests inject other ops
with the same signatures to check the orchestration on CPU with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch


def head_shard(n_q_heads: int, n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of query heads aligned to KV heads, as balanced as KV heads allow."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if n_kv_heads % world:
        raise ValueError(f"{n_kv_heads} kv heads cannot be split evenly over {world} ranks")
    r = n_q_heads // n_kv_heads
    per_kv = n_kv_heads // world
    return rank * per_kv * r, (rank + 1) * per_kv * r


def shard_config(cfg, world: int, rank: int):
    if world == 1:
        return cfg.replace(q_head_begin=0, q_head_end=0)
    b, e = head_shard(cfg.n_q_heads, cfg.n_kv_heads, world, rank)
    return cfg.replace(q_head_begin=b, q_head_end=e)


def group_spans_ranks(cfg, world: int) -> bool:
    """True when a proxy group (Hq/g query heads) is split across ranks."""
    if world == 1:
        return False
    b, e = head_shard(cfg.n_q_heads, cfg.n_kv_heads, world, 0)
    return (e - b) % (cfg.n_q_heads // cfg.n_groups) != 0


@dataclass
class Ops:
    """The hot-path calls (C-ABI by default); signatures follow paper_2509_24745_b200."""

    estimate: Callable
    pool: Callable
    proxy_scores: Callable
    budgets: Callable
    select: Callable


def default_ops() -> Ops:
    from . import _lib

    return Ops(_lib.estimate, _lib.pool, _lib.proxy_scores, _lib.budgets, _lib.select)


def estimate_sharded(cfg, Q_local, K_local, world: int, workspace=None, ops: Optional[Ops] = None,
                     all_reduce: Optional[Callable] = None, out=None):
    """A1-A6 for the local shard `cfg` (q_head_begin/end set).  Returns
    (kstar, budget, block_cnt, block_idx) for the local heads."""
    ops = ops or default_ops()
    if not group_spans_ranks(cfg, world):
        return ops.estimate(cfg, Q_local, K_local, workspace, out)
    if all_reduce is None:
        import torch.distributed as dist

        all_reduce = dist.all_reduce
    qsum, ksum = ops.pool(cfg, Q_local, K_local)          # fp32 partial sums, local heads
    all_reduce(qsum)                                      # the single exchange
    all_reduce(ksum)
    L = ops.proxy_scores(cfg, qsum, ksum, workspace)      # replicated per rank
    kstar, budget = ops.budgets(cfg, Q_local, K_local, workspace)
    cnt, idx = ops.select(cfg, L, kstar)
    if out is not None:
        for dst, src in zip(out, (kstar, budget, cnt, idx)):
            dst.copy_(src)
        return out
    return kstar, budget, cnt, idx


def forward_host_sharded(cfg_local, Qh, Kh, Vh, Oh, world: int, workspace=None, all_reduce=None):
    """One ProxyAttn layer for this rank's KV-aligned head shard, end to end from pinned HOST
    buffers (the e2e leg at N > 1): H2D of its query heads and their KV heads, A1-A6 with the
    pooled sums all-reduced when a proxy group spans ranks, A7 on the local
    heads, D2H of O into Oh.  Synchronises the current stream; returns the local K* (host)."""
    from . import _lib

    dev = torch.device("cuda", torch.cuda.current_device())
    Q = Qh.to(dev, non_blocking=True)
    K = Kh.to(dev, non_blocking=True)
    V = Vh.to(dev, non_blocking=True)
    kstar, _, cnt, idx = estimate_sharded(cfg_local, Q, K, world, workspace, all_reduce=all_reduce)
    O = _lib.prefill(cfg_local, Q, K, V, cnt, idx)
    Oh.copy_(O, non_blocking=True)
    ks = kstar.to("cpu", non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return ks


def gather_heads(t_local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """all_gather of a head-major local tensor into the full head dimension (verification)."""
    import torch.distributed as dist

    parts = [torch.empty_like(t_local) for _ in range(world)]
    dist.all_gather(parts, t_local.contiguous(), group=group)
    return torch.cat(parts, dim=0)


def work_share(block_cnt_full: torch.Tensor, n_kv_heads: int, world: int) -> list[float]:
    """Executed (head, row, block) units per rank under head sharding, as fractions."""
    H = block_cnt_full.shape[0]
    tot = float(block_cnt_full.sum())
    out = []
    for r in range(world):
        b, e = head_shard(H, n_kv_heads, world, r)
        out.append(float(block_cnt_full[b:e].sum()) / tot)
    return out


def row_align(cfg) -> int:
    """Block rows per attention work unit: 2 — the attention kernels work on block-row pairs
    (2q, 2q+1) of one head: at b = 64 packed into one 128-lane tile, at d = b = 128 sharing
    their K/V tiles (attn_tc9).  Row ranges aligned to it give outputs bit-identical to the
    unsharded launch (an unaligned edge splits a pair: within tolerance, not bitwise)."""
    return 2


def zigzag_rows(M: int, world: int, rank: int, align: int = 1) -> list[tuple[int, int]]:
    """Block-row ranges of `rank` under zig-zag sharding: chunks p and 2P-1-p of 2P
    near-equal chunks of [0, M) (empty ranges dropped), with inner edges on multiples of
    `align` rows."""
    if world < 1 or not (0 <= rank < world) or align < 1:
        raise ValueError("bad world/rank/align")
    Mu = (M + align - 1) // align
    edges = [min(M, align * ((Mu * k) // (2 * world))) for k in range(2 * world + 1)]
    out = []
    for c in (rank, 2 * world - 1 - rank):
        b, e = edges[c], edges[c + 1]
        if e > b:
            out.append((b, e))
    return sorted(out)


def estimate_rows(cfg, Q, K, ranges, workspace=None, out=None, estimate=None, kstar_given=False,
                  streams=None, workspaces=None, scores_only=False):
    """A1-A6 for the block-row ranges only (zig-zag row sharding): the first call computes
    Alg. 1's kstar for every head, the others reuse it (KSTAR_GIVEN); with kstar_given the
    caller has filled out[0] already (budgets_sharded) and every call reuses it.  Block lists
    are written for the rows of the ranges only.  Returns (kstar, budget, block_cnt, block_idx).

    With kstar_given, `streams` and one workspace per range, the ranges' estimates run
    concurrently (each is a short chain of small, latency-bound kernels; they write disjoint
    rows of the outputs), forked from and joined back to the current stream.  With
    scores_only (K* given, one workspace per range; a single range runs on the current
    stream) the calls stop before the selection (select_rows finishes from each range's
    workspace), so the K* exchange can overlap the score passes."""
    if estimate is None:
        from . import _lib

        estimate = _lib.estimate
    if scores_only:   # each range's L must survive in its own workspace until select_rows
        assert kstar_given and out is not None and workspaces and len(workspaces) >= len(ranges), \
            "scores_only needs kstar_given, out and one workspace per range"
    if kstar_given and streams and workspaces and len(ranges) > 1 and out is not None:
        cur = torch.cuda.current_stream()
        used = []
        for k, (b, e) in enumerate(ranges):
            s = streams[k % len(streams)]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                estimate(cfg.replace(row_begin=b, row_end=e, kstar_given=True, scores_only=scores_only), Q, K,
                         workspaces[k % len(workspaces)], out)
            used.append(s)
        for s in used:
            cur.wait_stream(s)
        return out
    for k, (b, e) in enumerate(ranges):
        ws = workspaces[k % len(workspaces)] if workspaces else workspace
        out = estimate(cfg.replace(row_begin=b, row_end=e, kstar_given=kstar_given or k > 0,
                                   scores_only=scores_only), Q, K, ws, out)
    return out


def select_rows(cfg, ranges, workspaces, kstar, out, select_ws=None):
    """A5-A6 of each row range from the L its scores_only estimate left in its workspace."""
    if select_ws is None:
        from . import _lib

        select_ws = _lib.select_ws
    for k, (b, e) in enumerate(ranges):
        select_ws(cfg.replace(row_begin=b, row_end=e), workspaces[k % len(workspaces)], kstar, out)
    return out


def budgets_sharded(cfg, Q, K, world: int, rank: int, workspace=None, budgets=None,
                    all_gather=None, out=None):
    """Alg. 1 (A4) sharded by KV-aligned head ranges under zig-zag row sharding: rank p runs
    it for its heads only and the per-head K* (Hq int32, 4 B each) are all-gathered, so the
    per-rank estimate no longer repeats Alg. 1 for every head (~0.3 ms at 128K).  K* of a
    head depends on that head's Q and K only, so the gathered vector equals the
    replicated one bit for bit.  Q/K are the full head-major tensors.  Returns (kstar, budget)
    for all heads; falls back to the replicated call when the KV heads do not split evenly."""
    if budgets is None:
        from . import _lib

        budgets = _lib.budgets
    Hq, Hkv = cfg.n_q_heads, cfg.n_kv_heads
    if world == 1 or Hkv % world:
        ks, bu = budgets(cfg, Q, K, workspace)
        if out is None:
            return ks, bu
        out[0].copy_(ks)
        out[1].copy_(bu)
        return out[0], out[1]
    if all_gather is None:
        import torch.distributed as dist

        all_gather = dist.all_gather_into_tensor
    b, e = head_shard(Hq, Hkv, world, rank)
    r = Hq // Hkv
    loc = cfg.replace(q_head_begin=b, q_head_end=e, row_begin=0, row_end=0)
    ks_loc, bu_loc = budgets(loc, Q[b:e], K[b // r:e // r], workspace)
    kstar = out[0] if out is not None else torch.empty(Hq, dtype=torch.int32, device=ks_loc.device)
    budget = out[1] if out is not None else torch.empty(Hq, dtype=torch.float32, device=ks_loc.device)
    all_gather(kstar, ks_loc.contiguous())                 # K*_h and b_h = K*_h / M, both as
    all_gather(budget, bu_loc.contiguous())                # the library computed them
    return kstar, budget


def prefill_rows(cfg, Q, K, V, block_cnt, block_idx, O, ranges, prefill=None):
    """Attention for the given block-row ranges only (other rows of O untouched)."""
    if prefill is None:
        from . import _lib

        prefill = _lib.prefill
    for b, e in ranges:
        prefill(cfg.replace(row_begin=b, row_end=e), Q, K, V, block_cnt, block_idx, O)
    return O


def row_work_share(block_cnt_full: torch.Tensor, world: int, align: int = 1) -> list[float]:
    """Executed (head, row, block) units per rank under zig-zag row sharding, as fractions."""
    per_row = block_cnt_full.double().sum(dim=0)
    tot = float(per_row.sum())
    M = per_row.numel()
    return [sum(float(per_row[b:e].sum()) for b, e in zigzag_rows(M, world, r, align)) / tot
            for r in range(world)]


def estimate_rows_overlapped(cfg, Q, K, ranges, world: int, rank: int, workspaces, out, alg1_workspace=None,
                             aux_stream=None, streams=None, estimate=None, select_ws=None, budgets=None,
                             all_gather=None, run_scores=None, run_select=None):
    """The row-sharded estimate with its one collective overlapped (bench.py's step at N > 1):
    the score passes (A1-A3, SCORES_ONLY, K* not needed yet) of the rank's row ranges run on
    `aux_stream` while the current stream runs the head-sharded Alg. 1 and the K* / budget
    all-gather (budgets_sharded); the selection (A5-A6, select_rows) follows both.  `out` =
    (kstar, budget, block_cnt, block_idx) for all heads; only the ranges' rows are written.
    run_scores / run_select replace the two phases (bench.py passes CUDA-graph replays).
    Without a CUDA stream (aux_stream None: CPU tests with injected ops) the phases run in
    program order."""
    kstar, budget, cnt, idx = out
    if run_scores is None:
        def run_scores():
            estimate_rows(cfg, Q, K, ranges, out=out, estimate=estimate, kstar_given=True, streams=streams,
                          workspaces=workspaces, scores_only=True)
    if run_select is None:
        def run_select():
            select_rows(cfg, ranges, workspaces, kstar, (cnt, idx), select_ws=select_ws)
    if aux_stream is None:
        run_scores()
        budgets_sharded(cfg, Q, K, world, rank, alg1_workspace, budgets=budgets, all_gather=all_gather,
                        out=(kstar, budget))
        run_select()
        return out
    cur = torch.cuda.current_stream()
    aux_stream.wait_stream(cur)
    with torch.cuda.stream(aux_stream):
        run_scores()
    budgets_sharded(cfg, Q, K, world, rank, alg1_workspace, budgets=budgets, all_gather=all_gather,
                    out=(kstar, budget))
    cur.wait_stream(aux_stream)
    run_select()
    return out
