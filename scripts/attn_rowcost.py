"""Per-row vs per-block cost of the sparse attention kernel: the bench's lists (bimodal
per-head budgets: many short rows) against static top-K lists with the same total blocks
(every row ~the same length), and dense.  Prints ms, blocks, ns per block, rows."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E402
import paper_2509_24745_b200 as pa
import workloads

N = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
dev = torch.device("cuda:0")
preset = {16384: "llama-16k", 32768: "llama-32k", 65536: "llama-64k"}.get(N, "llama-128k")
cfg = pa.Config(32, 8, d, N, b, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, d, seed=0, params=workloads.PRESETS[preset], device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, it=10):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(it):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


ks, _, cnt, idx = pa.estimate(cfg, Q, K)
O = torch.empty_like(Q)
tot = int(cnt.sum())
t = timed(lambda: pa.prefill(cfg, Q, K, V, cnt, idx, O))
out = {"N": N, "b": b, "d": d, "bench_lists": {"ms": t, "blocks": tot, "ns_per_block": t * 1e6 / tot,
                                               "kstar_min": int(ks.min()), "kstar_max": int(ks.max())}}
# static top-K with about the same total
M = cfg.M
lo, hi = 1, M
while lo < hi:
    mid = (lo + hi) // 2
    c2 = pa.estimate(cfg.replace(static_kstar=mid), Q, K)[2]
    if int(c2.sum()) < tot:
        lo = mid + 1
    else:
        hi = mid
cs = cfg.replace(static_kstar=lo)
_, _, c2, i2 = pa.estimate(cs, Q, K)
t2 = timed(lambda: pa.prefill(cfg, Q, K, V, c2, i2, O))
out["static_lists"] = {"kstar": lo, "ms": t2, "blocks": int(c2.sum()), "ns_per_block": t2 * 1e6 / int(c2.sum())}
t3 = timed(lambda: pa.dense_prefill(cfg, Q, K, V, O), it=3)
nd = 32 * M * (M + 1) // 2
out["dense"] = {"ms": t3, "blocks": nd, "ns_per_block": t3 * 1e6 / nd}
print(json.dumps(out))
