"""Union statistics of the attention work items at the bench config: per (head, row pair)
the union of the two ascending block lists vs the sum of their lengths."""
import numpy as np
import torch

import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E402
import paper_2509_24745_b200 as pa
import workloads

dev = torch.device("cuda:0")
N = 131072
cfg = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
cnt = cnt.cpu().numpy()
idx = idx.cpu().numpy()
M = cfg.M
tot = uni = 0
per_head = []
for h in range(32):
    th = uh = 0
    for m in range(M - 1, 0, -2):
        a = set(idx[h, m, :cnt[h, m]].tolist())
        b = set(idx[h, m - 1, :cnt[h, m - 1]].tolist())
        th += len(a) + len(b)
        uh += len(a | b)
    tot += th
    uni += uh
    per_head.append((int(kstar[h]), th, uh))
print("kstar:", sorted(kstar.cpu().numpy().tolist()))
print(f"sum cnt {tot}, union iterations {uni}, ideal {tot / 2:.0f}, union/ideal {uni / (tot / 2):.3f}")
for k, th, uh in sorted(per_head, key=lambda x: -x[1])[:8]:
    print(f"  kstar {k:4d}: blocks {th}, union {uh}, ratio {uh / (th / 2):.3f}")

# head pairs within each kv head (r = 4): adjacent vs sorted by kstar (nested lists: union = larger)
ks = kstar.cpu().numpy()
def pair_cost(pairs):
    tot = uni = 0
    for (a, b) in pairs:
        for m in range(M):
            la = set(idx[a, m, :cnt[a, m]].tolist()); lb = set(idx[b, m, :cnt[b, m]].tolist())
            tot += len(la) + len(lb); uni += len(la | lb)
    return uni / (tot / 2)
adj = [(4 * k + 2 * i, 4 * k + 2 * i + 1) for k in range(8) for i in range(2)]
srt = []
for k in range(8):
    hs = sorted(range(4 * k, 4 * k + 4), key=lambda h: -ks[h])
    srt += [(hs[0], hs[1]), (hs[2], hs[3])]
print("head pairs adjacent: union/ideal", round(pair_cost(adj), 3))
print("head pairs sorted by kstar within kv head: union/ideal", round(pair_cost(srt), 3))
print("kstar by kv head:", [sorted(ks[4 * k:4 * k + 4].tolist()) for k in range(8)])
