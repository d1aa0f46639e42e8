"""Union overhead of packing two 64-row work units into one 128-lane tile (block size 64),
on the bench inputs: (a) two heads of one KV head on the same block row, paired by count
(the kernel's plan), (b) two adjacent block rows (2p, 2p+1) of the same head.  Reports
sum(union) / (sum(cnt) / 2): 1.0 = no waste."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E402
import paper_2509_24745_b200 as pa
import workloads

N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
b = int(sys.argv[2]) if len(sys.argv) > 2 else 64
dev = torch.device("cuda:0")
cfg = pa.Config(32, 8, 128, N, b, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
_, _, cnt, idx = pa.estimate(cfg, Q, K)
M, H, r = cfg.M, 32, 4
ar = torch.arange(M, device=dev)
mask = torch.zeros(H, M, M, dtype=torch.bool, device=dev)
valid = ar[None, None, :] < cnt[:, :, None]
hh, mm, jj = torch.nonzero(valid, as_tuple=True)
mask[hh, mm, idx[hh, mm, jj].long()] = True
tot = float(cnt.double().sum())
# (a) head pairs by count per (kv, row)
ua = 0.0
for kv in range(8):
    c = cnt[kv * r:(kv + 1) * r].double()                      # [r, M]
    order = torch.argsort(-c, dim=0, stable=True)               # [r, M]
    for p in range(0, r, 2):
        ha = order[p] + kv * r
        hb = order[p + 1] + kv * r
        u = (mask[ha, ar] | mask[hb, ar]).sum()
        ua += float(u)
# (b) adjacent rows of one head
mb = mask[:, 0::2] | mask[:, 1::2] if M % 2 == 0 else None
ub = float(mb.sum())
print(json.dumps({"N": N, "b": b, "M": M, "sum_cnt": tot, "head_pairs_by_count": ua / (tot / 2),
                  "adjacent_rows": ub / (tot / 2)}))
