"""Bisection of the structured generator's beta scale for one attention shape so that the GPU
estimate's sparsity (gamma = 0.9, seed 0) matches a target, e.g. Table 8's Llama 128K
83.86 % for the head_dim-64 Llama-3.2-1B shape.  beta_hi = 3 beta_lo, sigma 0.93.

    python scripts/calibrate_shape.py Hq Hkv d N b target [lo hi]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E402
import paper_2509_24745_b200 as pa
import workloads

Hq, Hkv, d, N, b = (int(x) for x in sys.argv[1:6])
tgt = float(sys.argv[6])
a, bb = (float(sys.argv[7]), float(sys.argv[8])) if len(sys.argv) > 8 else (0.2, 3.0)
dev = torch.device("cuda:0")
cfg = pa.Config(Hq, Hkv, d, N, b, 4, 1, 0.9, 0)


def sp(lo):
    prm = workloads.StructParams(sigma=0.93, beta_lo=lo, beta_hi=3 * lo)
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=0, params=prm, device=dev)
    _, _, cnt, _ = pa.estimate(cfg, Q, K)
    M = cfg.M
    return float(1 - cnt.double().sum() / (Hq * M * (M + 1) / 2))


sa, sb = sp(a), sp(bb)
print(json.dumps({"lo": a, "sparsity": sa, "hi": bb, "sparsity_hi": sb}), flush=True)
best = None
for it in range(14):
    mid = 0.5 * (a + bb)
    sm = sp(mid)
    if best is None or abs(sm - tgt) < abs(best[1] - tgt):
        best = (mid, sm)
    if (sm - tgt) * (sa - tgt) > 0:
        a, sa = mid, sm
    else:
        bb, sb = mid, sm
print(json.dumps({"shape": [Hq, Hkv, d, N, b], "target": tgt, "beta_lo": round(best[0], 4),
                  "sparsity": round(best[1], 4)}), flush=True)
