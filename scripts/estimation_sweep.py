"""Estimation latency (A1-A6) vs proxy groups g and stride s on the Llama-3.1-8B shape,
against the same-run dense attention (Fig. 6b: estimation < 10 % of full attention, P:614;
Table 5 stride cost side; cost model g/(n s^2)).  JSON lines."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # noqa: E402
import paper_2509_24745_b200 as pa
import workloads

dev = torch.device("cuda:0")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


base = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
dense = timed(lambda: pa.dense_prefill(base, Q, K, V), reps=3)
print(json.dumps({"N": N, "dense_ms": dense}), flush=True)
for g in (1, 2, 4, 8):
    for s in (1, 2, 4, 8):
        cfg = base.replace(n_groups=g, stride=s)
        ws = pa.alloc_workspace(cfg, dev)
        out = (torch.empty(32, dtype=torch.int32, device=dev), torch.empty(32, device=dev),
               torch.empty(32, cfg.M, dtype=torch.int32, device=dev),
               torch.empty(32, cfg.M, cfg.M, dtype=torch.int32, device=dev))
        ms = timed(lambda: pa.estimate(cfg, Q, K, ws, out))
        cnt = out[2]
        sp = float(1 - cnt.double().sum() / (32 * cfg.M * (cfg.M + 1) / 2))
        print(json.dumps({"g": g, "s": s, "estimate_ms": round(ms, 4),
                          "est_over_dense": round(ms / dense, 5),
                          "cost_model": pa.cost_ratio(cfg), "sparsity": round(sp, 4)}), flush=True)
        del ws, out
