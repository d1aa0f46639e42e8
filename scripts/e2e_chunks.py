"""proxyattn_forward_host (pinned host buffers, 128K headline shape) wall time per call for
several row-chunk counts (PROXYATTN_HOST_CHUNKS is read once per process: one count per run)."""
import json
import os
import sys
import time

import numpy as np
import torch

import paper_2509_24745_b200 as pa
import workloads

dev = torch.device("cuda:0")
cfg = pa.Config(32, 8, 128, 131072, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, 131072, 128, seed=0, params=workloads.PRESETS["llama-128k"])
Qh, Kh, Vh = Q.pin_memory(), K.pin_memory(), V.pin_memory()
Oh = torch.empty_like(Qh).pin_memory()
ks = torch.empty(32, dtype=torch.int32).pin_memory()
dws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=dev)
for _ in range(3):
    pa.forward_host(cfg, Qh, Kh, Vh, Oh, dws, ks)
ts = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pa.forward_host(cfg, Qh, Kh, Vh, Oh, dws, ks)
    ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"chunks": os.environ.get("PROXYATTN_HOST_CHUNKS", "8"), "median_ms": float(np.median(ts)),
                  "min_ms": float(np.min(ts))}))
