"""Head-major vs token-major ([N][heads][d], the serving layout) at the 128K headline shape:
estimate + prefill time per layer, same values, graph replay, L2 flushed between steps."""
import json

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
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
out = {}
for name, c, q, k, v in (("head_major", cfg, Q, K, V),
                         ("token_major", cfg.replace(token_major=True),
                          *(t.transpose(0, 1).contiguous() for t in (Q, K, V)))):
    ws = pa.alloc_workspace(c, dev)
    res = (torch.empty(32, dtype=torch.int32, device=dev), torch.empty(32, dtype=torch.float32, device=dev),
           torch.empty(32, c.M, dtype=torch.int32, device=dev), torch.empty(32, c.M, c.M, dtype=torch.int32, device=dev))
    O = torch.empty_like(q)
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            pa.estimate(c, q, k, ws, out=res)
            pa.prefill(c, q, k, v, res[2], res[3], O)
        torch.cuda.synchronize()
        ge, gp = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(ge, stream=st):
            pa.estimate(c, q, k, ws, out=res)
        with torch.cuda.graph(gp, stream=st):
            pa.prefill(c, q, k, v, res[2], res[3], O)
        ts = []
        for _ in range(8):
            flush.zero_()
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(st)
            ge.replay()
            e[1].record(st)
            gp.replay()
            e[2].record(st)
            torch.cuda.synchronize()
            ts.append((e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])))
    ts.sort(key=lambda x: x[0] + x[1])
    out[name] = {"estimate_ms": round(ts[4][0], 3), "prefill_ms": round(ts[4][1], 3)}
    del ws, res, O
print(json.dumps(out))
