"""Packed variable-length batch through proxyattn_forward_varlen (one attention launch over all
sequences) against one estimate + prefill call per sequence, same inputs; prints ms."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2509_24745_b200 as pa
import workloads

lens = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [16384] * 8
dev = torch.device("cuda:0")
Hq, Hkv = 32, 8
seqs = [workloads.structured(Hq, Hkv, n, 128, seed=i, params=workloads.PRESETS["llama-16k"], device=dev)
        for i, n in enumerate(lens)]
tok = lambda t: t.transpose(0, 1).contiguous()  # noqa: E731
packed = [torch.cat([tok(s[j]) for s in seqs], 0) for j in range(3)]
cu = np.concatenate([[0], np.cumsum(lens)]).tolist()
cfg = pa.Config(Hq, Hkv, 128, 1, 128, 4, 1, 0.9, token_major=True)


def timed(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


t_packed = timed(lambda: pa.forward_varlen(cfg, cu, *packed))
# the same call replayed from a CUDA graph (the call is asynchronous and capturable): GPU time
wsv = torch.empty(pa.varlen_workspace_bytes(cfg, cu), dtype=torch.uint8, device=dev)
Ov = torch.empty_like(packed[0])
ksv = torch.zeros(len(lens), Hq, dtype=torch.int32, device=dev)
st = torch.cuda.Stream()
st.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(st):
    pa.forward_varlen(cfg, cu, *packed, O=Ov, workspace=wsv, kstar=ksv)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        pa.forward_varlen(cfg, cu, *packed, O=Ov, workspace=wsv, kstar=ksv)
torch.cuda.synchronize()
t_graph = timed(g.replay)
cfgs = [pa.Config(Hq, Hkv, 128, n, 128, 4, 1, 0.9) for n in lens]
wss = [pa.alloc_workspace(c, dev) for c in cfgs]


def loop():
    for c, w, (Q, K, V, _) in zip(cfgs, wss, seqs):
        _, _, cnt, idx = pa.estimate(c, Q, K, w)
        pa.prefill(c, Q, K, V, cnt, idx)


t_loop = timed(loop)
print(json.dumps({"lens": lens, "packed_one_launch_ms": t_packed, "packed_graph_replay_ms": t_graph,
                  "per_sequence_calls_ms": t_loop}))
