"""Time proxyattn_forward_host (pinned host Q/K/V in, O out; the bench's e2e leg) on a bench
workload and check its outputs equal the device-resident estimate + prefill bit for bit.

    python scripts/e2e_time.py --tag X [--workload llama3.1-8b-attn-128k] [--steps 7]
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_24745_b200 as pa  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="run")
    ap.add_argument("--workload", default="llama3.1-8b-attn-128k")
    ap.add_argument("--steps", type=int, default=7)
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda:0")
    cfg = pa.Config(w["n_q_heads"], w["n_kv_heads"], w["head_dim"], w["seq_len"], w["block_size"],
                    w["stride"], w["n_groups"], w["gamma"], w["min_budget_tokens"])
    Q, K, V, _ = workloads.structured(cfg.n_q_heads, cfg.n_kv_heads, cfg.seq_len, cfg.head_dim, seed=0,
                                      params=workloads.PRESETS[w["preset"]], device=dev)
    ks, _, cnt, idx = pa.estimate(cfg, Q, K)
    Odev = pa.prefill(cfg, Q, K, V, cnt, idx).cpu()
    del cnt, idx
    Qh, Kh, Vh = (t.cpu().pin_memory() for t in (Q, K, V))
    del Q, K, V
    torch.cuda.empty_cache()
    Oh = torch.empty_like(Qh).pin_memory()
    ksh = torch.empty(cfg.n_q_heads, dtype=torch.int32).pin_memory()
    ws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=dev)
    pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws, ksh)
    pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws, ksh)
    ts = []
    for _ in range(a.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws, ksh)
        ts.append((time.perf_counter() - t0) * 1e3)
    rec = dict(tag=a.tag, workload=a.workload, ms=statistics.median(ts), min_ms=min(ts),
               defines=os.environ.get("PROXYATTN_NVCC_DEFINES", ""), bitwise_equal_device=bool(torch.equal(Oh, Odev)),
               kstar_equal=bool(torch.equal(ksh, ks.cpu())))
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
