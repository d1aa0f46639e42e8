"""Time the A7 attention launch alone (and optionally the estimate) on a bench workload:
L2 flushed before every timed launch, CUDA events on the launching stream, median of K,
NVML SM clock median during the timed loop.  Used to compare experimental builds
(PROXYATTN_NVCC_DEFINES) — a line per run, tagged.

    python scripts/attn_time.py --tag base [--workload llama3.1-8b-attn-128k] [--steps 10]
        [--save-out /tmp/O.pt | --check-out /tmp/O.pt] [--estimate] [--dense]
"""
import argparse
import json
import os
import statistics
import sys

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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--save-out", default="")
    ap.add_argument("--check-out", default="")
    ap.add_argument("--estimate", action="store_true")
    ap.add_argument("--dense", action="store_true")
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    dev = torch.device("cuda:0")
    cfg = pa.Config(w["n_q_heads"], w["n_kv_heads"], w["head_dim"], w["seq_len"], w["block_size"],
                    w["stride"], w["n_groups"], w["gamma"], w["min_budget_tokens"],
                    static_kstar=w.get("static_kstar", 0))
    Q, K, V, _ = workloads.structured(cfg.n_q_heads, cfg.n_kv_heads, cfg.seq_len, cfg.head_dim, seed=0,
                                      params=workloads.PRESETS[w["preset"]], device=dev)
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
    O = torch.empty_like(Q)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def run():
        if a.dense:
            pa.dense_prefill(cfg, Q, K, V, O=O)
        elif a.estimate:
            pa.estimate(cfg, Q, K)
        else:
            pa.prefill(cfg, Q, K, V, cnt, idx, O=O)

    for _ in range(a.warmup):
        run()
    torch.cuda.synchronize()
    times = []
    with bench.ClockSampler(0) as clk:
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run()
            e1.record(st)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    units = int(cnt.long().sum()) if not a.dense else cfg.n_q_heads * cfg.M * (cfg.M + 1) // 2
    b, d = cfg.block_size, cfg.head_dim
    tf = units * 4 * b * b * d / (ms * 1e-3) / 1e12
    rec = dict(tag=a.tag, workload=a.workload, ms=ms, min_ms=min(times), tflops=tf, units=units,
               defines=os.environ.get("PROXYATTN_NVCC_DEFINES", ""), clocks=getattr(clk, "result", None))
    if a.save_out:
        torch.save(O.cpu(), a.save_out)
    if a.check_out and os.path.exists(a.check_out):
        ref = torch.load(a.check_out).to(dev)
        diff = (O.float() - ref.float()).abs()
        rec["max_diff_vs_ref"] = float(diff.max())
        rec["mean_diff_vs_ref"] = float(diff.mean())
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
