"""Validate bench.py's extrapolated oracle time against a FULL oracle layer on the same host:
the 32K config B layer (Llama-3.1-8B shape) timed un-sampled (pool, proxy scores, Alg. 1,
selection, attention) vs oracle_sample()'s bounded-sample extrapolation, same inputs, same
thread count.  CPU only (inputs from the CPU generator).

    python scripts/oracle_extrapolation_check.py [--threads T]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import oracle  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=0)
    a = ap.parse_args()
    if a.threads:
        oracle.set_num_threads(a.threads)
    w = dict(bench.WORKLOAD, seq_len=32768, preset="llama-32k", name="llama3.1-8b-attn-32k")
    Q, K, V, _ = bench.gen_inputs(w, "cpu")
    est_ms, sample, cores, parts = bench.oracle_sample(w, Q, K, V)
    oc = oracle.Cfg(w["n_q_heads"], w["n_kv_heads"], w["head_dim"], w["seq_len"], w["block_size"],
                    w["stride"], w["n_groups"], w["gamma"], w["min_budget_tokens"], round_bf16=True)
    Qf, Kf, Vf = (t.float().numpy() for t in (Q, K, V))
    t0 = time.perf_counter()
    Pq, Pk, sc = oracle.pool(oc, Qf, Kf)
    _, L = oracle.proxy_scores(oc, Pq, Pk, sc)
    ks, _, _, _ = oracle.budgets(oc, Qf, Kf)
    cnt, idx, _ = oracle.select(oc, L, ks)
    oracle.attention(oc, Qf, Kf, Vf, cnt, idx)
    full_ms = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"workload": w["name"], "threads": oracle.num_threads(), "full_layer_ms": full_ms,
                      "extrapolated_ms": est_ms, "ratio_extrapolated_over_full": est_ms / full_ms,
                      "sample": sample, "sample_stage_s": parts}))


if __name__ == "__main__":
    main()
