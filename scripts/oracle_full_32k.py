"""The oracle's FULL layer on BASELINE config B (Llama-3.1-8B shape, 32K, b = 128, s = 4,
g = 1, gamma = 0.9; BASELINE.md "CPU baseline plan": full estimation plus sparse attention),
timed stage by stage on the box's host cores, and the GPU layer (bench.py's launch
configuration) compared with it on EVERY element:

* L: |dL| <= 1e-4 on every causal cell of every block row;
* K*: exact on heads whose budget margin > 1e-4, |dK*| <= 1 otherwise;
* block lists: every (head, row), the near-tie rule of tests/test_gpu_parity.check_masks;
* O: every (head, row) with the GPU lists injected, bf16 tolerance (max 2e-2, mean 2e-3).

    python scripts/oracle_full_32k.py [--out profiles/r02_oracle_full_32k.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import paper_2509_24745_b200 as pa  # noqa: E402
import workloads  # noqa: E402
from test_gpu_parity import check_masks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="llama3.1-8b-attn-32k")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    w = dict(bench.WORKLOAD, seq_len=32768, preset="llama-32k", name="llama3.1-8b-attn-32k")
    dev = torch.device("cuda:0")
    Hq, Hkv, d, N, b = w["n_q_heads"], w["n_kv_heads"], w["head_dim"], w["seq_len"], w["block_size"]
    cfg = pa.Config(Hq, Hkv, d, N, b, w["stride"], w["n_groups"], w["gamma"], w["min_budget_tokens"])
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=0, params=workloads.PRESETS[w["preset"]], device=dev)
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K)
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
    qsum, ksum = pa.pool(cfg, Q, K)
    L = pa.proxy_scores(cfg, qsum, ksum)
    torch.cuda.synchronize()
    oc = oracle.Cfg(Hq, Hkv, d, N, b, w["stride"], w["n_groups"], w["gamma"], w["min_budget_tokens"],
                    round_bf16=True)
    Qf, Kf, Vf = (t.float().cpu().numpy() for t in (Q, K, V))
    M = oc.M
    t = {}
    t0 = time.perf_counter()
    Pq, Pk, sc = oracle.pool(oc, Qf, Kf)
    t["pool_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, Lref = oracle.proxy_scores(oc, Pq, Pk, sc)
    t["proxy_scores_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ks_ref, _, bmg, _ = oracle.budgets(oc, Qf, Kf)
    t["budgets_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    ocnt, oidx, _ = oracle.select(oc, Lref, ks_ref)
    t["select_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    oracle.attention(oc, Qf, Kf, Vf, ocnt, oidx)           # the oracle's own layer (timed)
    t["attention_s"] = time.perf_counter() - t0
    total_s = sum(t.values())

    # parity, every element
    Lg = L.cpu().numpy().astype(np.float64)
    tri = np.tril_indices(M)
    dL = float(np.max(np.abs(Lg[0][tri] - Lref[0][tri])))
    assert dL <= 1e-4, dL
    ks = kstar.cpu().numpy()
    ok = bmg > 1e-4
    assert np.array_equal(ks[ok], ks_ref[ok]) and np.all(np.abs(ks.astype(int) - ks_ref.astype(int)) <= 1)
    exact_rows, near_rows = check_masks(oc, Lref, ks, cnt, idx)
    t0 = time.perf_counter()
    Oref = oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy())   # GPU lists injected
    t_inj = time.perf_counter() - t0
    err = np.abs(O.float().cpu().numpy() - Oref)
    o_max, o_mean = float(err.max()), float(err.mean())
    assert o_max <= 2e-2 and o_mean <= 2e-3, (o_max, o_mean)
    rec = {
        "workload": w["name"], "config": "BASELINE config B (32K, Llama-3.1-8B shape, b=128, s=4, g=1, gamma=0.9)",
        "oracle_full_layer_s": total_s, "oracle_stage_s": t, "oracle_threads": oracle.num_threads(),
        "host_cpu": bench.host_cpu(),
        "parity": {"L_max_abs": dL, "kstar_exact_heads": int(ok.sum()), "heads": Hq,
                   "lists_exact_rows": exact_rows, "lists_near_tie_rows": near_rows,
                   "O_max_abs": o_max, "O_mean_abs": o_mean, "O_elements": int(err.size),
                   "oracle_attention_injected_s": t_inj},
        "sparsity_gpu": 1.0 - float(cnt.long().sum()) / (Hq * M * (M + 1) / 2),
    }
    print(json.dumps(rec))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
