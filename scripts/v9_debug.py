"""Debug driver for the row-pair attention kernel (attn_tc9): a few small sparse prefills on
cuda:0, each compared with the fp64 oracle; with a -DPA_WAIT_LOG build a stalled barrier wait
is printed (source line, block, thread) when the process exits."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2509_24745_b200 as pa  # noqa: E402
import workloads  # noqa: E402

dev = torch.device("cuda:0")
D = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cases = [(2, 1, 256), (2, 1, 384), (8, 2, 1024), (8, 2, 3000)]
for Hq, Hkv, N in cases:
    cfg = pa.Config(Hq, Hkv, D, N, 128, 4, 1, 0.9)
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, D, seed=0, device="cpu")
    Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
    kstar, budget, cnt, idx = pa.estimate(cfg, Qd, Kd)
    torch.cuda.synchronize()
    print("case d", D, Hq, Hkv, N, "cnt sum", int(cnt.sum()), flush=True)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    torch.cuda.synchronize()
    oc = oracle.Cfg(Hq, Hkv, D, N, 128, 4, 1, 0.9, round_bf16=True)
    Oref = oracle.attention(oc, Q.float().numpy(), K.float().numpy(), V.float().numpy(),
                            cnt.cpu().numpy(), idx.cpu().numpy())
    err = np.abs(O.float().cpu().numpy() - Oref)
    print(f"  max |dO| {err.max():.3e} mean {err.mean():.3e}", flush=True)
    M = cfg.M
    for h in range(Hq):
        for m in range(M):
            e = err[h, m * 128:(m + 1) * 128]
            if e.max() > 2e-2:
                lst = idx[h, m, :cnt[h, m]].tolist()
                print(f"    bad h {h} row {m} max {e.max():.3e} list {lst} rows>tol {int((e.max(axis=1) > 2e-2).sum())}", flush=True)
print("done")
