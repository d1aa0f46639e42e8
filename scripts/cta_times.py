"""Per-CTA timing of the attention launch (PROXYATTN_CTA_TIMES, attn_tc7): SM busy fraction,
per-CTA fixed cost vs per-block cost (least squares), and where the time goes."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("PROXYATTN_ATTN", "7")
os.environ["PROXYATTN_CTA_TIMES"] = "1"
import paper_2509_24745_b200 as pa
import workloads

dev = torch.device("cuda:0")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
kstar, _, cnt, idx = pa.estimate(cfg, Q, K)
O = torch.empty_like(Q)
for _ in range(3):
    pa.prefill(cfg, Q, K, V, cnt, idx, O)
torch.cuda.synchronize()
ncta = 32 * cfg.M
tr = np.zeros(ncta * 4, np.int64)
pa._lib._check(pa.lib().proxyattn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), tr.size))
tr = tr.reshape(ncta, 4)
t0, t1 = tr[:, 0].min(), tr[:, 1].max()
dur = (tr[:, 1] - tr[:, 0]).astype(float)
blocks = tr[:, 3] & ((1 << 20) - 1)
rerun = (tr[:, 3] >> 20) > 0
print(f"kernel span {(t1 - t0) / 1e6:.3f} ms, CTAs {ncta}, re-run rows {int(rerun.sum())}")
busy = np.zeros(148)
for sm in range(148):
    sel = tr[:, 2] == sm
    busy[sm] = dur[sel].sum()
print(f"SM busy: mean {busy.mean() / (t1 - t0):.3f}, min {busy.min() / (t1 - t0):.3f}")
A = np.stack([np.ones(ncta), blocks], 1)
coef, *_ = np.linalg.lstsq(A, dur, rcond=None)
print(f"fit: CTA duration = {coef[0]:.0f} ns + {coef[1]:.1f} ns/block")
for lo, hi in ((1, 2), (2, 4), (4, 8), (8, 16), (16, 64), (64, 256), (256, 2000)):
    sel = (blocks >= lo) & (blocks < hi)
    if sel.any():
        print(f"  blocks [{lo},{hi}): {sel.sum():6d} CTAs, mean dur {dur[sel].mean():9.0f} ns, "
              f"ns/block {(dur[sel] / blocks[sel]).mean():7.1f}, time share {dur[sel].sum() / dur.sum():.3f}")
# end-to-start gaps on each SM (launch / drain overhead between consecutive CTAs)
gaps = []
for sm in range(148):
    sel = np.where(tr[:, 2] == sm)[0]
    order = sel[np.argsort(tr[sel, 0])]
    g = tr[order[1:], 0] - tr[order[:-1], 1]
    gaps.extend(g.tolist())
gaps = np.array(gaps)
print(f"gap between CTAs on an SM: median {np.median(gaps):.0f} ns, mean {gaps.mean():.0f} ns, total share "
      f"{gaps[gaps > 0].sum() / (148 * (t1 - t0)):.3f}")
