"""Per-event clock64 timeline of one heavy attention CTA (PROXYATTN_TRACE) at the bench config."""
import ctypes
import os
import sys

import numpy as np
import torch

import paper_2509_24745_b200 as pa
import workloads

dev = torch.device("cuda:0")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
kstar, _, cnt, idx = pa.estimate(cfg, Q, K)
h = int(torch.argmax(kstar))
r, M = 4, cfg.M
nrp = (M + 1) // 2
bid = (h // r) * (r * nrp) + 0 * r + (h % r)       # rows (M-1, M-2) of the densest head
os.environ["PROXYATTN_TRACE"] = str(bid)
O = pa.prefill(cfg, Q, K, V, cnt, idx)
torch.cuda.synchronize()
tr = np.zeros(2 * 256 * 2 * 8, np.int64)
pa._lib._check(pa.lib().proxyattn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), tr.size))
tr = tr.reshape(2, 256, 2, 8)
mma, sm = tr[0], tr[1]
t0 = mma[0, 0, 0]
print(f"head {h} kstar {int(kstar[h])} rows {M-1},{M-2} cnt {int(cnt[h, M-1])},{int(cnt[h, M-2])}")
print("MMA side (union step u, slot): wait_P | P0 ready | P1 ready | PV+nextS issued   (clk rel. to u=0)")
for u in list(range(0, 4)) + list(range(60, 68)):
    for s in range(2):
        e = mma[u, s]
        if e[0]:
            print(f"  u={u:3d} s={s}: " + " ".join(f"{int(x - t0):9d}" for x in e[:4]))
print("Softmax side (own iter j, slot): wait_S | S ready | max done | P0 rel | P1 rel")
for j in list(range(0, 4)) + list(range(60, 68)):
    for s in range(2):
        e = sm[j, s]
        if e[0]:
            print(f"  j={j:3d} s={s}: " + " ".join(f"{int(x - t0):9d}" for x in e[:5]))
# steady-state averages
def d(a, b):
    return np.median(a - b)
ss = sm[40:200]
valid = ss[:, :, 0] > 0
for s in range(2):
    v = ss[:, s][valid[:, s]]
    print(f"slot {s}: S-wait {d(v[:,1], v[:,0]):.0f}  load+max {d(v[:,2], v[:,1]):.0f}  half0 {d(v[:,3], v[:,2]):.0f}  half1 {d(v[:,4], v[:,3]):.0f}  iter {np.median(np.diff(v[:,1])):.0f}")
    print(f"        exps0 {d(v[:,5], v[:,2]):.0f}  st0+odone {d(v[:,7], v[:,5]):.0f}  fence+arrive0 {d(v[:,3], v[:,7]):.0f}  exps1 {d(v[:,6], v[:,3]):.0f}  st1+arrive1 {d(v[:,4], v[:,6]):.0f}")
mm = mma[40:200]
for s in range(2):
    v = mm[:, s][mm[:, s, 0] > 0]
    print(f"MMA slot {s}: P0 wait {d(v[:,1], v[:,0]):.0f}  P1 wait {d(v[:,2], v[:,1]):.0f}  issue {d(v[:,3], v[:,2]):.0f}")
