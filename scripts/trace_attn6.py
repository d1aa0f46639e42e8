"""Per-event clock64 timeline of the densest head's last-row CTA of attn_tc6 (PROXYATTN_TRACE)."""
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
bid = (h // r) * (r * M) + (h % r)          # row M-1 of head h (heaviest rows first)
os.environ["PROXYATTN_TRACE"] = str(bid)
for _ in range(2):
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
torch.cuda.synchronize()
tr = np.zeros(2 * 512 * 8, np.int64)
pa._lib._check(pa.lib().proxyattn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), tr.size))
mma = tr[:4096].reshape(512, 8)
sm = tr[4096:].reshape(256, 2, 8)
t0 = mma[0, 0]
c = int(cnt[h, M - 1])
print(f"head {h} kstar {int(kstar[h])} row {M-1} cnt {c}")
print("MMA (j): wait V,P | P0 ready | P1 ready | PV + S(j+2) issued")
for j in list(range(0, 6)) + list(range(100, 108)):
    if mma[j, 0]:
        print(f"  j={j:3d}: " + " ".join(f"{int(x - t0):9d}" for x in mma[j, :4]))
print("Softmax (js, s): wait S | S ready | max | P0 rel | P1 rel | exps0 | exps1 | O ready")
for js in list(range(0, 3)) + list(range(50, 54)):
    for s in range(2):
        e = sm[js, s]
        if e[0]:
            print(f"  js={js:3d} s={s}: " + " ".join(f"{int(x - t0):9d}" for x in e))


def d(a, b):
    return np.median(a - b)


for s in range(2):
    v = sm[20:200, s]
    v = v[v[:, 0] > 0]
    print(f"stream {s}: S-wait {d(v[:,1], v[:,0]):.0f}  ld+max {d(v[:,2], v[:,1]):.0f}  exps0 {d(v[:,5], v[:,2]):.0f}"
          f"  st0+odone {d(v[:,7], v[:,5]):.0f}  rescale+arrive0 {d(v[:,3], v[:,7]):.0f}  exps1 {d(v[:,6], v[:,3]):.0f}"
          f"  st1+arrive1 {d(v[:,4], v[:,6]):.0f}  iter {np.median(np.diff(v[:,1])):.0f}")
v = mma[40:400]
v = v[v[:, 0] > 0]
print(f"MMA: P0 wait {d(v[:,1], v[:,0]):.0f}  P1 wait {d(v[:,2], v[:,1]):.0f}  issue {d(v[:,3], v[:,2]):.0f}"
      f"  per j {np.median(np.diff(v[:,0])):.0f}")
