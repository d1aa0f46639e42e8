"""Per-event clock64 timeline of the densest head's last-row CTA of attn_tc7 (PROXYATTN_TRACE,
PROXYATTN_ATTN=7): PV-issuer waits and per-block softmax durations of both streams."""
import ctypes
import os
import sys

import numpy as np
import torch

import paper_2509_24745_b200 as pa
import workloads

os.environ.setdefault("PROXYATTN_ATTN", "7")
dev = torch.device("cuda:0")
N = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
cfg = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
kstar, _, cnt, idx = pa.estimate(cfg, Q, K)
h = int(torch.argmax(kstar))
r, M = 4, cfg.M
bid = (h // r) * (r * M) + (h % r)
os.environ["PROXYATTN_TRACE"] = str(bid)
for _ in range(2):
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
torch.cuda.synchronize()
tr = np.zeros(2 * 512 * 8, np.int64)
pa._lib._check(pa.lib().proxyattn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), tr.size))
pv = tr[:4096].reshape(512, 8)
sm = tr[4096:].reshape(256, 2, 8)
t0 = pv[0, 0]
print(f"head {h} kstar {int(kstar[h])} row {M-1} cnt {int(cnt[h, M - 1])}")
print("PV issuer (j): wait V,P | P0 ready | P1 ready | issued")
for j in list(range(0, 6)) + list(range(100, 106)):
    if pv[j, 0]:
        print(f"  j={j:3d}: " + " ".join(f"{int(x - t0):9d}" for x in pv[j, :4]))
print("softmax (js, s): start | end")
for js in list(range(1, 4)) + list(range(50, 54)):
    for s in range(2):
        e = sm[js, s]
        if e[0]:
            print(f"  js={js:3d} s={s}: {int(e[0] - t0):9d} {int(e[4] - t0):9d}  dur {int(e[4] - e[0])}")
for s in range(2):
    v = sm[20:200, s]
    v = v[v[:, 0] > 0]
    print(f"stream {s}: block {np.median(v[:, 4] - v[:, 0]):.0f}  iter {np.median(np.diff(v[:, 0])):.0f}")
v = pv[40:400]
v = v[v[:, 0] > 0]
print(f"PV: P0 wait {np.median(v[:,1]-v[:,0]):.0f}  P1 wait {np.median(v[:,2]-v[:,1]):.0f}  issue {np.median(v[:,3]-v[:,2]):.0f}"
      f"  per j {np.median(np.diff(v[:,0])):.0f}")
