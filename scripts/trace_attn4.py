"""Timeline of one heavy attn_tc4 CTA (PROXYATTN_ATTN=4, PROXYATTN_TRACE)."""
import ctypes, os, sys
import numpy as np, torch
import paper_2509_24745_b200 as pa, workloads
dev = torch.device("cuda:0"); N = 131072
cfg = pa.Config(32, 8, 128, N, 128, 4, 1, 0.9, 0)
Q, K, V, _ = workloads.structured(32, 8, N, 128, seed=0, params=workloads.PRESETS["llama-128k"], device=dev)
kstar, _, cnt, idx = pa.estimate(cfg, Q, K)
h = int(torch.argmax(kstar)); r, M = 4, cfg.M
bid = (h // r) * (r * M) + 0 * r + (h % r)
os.environ["PROXYATTN_TRACE"] = str(bid); os.environ["PROXYATTN_ATTN"] = "4"
O = pa.prefill(cfg, Q, K, V, cnt, idx); torch.cuda.synchronize()
tr = np.zeros(2 * 256 * 2 * 8, np.int64)
pa._lib._check(pa.lib().proxyattn_debug_trace(tr.ctypes.data_as(ctypes.c_void_p), tr.size))
tr = tr.reshape(2, 256, 2, 8); mma, sm = tr[0, :, 0], tr[1]
print(f"head {h} kstar {int(kstar[h])} cnt {int(cnt[h, M-1])}")
d = lambda a, b: float(np.median(a - b))
v = mma[40:200]; v = v[v[:, 0] > 0]
print(f"MMA: P0 wait {d(v[:,1], v[:,0]):.0f}  P1 wait {d(v[:,2], v[:,1]):.0f}  issue PV+S {d(v[:,3], v[:,2]):.0f}  iter {np.median(np.diff(v[:,0])):.0f}")
for c in range(2):
    w = sm[40:200, c]; w = w[w[:, 0] > 0]
    print(f"softmax half {c}: S-wait {d(w[:,1], w[:,0]):.0f}  load+max {d(w[:,2], w[:,1]):.0f}  exchange {d(w[:,3], w[:,2]):.0f}  exps {d(w[:,4], w[:,3]):.0f}  st+release {d(w[:,5], w[:,4]):.0f}  iter {np.median(np.diff(w[:,1])):.0f}")
