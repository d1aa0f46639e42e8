import numpy as np, torch, oracle, paper_2509_24745_b200 as pa
import sys; sys.path.insert(0, "tests")
from test_gpu_parity import *
cfg = llama_small(N=2048, gamma=1.0, heads=(4, 1))
g = torch.Generator().manual_seed(21)
Q = (torch.randn(4, 2048, 128, generator=g) * 0.5 + 0.5); Q[3] = -Q[3]
K = torch.randn(1, 2048, 128, generator=g) * 0.5
V = torch.randn(1, 2048, 128, generator=g)
K[0, 7 * 128 + 5] = 2.5; K[0, 9 * 128 + 77] = 10.0; K[0, 12 * 128 + 1] = -20.0
Q, K, V = Q.bfloat16(), K.bfloat16(), V.bfloat16()
Qd, Kd, Vd = to_dev(Q, K, V)
_, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
ref = oracle.attention(ocfg_of(cfg), np32(Q), np32(K), np32(V), cnt.cpu().numpy(), idx.cpu().numpy())
err = np.abs(np32(O) - ref).reshape(4, 16, 128, 128).max(axis=(2, 3))
np.set_printoptions(linewidth=200, precision=3)
print(err)
