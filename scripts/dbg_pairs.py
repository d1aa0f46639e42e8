import numpy as np, torch, sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle, workloads
import paper_2509_24745_b200 as pa
from test_gpu_parity import ocfg_of, np32, to_dev
for (d, b, N, heads, g, seed, stride) in [(64, 64, 1000, (6, 2), 2, 3, 2), (128, 64, 1000, (6, 2), 2, 3, 2), (64, 64, 1024, (6, 2), 2, 3, 2), (64, 64, 1000, (6, 2), 2, 3, 4)]:
    cfg = pa.Config(n_q_heads=heads[0], n_kv_heads=heads[1], head_dim=d, seq_len=N, block_size=b,
                    stride=stride, n_groups=g, gamma=0.9)
    Q, K, V, _ = workloads.structured(heads[0], heads[1], N, d, seed=seed)
    Qd, Kd, Vd = to_dev(Q, K, V)
    ks, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
    O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
    ref = oracle.attention(ocfg_of(cfg), np32(Q), np32(K), np32(V), cnt.cpu().numpy(), idx.cpu().numpy())
    err = np.abs(np32(O) - ref)
    M = cfg.M
    e = np.zeros((heads[0], M))
    for m in range(M):
        e[:, m] = np.nanmax(err[:, m * b:(m + 1) * b], axis=(1, 2))
    print((d, b, N, stride), "max", np.nanmax(err))
    bad = np.argwhere(e > 2e-2)
    print("bad (h,m):", bad.tolist()[:40])
    print("cnt:\n", cnt.cpu().numpy())
