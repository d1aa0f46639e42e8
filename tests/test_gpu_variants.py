"""GPU: the selectable attention kernels kept for comparison (PROXYATTN_ATTN = 3..8: v3 two rows
per CTA — also the dense baseline —, v4 double-buffered S, v5 column-split softmax, v6 two
streams with online rescaling, v7 fixed reference, v8 persistent = the default) each against
the fp64 oracle with the same injected lists.  The variant is read once per process, so each
runs in a subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, torch, sys
sys.path.insert(0, %(root)r)
import oracle, workloads
import paper_2509_24745_b200 as pa
N, b = 2048, 128
cfg = pa.Config(8, 2, 128, N, b, 4, 1, 0.9)
Q, K, V, _ = workloads.structured(8, 2, N, 128, seed=77)
dev = torch.device("cuda:0")
Qd, Kd, Vd = (t.to(dev) for t in (Q, K, V))
kstar, _, cnt, idx = pa.estimate(cfg, Qd, Kd)
O = pa.prefill(cfg, Qd, Kd, Vd, cnt, idx)
Od = pa.dense_prefill(cfg, Qd, Kd, Vd)
oc = oracle.Cfg(8, 2, 128, N, b, 4, 1, 0.9, round_bf16=True)
Qf, Kf, Vf = (t.float().numpy() for t in (Q, K, V))
for got, ref in ((O, oracle.attention(oc, Qf, Kf, Vf, cnt.cpu().numpy(), idx.cpu().numpy())),
                 (Od, oracle.dense(oc, Qf, Kf, Vf))):
    err = np.abs(got.float().cpu().numpy() - ref)
    assert err.max() <= 2e-2 and err.mean() <= 2e-3, (err.max(), err.mean())
print("ok")
"""


@pytest.mark.parametrize("variant", ["3", "4", "5", "6", "7", "8"])
def test_attention_variant_matches_oracle(variant):
    env = dict(os.environ, PROXYATTN_ATTN=variant)
    r = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT}], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
