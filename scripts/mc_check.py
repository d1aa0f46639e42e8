"""Multicast-attention debugging aid: prefill at a given shape with the current library and
compare with a saved reference output (or save one).
    python scripts/mc_check.py N HQ HKV [--save path | --check path]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2509_24745_b200 as pa  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("N", type=int)
ap.add_argument("hq", type=int)
ap.add_argument("hkv", type=int)
ap.add_argument("--save", default="")
ap.add_argument("--check", default="")
ap.add_argument("--preset", default="")
a = ap.parse_args()
dev = torch.device("cuda:0")
cfg = pa.Config(a.hq, a.hkv, 128, a.N, 128, 4, 1, 0.9)
Q, K, V, _ = workloads.structured(a.hq, a.hkv, a.N, 128, seed=3, device=dev,
                                  **({"params": workloads.PRESETS[a.preset]} if a.preset else {}))
_, _, cnt, idx = pa.estimate(cfg, Q, K)
O = pa.prefill(cfg, Q, K, V, cnt, idx)
torch.cuda.synchronize()
if a.save:
    torch.save(O.cpu(), a.save)
    print("saved", a.N, a.hq, a.hkv)
if a.check:
    ref = torch.load(a.check).to(dev)
    print("N", a.N, "heads", a.hq, a.hkv, "bitwise", torch.equal(O, ref), "max diff", float((O.float() - ref.float()).abs().max()))
