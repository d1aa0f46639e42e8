"""One cuDNN SDPA dense causal launch on the 128K headline inputs, bracketed by
cudaProfilerStart/Stop so that `ncu --profile-from-start off` captures exactly the vendor
kernel (comparison evidence for A7 / A8: clocks, tensor / XU pipe use, L2 -> SMEM traffic).

    ncu --set full --clock-control none --profile-from-start off -o out python scripts/cudnn_ncu.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "llama3.1-8b-attn-128k"
    w = bench.WORKLOADS[wl]
    dev = torch.device("cuda:0")
    Hq, Hkv, d, N = w["n_q_heads"], w["n_kv_heads"], w["head_dim"], w["seq_len"]
    Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=0, params=workloads.PRESETS[w["preset"]], device=dev)
    r = Hq // Hkv
    q = Q.unsqueeze(0)
    k = K.repeat_interleave(r, dim=0).unsqueeze(0)
    v = V.repeat_interleave(r, dim=0).unsqueeze(0)
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        for _ in range(2):
            F.scaled_dot_product_attention(q, k, v, is_causal=True)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        F.scaled_dot_product_attention(q, k, v, is_causal=True)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
    print("ok")


if __name__ == "__main__":
    main()
