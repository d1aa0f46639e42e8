"""Seeded synthetic Q/K/V generators (test and bench infrastructure).

This module holds NONE of the method's arithmetic (no pooling, scoring, budgets,
selection or attention); it only draws inputs, so both the CUDA path and the CPU oracle
consume the same tensors.  Recipes:

* ``iid``: Q, K, V ~ N(0, 1) i.i.d. (config A of BASELINE.json: "fp32 random Q/K/V").
* ``structured``: SURVEY.md §8(d) generator realising the paper's observations — a
  shared AR(1) focus process across heads (head consistency), per-head
  temperature beta_h (heads differ mainly in sparsity), attention sinks and
  needle keys (vertical patterns), local correlation (slash pattern):

      c_t = rho c_{t-1} + sqrt(1 - rho^2) eps_t                 (shared by all heads)
      K[kvh][t] = a c_t + sigma eps_{kvh,t} + [t < 4] A_sink sqrt(d) u + [t in needles] A_n sqrt(d) v
      Q[h][t]   = beta_h (a c_t + sigma eps_{h,t} + u + v),   beta_h ~ logU[beta_lo, beta_hi]
      V ~ N(0, 1)

  rounded to bf16.  Parameters are frozen per bench config in ``PRESETS``.
* ``needle``: a single key boosted against all queries (AC5 of S:526).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class StructParams:
    rho: float = 0.999
    sigma: float = 1.0
    a: float = 1.0
    A_sink: float = 2.0
    A_n: float = 2.5
    n_needles: int = 8
    beta_lo: float = 0.3
    beta_hi: float = 1.0


# Frozen per-config parameters (calibration recorded in DESIGN.md).
# Calibrated on B200 with scripts/calibrate.py (GPU estimate, seed 0, gamma = 0.9) against
# Table 8: Llama 128K target 83.86 % -> beta in [0.48, 1.44], sigma 0.93
# (sigma 1.0 gave 83.40 %, 0.85 gave 84.51 %); Qwen 64K (min budget 2048) target 74.12 % ->
# beta in [0.5, 1.5], sigma 0.9 (sigma 1.0: 73.42 %, 0.85: 74.53 %).
PRESETS: dict[str, StructParams] = {
    "default": StructParams(),
    "llama-128k": StructParams(sigma=0.93, beta_lo=0.48, beta_hi=1.44),
    "qwen-64k": StructParams(sigma=0.9, beta_lo=0.5, beta_hi=1.5),
    # scripts/calibrate_len.py (bisection on beta_lo, beta_hi = 3 beta_lo, sigma 0.93) against
    # P:941 Table 8 Llama: 16K 73.31 % (got 73.31), 32K 78.27 (78.28), 64K 83.19 (83.19);
    # 256K is not reported by the paper: scripts/calibrate_shape.py 32 8 128 262144 128
    # 0.8386 holds it at the 128K value (got 83.86 %; the paper's sparsity grows with length,
    # Table 8, so this is the conservative reading).
    "llama-16k": StructParams(sigma=0.93, beta_lo=0.311, beta_hi=0.933),
    "llama-32k": StructParams(sigma=0.93, beta_lo=0.4291, beta_hi=1.2873),
    "llama-64k": StructParams(sigma=0.93, beta_lo=0.548, beta_hi=1.644),
    "llama-256k": StructParams(sigma=0.93, beta_lo=0.6245, beta_hi=1.8735),
    # scripts/calibrate_shape.py 32 8 64 131072 128 0.8386: the head_dim-64 Llama-3.2-1B
    # shape at 128K calibrated to the same Table 8 Llama 128K sparsity (got 83.86 %); the
    # paper reports no d = 64 model, so the target is the 8B one
    "llama1b-128k": StructParams(sigma=0.93, beta_lo=0.9089, beta_hi=2.7267),
}


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def iid(n_q_heads: int, n_kv_heads: int, seq_len: int, head_dim: int, seed: int,
        dtype=torch.float32, device="cpu"):
    """Q [Hq][N][d], K/V [Hkv][N][d] ~ N(0,1), cast to ``dtype``."""
    g = _gen(device, seed)
    Q = torch.randn(n_q_heads, seq_len, head_dim, generator=g, device=device).to(dtype)
    K = torch.randn(n_kv_heads, seq_len, head_dim, generator=g, device=device).to(dtype)
    V = torch.randn(n_kv_heads, seq_len, head_dim, generator=g, device=device).to(dtype)
    return Q, K, V


def _ar1(seq_len: int, head_dim: int, rho: float, rng: np.random.Generator) -> np.ndarray:
    from scipy.signal import lfilter

    eps = rng.standard_normal((seq_len, head_dim))
    x = eps * np.sqrt(1.0 - rho * rho)
    x[0] = eps[0]                          # stationary start: c_0 ~ N(0, 1)
    return lfilter([1.0], [1.0, -rho], x, axis=0, zi=np.zeros((1, head_dim)))[0]


def structured(n_q_heads: int, n_kv_heads: int, seq_len: int, head_dim: int, seed: int,
               params: StructParams = StructParams(), dtype=torch.bfloat16, device="cpu"):
    """The §8(d) structured generator; returns (Q, K, V, meta)."""
    p = params
    rng = np.random.default_rng(seed)
    c = torch.from_numpy(_ar1(seq_len, head_dim, p.rho, rng).astype(np.float32)).to(device)
    u = rng.standard_normal(head_dim)
    u /= np.linalg.norm(u)
    v = rng.standard_normal(head_dim)
    v /= np.linalg.norm(v)
    u_t = torch.from_numpy(u.astype(np.float32)).to(device)
    v_t = torch.from_numpy(v.astype(np.float32)).to(device)
    beta = np.exp(rng.uniform(np.log(p.beta_lo), np.log(p.beta_hi), size=n_q_heads))
    needles = np.sort(rng.choice(seq_len, size=min(p.n_needles, seq_len), replace=False))
    g = _gen(device, seed + 1)
    sd = float(np.sqrt(head_dim))
    K = torch.empty(n_kv_heads, seq_len, head_dim, dtype=dtype, device=device)
    V = torch.empty_like(K)
    Q = torch.empty(n_q_heads, seq_len, head_dim, dtype=dtype, device=device)
    base = p.a * c
    needle_idx = torch.from_numpy(needles).to(device)
    for kvh in range(n_kv_heads):
        x = base + p.sigma * torch.randn(seq_len, head_dim, generator=g, device=device)
        x[: min(4, seq_len)] += p.A_sink * sd * u_t
        x[needle_idx] += p.A_n * sd * v_t
        K[kvh] = x.to(dtype)
    for kvh in range(n_kv_heads):
        V[kvh] = torch.randn(seq_len, head_dim, generator=g, device=device).to(dtype)
    for h in range(n_q_heads):
        x = base + p.sigma * torch.randn(seq_len, head_dim, generator=g, device=device) + u_t + v_t
        Q[h] = (float(beta[h]) * x).to(dtype)
    meta = dict(beta=beta.tolist(), needles=needles.tolist(), params=p.__dict__)
    return Q, K, V, meta


def needle(n_heads: int, seq_len: int, head_dim: int, pos: int, boost: float, seed: int,
           dtype=torch.float32):
    """Q, K, V ~ N(0,1)/sqrt(d)-scaled with key `pos` aligned to every query so that its
    logit is raised by `boost` ("K row j has large dot product with all Q rows")."""
    g = _gen("cpu", seed)
    Q = torch.randn(n_heads, seq_len, head_dim, generator=g) * 0.1
    K = torch.randn(n_heads, seq_len, head_dim, generator=g) * 0.1
    V = torch.randn(n_heads, seq_len, head_dim, generator=g)
    w = torch.randn(head_dim, generator=g)
    w /= w.norm()
    Q += w                                   # every query has a unit component along w
    K[:, pos] = boost * np.sqrt(head_dim) * w  # logit(t, pos) ~ boost
    return Q.to(dtype), K.to(dtype), V.to(dtype)


def needle_in_cold_block(n_blocks: int, block_size: int, head_dim: int, seed: int, boost: float = 12.0,
                         bias_hi: float = 2.0, dtype=torch.float32):
    """One head (Q, K, V [1][N][d], N = n_blocks * block_size) for SPEC's granularity
    criterion (AC5; the needle construction of S:372 and S:405): every query is a unit
    vector w plus small noise; the keys of block n carry a block-level logit bias
    beta_n ~ U[0, bias_hi] along w (distractor blocks with elevated AVERAGE scores) plus
    small noise, except one "cold" block n* (beta = 0) that hides a single needle key whose
    logit is `boost` for every query.  Returns (Q, K, V, n_star, needle_pos).  Deterministic
    in `seed`."""
    g = _gen("cpu", seed)
    rng = np.random.default_rng(seed)
    N = n_blocks * block_size
    n_star = 1 + seed % max(1, min(8, n_blocks - 2))
    pos = n_star * block_size + int(rng.integers(0, block_size))
    w = torch.randn(head_dim, generator=g)
    w /= w.norm()
    beta = torch.tensor(rng.uniform(0.0, bias_hi, n_blocks), dtype=torch.float32)
    beta[n_star] = 0.0
    sd = float(np.sqrt(head_dim))
    Q = (w + 0.05 * torch.randn(N, head_dim, generator=g)).unsqueeze(0)
    K = 0.05 * torch.randn(N, head_dim, generator=g)
    K += (beta.repeat_interleave(block_size) * sd).unsqueeze(1) * w     # logit ~ beta_n per token
    K[pos] = boost * sd * w                                              # the needle: logit ~ boost
    V = torch.randn(1, N, head_dim, generator=g)
    return Q.to(dtype), K.unsqueeze(0).to(dtype), V.to(dtype), n_star, pos
