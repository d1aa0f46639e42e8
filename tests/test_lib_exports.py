"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every symbol that
include/proxyattn.h declares, and its host-side validation (no device work) follows the
config invariants.  No compute call is made without a GPU."""
import os
import re
import subprocess

import pytest

import paper_2509_24745_b200 as pa
from paper_2509_24745_b200 import build as pbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "proxyattn.h")


@pytest.fixture(scope="module")
def so():
    return pbuild.build()


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|double|const char\*)\s+(proxyattn_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["proxyattn_estimate", "proxyattn_prefill", "proxyattn_dense_prefill",
              "proxyattn_workspace_bytes", "proxyattn_pool", "proxyattn_proxy_scores",
              "proxyattn_budgets", "proxyattn_select", "proxyattn_cost_ratio",
              "proxyattn_last_error", "proxyattn_forward_host"]:
        assert s in syms


def test_library_exports_every_declared_symbol(so):
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (proxyattn_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert set(pa.EXPORTS) <= exported


def test_library_contains_sm100a_tcgen05_code(so):
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass          # tcgen05.mma
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass             # tcgen05.ld
    elf = subprocess.run(["cuobjdump", "-lelf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in elf


def test_loads_and_validates_configs_on_host(so):
    pa.lib()
    good = pa.Config(32, 8, 128, 32768, 128, 4, 1, 0.9)
    ws = pa.workspace_bytes(good)
    Ns, M = 32768 // 4, 256
    assert ws >= 2 * Ns * 128 * 2 + Ns * 4 + M * M * 4
    assert pa.cost_ratio(good) == pytest.approx(1 / 512)
    bad = {
        "gamma 0": (good.replace(gamma=0.0), pa._lib.E_CONFIG),
        "gamma > 1": (good.replace(gamma=1.5), pa._lib.E_CONFIG),
        "Hq % Hkv": (good.replace(n_q_heads=30), pa._lib.E_CONFIG),
        "Hkv % g": (good.replace(n_groups=3), pa._lib.E_CONFIG),
        "b % s": (good.replace(stride=3), pa._lib.E_CONFIG),
        "d = 96 in bf16": (good.replace(head_dim=96), pa._lib.E_UNSUPPORTED),
        "b = 256 in bf16": (good.replace(block_size=256), pa._lib.E_UNSUPPORTED),
        "shard not kv-aligned": (good.replace(q_head_begin=2, q_head_end=8), pa._lib.E_CONFIG),
        "M > 16384 (b = 128)": (good.replace(seq_len=16384 * 128 + 1), pa._lib.E_UNSUPPORTED),
        "M > 16384 (b = 64)": (good.replace(seq_len=16384 * 64 + 1, block_size=64), pa._lib.E_UNSUPPORTED),
    }
    for name, (cfg, code) in bad.items():
        with pytest.raises(pa.ProxyAttnError) as ei:
            pa.workspace_bytes(cfg)
        assert ei.value.code == code, name
    # the largest supported M (16384 block rows: 2M tokens at b = 128, 1M at b = 64)
    assert pa.workspace_bytes(good.replace(seq_len=16384 * 128)) > 0
    assert pa.workspace_bytes(good.replace(seq_len=16384 * 64, block_size=64)) > 0
    # ragged N is accepted: M = ceil(N / b)
    assert pa.workspace_bytes(good.replace(seq_len=32768 + 64)) > 0
    # FP32_DEBUG accepts the small config A shape (d=64, b=64)
    a = pa.Config(8, 2, 64, 1024, 64, 4, 2, 0.9, fp32_debug=True)
    assert pa.workspace_bytes(a) > 0
    # ... and so does the bf16 build (d in {64, 128}, b in {64, 128})
    for d, b in ((64, 64), (64, 128), (128, 64)):
        assert pa.workspace_bytes(pa.Config(8, 2, d, 1024, b, 4, 2, 0.9)) > 0


def test_shard_group_arithmetic():
    # Qwen 28/4, g=4 sharded over 2 ranks: each rank touches 2 complete groups
    cfg = pa.Config(28, 4, 128, 4096, 128, 4, 4, 0.9, q_head_begin=14, q_head_end=28)
    assert pa._lib._local_groups(cfg) == 2
    # Llama g=1 over 8 ranks: every rank touches the single (partial) group
    cfg = pa.Config(32, 8, 128, 4096, 128, 4, 1, 0.9, q_head_begin=4, q_head_end=8)
    assert pa._lib._local_groups(cfg) == 1


def test_token_major_and_varlen_configs_on_host(so):
    good = pa.Config(32, 8, 128, 4096, 128, 4, 1, 0.9)
    tok = good.replace(token_major=True)
    assert pa.workspace_bytes(tok) == pa.workspace_bytes(good)   # scratch is layout-free
    assert pa.workspace_bytes(tok.replace(q_token_stride=4096 + 8, kv_token_stride=1024)) > 0
    bad = {
        "q stride below the local heads": tok.replace(q_token_stride=32 * 128 - 8),
        "kv stride below the local heads": tok.replace(kv_token_stride=8 * 128 - 8),
        "stride not 16-byte": tok.replace(q_token_stride=32 * 128 + 4),
        "strides without the flag": good.replace(q_token_stride=8192),
    }
    for name, cfg in bad.items():
        with pytest.raises(pa.ProxyAttnError) as ei:
            pa.workspace_bytes(cfg)
        assert ei.value.code == pa._lib.E_CONFIG, name
    # varlen: estimate scratch sized by the longest sequence, plus every sequence's block lists
    # (one attention launch over all of them): more than the longest one alone, and growing
    # with the other sequences; validation of cu_seqlens
    one = pa.varlen_workspace_bytes(tok, [0, 4096])
    three = pa.varlen_workspace_bytes(tok, [0, 1000, 5096, 5096])
    assert three > one
    assert pa.varlen_workspace_bytes(tok, [0, 1000, 5096, 9192]) > three
    for cu in ([1, 100], [0, 100, 50]):
        with pytest.raises(pa.ProxyAttnError):
            pa.varlen_workspace_bytes(tok, cu)
    with pytest.raises(pa.ProxyAttnError):                     # needs the token-major layout
        pa.varlen_workspace_bytes(good, [0, 100])
