"""ProxyAttn (arXiv 2509.24745) hot path for NVIDIA B200 (sm_100a).

The package is a thin Python face over ``libproxyattn.so`` (C-ABI declared in
``include/proxyattn.h``): proxy-head pooling, proxy block scoring, Alg. 1 budgets with
per-head block selection, and tcgen05 block-sparse causal prefill attention.
"""
from ._lib import (  # noqa: F401
    EXPORTS,
    Config,
    ProxyAttnError,
    alloc_workspace,
    avgpool_estimate,
    avgpool_scores,
    avgpool_workspace_bytes,
    budgets,
    build_info,
    cost_ratio,
    debug_umma,
    dense_prefill,
    estimate,
    forward_host,
    forward_host_workspace_bytes,
    forward_varlen,
    lib,
    pool,
    prefill,
    proxy_scores,
    select,
    select_ws,
    varlen_workspace_bytes,
    with_strides,
    workspace_bytes,
)
