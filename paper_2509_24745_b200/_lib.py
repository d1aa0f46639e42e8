"""ctypes binding of libproxyattn (include/proxyattn.h) — argument marshalling only.

Every compute step runs in the CUDA kernels behind the C-ABI; this module only turns
torch tensors into device pointers and the current CUDA stream into a cudaStream_t.
It fails loudly when the shared library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, replace

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_PKG, "libproxyattn.so")

FLAG_FP32_DEBUG = 0x1
FLAG_CHECK = 0x2
FLAG_FORCE_SINK = 0x4
FLAG_CONSTANT_K = 0x8
FLAG_DESIGNATED_HEAD = 0x10
FLAG_TOKEN_MAJOR = 0x20
FLAG_KSTAR_GIVEN = 0x40
FLAG_SCORES_ONLY = 0x80
FLAG_CHECK_FINITE = 0x100

OK = 0
E_CONFIG = -1
E_UNSUPPORTED = -2
E_SHAPE = -3
E_WORKSPACE = -4
E_CUDA = -5
E_NONFINITE = -6


class ProxyAttnError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"proxyattn error {code}: {msg}")
        self.code = code


class _CCfg(ctypes.Structure):
    _fields_ = [
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("seq_len", ctypes.c_int64),
        ("block_size", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("n_groups", ctypes.c_int32),
        ("gamma", ctypes.c_float),
        ("min_budget_tokens", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("q_head_begin", ctypes.c_int32),
        ("q_head_end", ctypes.c_int32),
        ("static_kstar", ctypes.c_int32),
        ("row_begin", ctypes.c_int32),
        ("row_end", ctypes.c_int32),
        ("q_token_stride", ctypes.c_int64),
        ("kv_token_stride", ctypes.c_int64),
    ]


@dataclass(frozen=True)
class Config:
    """proxyattn_cfg (S:27-34 AttnConfig plus the build flags and the head shard)."""

    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    seq_len: int
    block_size: int = 128
    stride: int = 4
    n_groups: int = 1
    gamma: float = 0.9
    min_budget_tokens: int = 0
    fp32_debug: bool = False
    check: bool = False
    q_head_begin: int = 0
    q_head_end: int = 0
    force_sink: bool = False        # method variants
    constant_k: bool = False
    designated_head: bool = False
    static_kstar: int = 0
    row_begin: int = 0              # prefill row range (zig-zag row sharding); 0/0 = all rows
    row_end: int = 0
    kstar_given: bool = False       # estimate: kstar is an input (row-range calls after the first)
    scores_only: bool = False       # estimate: stop before the selection (select_ws finishes)
    token_major: bool = False       # Q/K/V/O as [N][heads][d] with token strides (0 = packed)
    q_token_stride: int = 0
    kv_token_stride: int = 0
    check_finite: bool = False      # validate Q/K/V (NaN / Inf -> E_NONFINITE, S:49 / S:319)

    @property
    def M(self) -> int:
        return -(-self.seq_len // self.block_size)     # ceil: a partial last block is padded

    @property
    def Ns(self) -> int:
        return -(-self.seq_len // self.stride)

    @property
    def r(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    @property
    def local_heads(self) -> tuple[int, int]:
        return self.q_head_begin, (self.q_head_end or self.n_q_heads)

    @property
    def Hl(self) -> int:
        b, e = self.local_heads
        return e - b

    @property
    def dtype(self) -> torch.dtype:
        return torch.float32 if self.fp32_debug else torch.bfloat16

    def replace(self, **kw) -> "Config":
        return replace(self, **kw)

    def c(self) -> _CCfg:
        flags = ((FLAG_FP32_DEBUG if self.fp32_debug else 0) | (FLAG_CHECK if self.check else 0)
                 | (FLAG_FORCE_SINK if self.force_sink else 0)
                 | (FLAG_CONSTANT_K if self.constant_k else 0)
                 | (FLAG_DESIGNATED_HEAD if self.designated_head else 0)
                 | (FLAG_TOKEN_MAJOR if self.token_major else 0)
                 | (FLAG_KSTAR_GIVEN if self.kstar_given else 0)
                 | (FLAG_SCORES_ONLY if self.scores_only else 0)
                 | (FLAG_CHECK_FINITE if self.check_finite else 0))
        return _CCfg(self.n_q_heads, self.n_kv_heads, self.head_dim, self.seq_len,
                     self.block_size, self.stride, self.n_groups, float(self.gamma),
                     self.min_budget_tokens, flags, self.q_head_begin, self.q_head_end,
                     self.static_kstar, self.row_begin, self.row_end, self.q_token_stride,
                     self.kv_token_stride)


_lib = None
_P = ctypes.c_void_p
_CP = ctypes.POINTER(_CCfg)

_SIGS = {
    "proxyattn_workspace_bytes": ([_CP, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "proxyattn_estimate": ([_CP, _P, _P, _P, ctypes.c_size_t, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_prefill": ([_CP, _P, _P, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_dense_prefill": ([_CP, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_pool": ([_CP, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_proxy_scores": ([_CP, _P, _P, _P, ctypes.c_size_t, _P, _P], ctypes.c_int),
    "proxyattn_budgets": ([_CP, _P, _P, _P, ctypes.c_size_t, _P, _P, _P], ctypes.c_int),
    "proxyattn_select": ([_CP, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_select_ws": ([_CP, _P, ctypes.c_size_t, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_forward_host_workspace_bytes": ([_CP, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "proxyattn_forward_host": ([_CP, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "proxyattn_cost_ratio": ([_CP], ctypes.c_double),
    "proxyattn_last_error": ([], ctypes.c_char_p),
    "proxyattn_build_info": ([], ctypes.c_char_p),
    "proxyattn_debug_umma": ([_P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_avgpool_workspace_bytes": ([_CP, ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
    "proxyattn_avgpool_scores": ([_CP, _P, _P, _P, ctypes.c_size_t, _P, _P], ctypes.c_int),
    "proxyattn_avgpool_estimate": ([_CP, _P, _P, _P, ctypes.c_size_t, _P, _P, _P, _P, _P], ctypes.c_int),
    "proxyattn_varlen_workspace_bytes": ([_CP, ctypes.c_int32, _P, ctypes.POINTER(ctypes.c_size_t)],
                                         ctypes.c_int),
    "proxyattn_forward_varlen": ([_CP, ctypes.c_int32, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P, _P],
                                 ctypes.c_int),
}

EXPORTS = tuple(_SIGS)


def lib() -> ctypes.CDLL:
    """Load libproxyattn.so (built by __graft_entry__.build()); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(
                f"{SO_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(SO_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc != OK:
        raise ProxyAttnError(rc, lib().proxyattn_last_error().decode())


def _ptr(t: torch.Tensor | None, dtype: torch.dtype | None = None, cuda: bool = True):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"expected a {dtype} tensor, got {t.dtype}")
    if cuda and not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _tptr(t: torch.Tensor | None, cfg: "Config", role: str = "q"):
    """Pointer of a Q/K/V/O tensor (role "q" for Q / O, "kv" for K / V) in cfg's element type:
    contiguous head-major, or token-major [N][heads][d] whose token stride is the one in cfg
    (0 = packed: local heads x d) with rows of d contiguous elements."""
    if t is None:
        return None
    if not cfg.token_major:
        return _ptr(t, cfg.dtype)
    if t.dtype != cfg.dtype or not t.is_cuda:
        raise ValueError(f"expected a CUDA {cfg.dtype} tensor, got {t.dtype} on {t.device}")
    if t.dim() != 3 or t.stride(2) != 1 or (t.shape[1] > 1 and t.stride(1) != t.shape[2]):
        raise ValueError("token-major tensors must be [N][heads][d] with contiguous heads x d rows")
    heads = cfg.Hl if role == "q" else cfg.Hl // cfg.r
    want = (cfg.q_token_stride if role == "q" else cfg.kv_token_stride) or heads * cfg.head_dim
    if t.shape[0] > 1 and t.stride(0) != want:
        raise ValueError(f"{role} token stride {t.stride(0)} != the config's {want} (use with_strides)")
    return ctypes.c_void_p(t.data_ptr())


def with_strides(cfg: "Config", Q: torch.Tensor, K: torch.Tensor) -> "Config":
    """Token-major config whose token strides are taken from the tensors (e.g. head slices
    of a packed [N][H][d] activation)."""
    return cfg.replace(token_major=True, q_token_stride=Q.stride(0), kv_token_stride=K.stride(0))


def _like_q(cfg: "Config", Q: torch.Tensor) -> torch.Tensor:
    """An output with Q's layout (token-major outputs share Q's token stride)."""
    if not cfg.token_major or Q.is_contiguous():
        return torch.empty_like(Q)
    n, h, d = Q.shape
    buf = torch.empty(n * Q.stride(0), dtype=Q.dtype, device=Q.device)
    return buf.as_strided((n, h, d), (Q.stride(0), d, 1))


def _stream(device: torch.device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _cfg_ref(cfg: Config):
    return ctypes.byref(cfg.c())


def workspace_bytes(cfg: Config) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().proxyattn_workspace_bytes(_cfg_ref(cfg), ctypes.byref(n)))
    return n.value


def alloc_workspace(cfg: Config, device) -> torch.Tensor:
    return torch.empty(workspace_bytes(cfg), dtype=torch.uint8, device=device)


def _check_out(cfg: Config, out, lists: bool = True) -> None:
    """Shapes / dtypes / device of (kstar, budget, block_cnt, block_idx) output tensors."""
    Hl, M = cfg.Hl, cfg.M
    want = [((Hl,), torch.int32), ((Hl,), torch.float32), ((Hl, M), torch.int32), ((Hl, M, M), torch.int32)]
    for k, (t, (shape, dt)) in enumerate(zip(out, want)):
        if t is None and k >= 2 and not lists:
            continue
        if t is None or tuple(t.shape) != shape or t.dtype != dt or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"output {k} must be a contiguous CUDA {dt} tensor of shape {shape}")


def estimate(cfg: Config, Q: torch.Tensor, K: torch.Tensor, workspace: torch.Tensor | None = None,
             out: tuple | None = None):
    """proxyattn_estimate -> (kstar [Hl] i32, budget [Hl] f32, block_cnt [Hl][M] i32,
    block_idx [Hl][M][M] i32)."""
    dev = Q.device
    if workspace is None:
        workspace = alloc_workspace(cfg, dev)
    if out is None:
        Hl, M = cfg.Hl, cfg.M
        out = (torch.empty(Hl, dtype=torch.int32, device=dev),
               torch.empty(Hl, dtype=torch.float32, device=dev),
               torch.empty(Hl, M, dtype=torch.int32, device=dev),
               torch.empty(Hl, M, M, dtype=torch.int32, device=dev))
    _check_out(cfg, out, lists=not cfg.scores_only)
    kstar, budget, cnt, idx = out
    _check(lib().proxyattn_estimate(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _ptr(workspace),
                                    workspace.numel(), _ptr(kstar), _ptr(budget), _ptr(cnt),
                                    _ptr(idx), _stream(dev)))
    return kstar, budget, cnt, idx


def prefill(cfg: Config, Q, K, V, block_cnt, block_idx, O=None):
    """proxyattn_prefill -> O [Hl][N][d]."""
    if O is None:
        O = _like_q(cfg, Q)
    if tuple(block_cnt.shape) != (cfg.Hl, cfg.M) or tuple(block_idx.shape) != (cfg.Hl, cfg.M, cfg.M):
        raise ValueError("block lists must be [Hl][M] and [Hl][M][M]")
    _check(lib().proxyattn_prefill(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _tptr(V, cfg, "kv"),
                                   _ptr(block_cnt, torch.int32), _ptr(block_idx, torch.int32), _tptr(O, cfg),
                                   _stream(Q.device)))
    return O


def dense_prefill(cfg: Config, Q, K, V, O=None):
    """proxyattn_dense_prefill -> O [Hl][N][d]."""
    if O is None:
        O = _like_q(cfg, Q)
    _check(lib().proxyattn_dense_prefill(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _tptr(V, cfg, "kv"),
                                         _tptr(O, cfg), _stream(Q.device)))
    return O


def pool(cfg: Config, Q, K):
    """proxyattn_pool -> fp32 (qsum, ksum) [g_l][N/s][d]."""
    gl = _local_groups(cfg)
    shape = (gl, cfg.Ns, cfg.head_dim)
    qsum = torch.empty(shape, dtype=torch.float32, device=Q.device)
    ksum = torch.empty_like(qsum)
    _check(lib().proxyattn_pool(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _ptr(qsum), _ptr(ksum),
                                _stream(Q.device)))
    return qsum, ksum


def proxy_scores(cfg: Config, qsum, ksum, workspace=None):
    """proxyattn_proxy_scores -> L [g_l][M][M] fp32 (log domain, -inf above the diagonal)."""
    if workspace is None:
        workspace = alloc_workspace(cfg, qsum.device)
    L = torch.empty(_local_groups(cfg), cfg.M, cfg.M, dtype=torch.float32, device=qsum.device)
    _check(lib().proxyattn_proxy_scores(_cfg_ref(cfg), _ptr(qsum), _ptr(ksum), _ptr(workspace),
                                        workspace.numel(), _ptr(L), _stream(qsum.device)))
    return L


def budgets(cfg: Config, Q, K, workspace=None):
    """proxyattn_budgets -> (kstar [Hl] i32, budget [Hl] f32)."""
    if workspace is None:
        workspace = alloc_workspace(cfg, Q.device)
    kstar = torch.empty(cfg.Hl, dtype=torch.int32, device=Q.device)
    budget = torch.empty(cfg.Hl, dtype=torch.float32, device=Q.device)
    _check(lib().proxyattn_budgets(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _ptr(workspace),
                                   workspace.numel(), _ptr(kstar), _ptr(budget),
                                   _stream(Q.device)))
    return kstar, budget


def select(cfg: Config, L, kstar):
    """proxyattn_select -> (block_cnt [Hl][M], block_idx [Hl][M][M])."""
    cnt = torch.empty(cfg.Hl, cfg.M, dtype=torch.int32, device=L.device)
    idx = torch.empty(cfg.Hl, cfg.M, cfg.M, dtype=torch.int32, device=L.device)
    _check(lib().proxyattn_select(_cfg_ref(cfg), _ptr(L), _ptr(kstar), _ptr(cnt), _ptr(idx),
                                  _stream(L.device)))
    return cnt, idx


def select_ws(cfg: Config, workspace, kstar, out):
    """proxyattn_select_ws: A5-A6 of rows [row_begin, row_end) from the L a scores_only
    estimate left in `workspace`; writes out = (block_cnt, block_idx)."""
    _check_out(cfg, (kstar, torch.empty(cfg.Hl, device=kstar.device)) + tuple(out))
    cnt, idx = out
    _check(lib().proxyattn_select_ws(_cfg_ref(cfg), _ptr(workspace), workspace.numel(), _ptr(kstar),
                                     _ptr(cnt), _ptr(idx), _stream(workspace.device)))
    return cnt, idx


def forward_host_workspace_bytes(cfg: Config) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().proxyattn_forward_host_workspace_bytes(_cfg_ref(cfg), ctypes.byref(n)))
    return n.value


def forward_host(cfg: Config, Qh, Kh, Vh, Oh, device_ws, kstar_h=None):
    """proxyattn_forward_host on host (CPU, ideally pinned) tensors; synchronises."""
    h = dict(dtype=cfg.dtype, cuda=False)
    _check(lib().proxyattn_forward_host(_cfg_ref(cfg), _ptr(Qh, **h), _ptr(Kh, **h), _ptr(Vh, **h), _ptr(Oh, **h),
                                        _ptr(kstar_h, torch.int32, cuda=False), _ptr(device_ws), device_ws.numel(),
                                        _stream(device_ws.device)))
    return Oh


def _cu(cu_seqlens) -> torch.Tensor:
    cu = torch.as_tensor(cu_seqlens, dtype=torch.int64).cpu().contiguous()
    if cu.dim() != 1 or cu.numel() < 1:
        raise ValueError("cu_seqlens must be a 1-D list of n_seqs + 1 offsets")
    return cu


def varlen_workspace_bytes(cfg: Config, cu_seqlens) -> int:
    cu = _cu(cu_seqlens)
    n = ctypes.c_size_t(0)
    _check(lib().proxyattn_varlen_workspace_bytes(_cfg_ref(cfg), cu.numel() - 1,
                                                  ctypes.c_void_p(cu.data_ptr()), ctypes.byref(n)))
    return n.value


def forward_varlen(cfg: Config, cu_seqlens, Q, K, V, O=None, workspace=None, kstar=None):
    """proxyattn_forward_varlen: packed token-major Q/K/V [total][heads][d], sequence i =
    tokens [cu[i], cu[i+1]); each sequence is its own ProxyAttn layer.  Returns (O, kstar
    [n_seqs][Hl] int32)."""
    if not cfg.token_major:
        cfg = with_strides(cfg, Q, K)
    cu = _cu(cu_seqlens)
    n = cu.numel() - 1
    if workspace is None:
        workspace = torch.empty(varlen_workspace_bytes(cfg, cu), dtype=torch.uint8, device=Q.device)
    if O is None:
        O = _like_q(cfg, Q)
    if kstar is None:
        kstar = torch.zeros(max(n, 1), cfg.Hl, dtype=torch.int32, device=Q.device)
    _check(lib().proxyattn_forward_varlen(_cfg_ref(cfg), n, ctypes.c_void_p(cu.data_ptr()),
                                          _tptr(Q, cfg), _tptr(K, cfg, "kv"), _tptr(V, cfg, "kv"), _tptr(O, cfg),
                                          _ptr(workspace), workspace.numel(), _ptr(kstar),
                                          _stream(Q.device)))
    return O, kstar[:n]


def avgpool_workspace_bytes(cfg: Config) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().proxyattn_avgpool_workspace_bytes(_cfg_ref(cfg), ctypes.byref(n)))
    return n.value


def avgpool_scores(cfg: Config, Q, K, workspace=None):
    """proxyattn_avgpool_scores -> S [Hl][M][M] fp32: the seq-avgpool comparator's per-head
    log-domain block scores, -inf above the diagonal."""
    if workspace is None:
        workspace = torch.empty(avgpool_workspace_bytes(cfg), dtype=torch.uint8, device=Q.device)
    S = torch.empty(cfg.Hl, cfg.M, cfg.M, dtype=torch.float32, device=Q.device)
    _check(lib().proxyattn_avgpool_scores(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _ptr(workspace),
                                          workspace.numel(), _ptr(S), _stream(Q.device)))
    return S


def avgpool_estimate(cfg: Config, Q, K, workspace=None, out: tuple | None = None):
    """proxyattn_avgpool_estimate -> (kstar, budget, block_cnt, block_idx), the comparator's
    selection (the same Alg. 1 budgets and Eq. 3 rule on per-head avgpool maps)."""
    dev = Q.device
    if workspace is None:
        workspace = torch.empty(avgpool_workspace_bytes(cfg), dtype=torch.uint8, device=dev)
    if out is None:
        Hl, M = cfg.Hl, cfg.M
        out = (torch.empty(Hl, dtype=torch.int32, device=dev), torch.empty(Hl, dtype=torch.float32, device=dev),
               torch.empty(Hl, M, dtype=torch.int32, device=dev), torch.empty(Hl, M, M, dtype=torch.int32, device=dev))
    _check_out(cfg, out)
    kstar, budget, cnt, idx = out
    _check(lib().proxyattn_avgpool_estimate(_cfg_ref(cfg), _tptr(Q, cfg), _tptr(K, cfg, "kv"), _ptr(workspace),
                                            workspace.numel(), _ptr(kstar), _ptr(budget), _ptr(cnt), _ptr(idx),
                                            _stream(dev)))
    return kstar, budget, cnt, idx


def cost_ratio(cfg: Config) -> float:
    return lib().proxyattn_cost_ratio(_cfg_ref(cfg))


def build_info() -> str:
    return lib().proxyattn_build_info().decode()


def debug_umma(A: torch.Tensor, B: torch.Tensor):
    """proxyattn_debug_umma -> (C_ss = A B^T, C_ts = A B), fp32 [128][128]."""
    Css = torch.empty(128, 128, dtype=torch.float32, device=A.device)
    Cts = torch.empty_like(Css)
    _check(lib().proxyattn_debug_umma(_ptr(A), _ptr(B), _ptr(Css), _ptr(Cts), _stream(A.device)))
    return Css, Cts


def _local_groups(cfg: Config) -> int:
    b, e = cfg.local_heads
    gq = cfg.n_q_heads // cfg.n_groups
    return (e - 1) // gq - b // gq + 1
