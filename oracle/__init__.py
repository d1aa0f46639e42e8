"""ctypes binding of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2509_24745_b200``) never imports it and shares no code with it.

Every function mirrors one step of SURVEY.md §8(c) (O1-O10), which follows
PAPER.md Eq. 1-3 and Alg. 1.  Arrays are numpy; inputs Q/K/V are float32
``[H][N][d]`` (bf16 values upcast exactly), outputs are float64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, IEEE semantics, OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
             _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _SO)
    return _SO


class _CCfg(ctypes.Structure):
    _fields_ = [
        ("n_q_heads", ctypes.c_int32),
        ("n_kv_heads", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("seq_len", ctypes.c_int64),
        ("block_size", ctypes.c_int32),
        ("stride", ctypes.c_int32),
        ("n_groups", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("min_budget_tokens", ctypes.c_int32),
        ("round_bf16", ctypes.c_int32),
        ("force_sink", ctypes.c_int32),
        ("constant_k", ctypes.c_int32),
        ("designated_head", ctypes.c_int32),
        ("static_kstar", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class Cfg:
    """AttnConfig."""

    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    seq_len: int
    block_size: int
    stride: int
    n_groups: int
    gamma: float
    min_budget_tokens: int = 0
    round_bf16: bool = False
    force_sink: bool = False        # method variants
    constant_k: bool = False
    designated_head: bool = False
    static_kstar: int = 0

    @property
    def M(self) -> int:
        return -(-self.seq_len // self.block_size)      # ceil: the last block may be padded

    @property
    def Ns(self) -> int:
        return -(-self.seq_len // self.stride)

    def c(self) -> _CCfg:
        return _CCfg(self.n_q_heads, self.n_kv_heads, self.head_dim, self.seq_len,
                     self.block_size, self.stride, self.n_groups, float(self.gamma),
                     self.min_budget_tokens, int(bool(self.round_bf16)), int(bool(self.force_sink)),
                     int(bool(self.constant_k)), int(bool(self.designated_head)),
                     int(self.static_kstar))

    def replace(self, **kw) -> "Cfg":
        d = dict(self.__dict__)
        d.update(kw)
        return Cfg(**d)


_lib = None
_P = ctypes.c_void_p


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        cp = ctypes.POINTER(_CCfg)
        L.oracle_validate.argtypes = [cp]
        L.oracle_validate.restype = ctypes.c_int
        L.oracle_rne_bf16.argtypes = [ctypes.c_double]
        L.oracle_rne_bf16.restype = ctypes.c_double
        L.oracle_group_of_q.argtypes = [cp, ctypes.c_int]
        L.oracle_group_of_q.restype = ctypes.c_int
        L.oracle_pool.argtypes = [cp, _P, _P, _P, _P, ctypes.POINTER(ctypes.c_double)]
        L.oracle_pool.restype = None
        L.oracle_proxy_scores.argtypes = [cp, _P, _P, ctypes.c_double, _P, ctypes.c_int, _P, _P]
        L.oracle_proxy_scores.restype = None
        L.oracle_budget_from_mass.argtypes = [_P, ctypes.c_int, ctypes.c_double,
                                              ctypes.POINTER(ctypes.c_double)]
        L.oracle_budget_from_mass.restype = ctypes.c_int
        L.oracle_budgets.argtypes = [cp, _P, _P, _P, ctypes.c_int, _P, _P, _P, _P]
        L.oracle_budgets.restype = None
        L.oracle_row_count.argtypes = [cp, ctypes.c_int, ctypes.c_int]
        L.oracle_row_count.restype = ctypes.c_int
        L.oracle_select.argtypes = [cp, _P, _P, _P, ctypes.c_int, _P, _P, _P]
        L.oracle_select.restype = None
        L.oracle_attention.argtypes = [cp, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P]
        L.oracle_attention.restype = None
        L.oracle_dense.argtypes = [cp, _P, _P, _P, _P, ctypes.c_int, _P]
        L.oracle_dense.restype = None
        L.oracle_cost_ratio.argtypes = [cp]
        L.oracle_cost_ratio.restype = ctypes.c_double
        L.oracle_num_threads.argtypes = []
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        L.oracle_set_num_threads.restype = None
        L.oracle_seq_avgpool_scores.argtypes = [cp, _P, _P, _P]
        L.oracle_seq_avgpool_scores.restype = None
        L.oracle_select_heads.argtypes = [cp, _P, _P, _P, _P, _P]
        L.oracle_select_heads.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32))


def _i32(a) -> np.ndarray | None:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _items(items) -> np.ndarray | None:
    """(head, block row) pairs as an [n][2] int32 array (accepts flat or paired input)."""
    if items is None:
        return None
    return np.ascontiguousarray(np.asarray(items, dtype=np.int32).reshape(-1, 2))


def validate(cfg: Cfg) -> bool:
    c = cfg.c()
    return lib().oracle_validate(ctypes.byref(c)) == 0


def _check(cfg: Cfg) -> _CCfg:
    c = cfg.c()
    if lib().oracle_validate(ctypes.byref(c)) != 0:
        raise ValueError(f"invalid config {cfg}")
    return c


def rne_bf16(x: float) -> float:
    return lib().oracle_rne_bf16(float(x))


def group_of_q(cfg: Cfg, h: int) -> int:
    c = _check(cfg)
    return lib().oracle_group_of_q(ctypes.byref(c), h)


def pool(cfg: Cfg, Q, K):
    """O3: pooled sums Pq, Pk [g][N/s][d] (bf16-rounded when cfg.round_bf16) and the scale."""
    c = _check(cfg)
    Q, K = _f32(Q), _f32(K)
    assert Q.shape == (cfg.n_q_heads, cfg.seq_len, cfg.head_dim)
    assert K.shape == (cfg.n_kv_heads, cfg.seq_len, cfg.head_dim)
    Pq = np.zeros((cfg.n_groups, cfg.Ns, cfg.head_dim), np.float64)
    Pk = np.zeros_like(Pq)
    sc = ctypes.c_double(0.0)
    lib().oracle_pool(ctypes.byref(c), _ptr(Q), _ptr(K), _ptr(Pq), _ptr(Pk), ctypes.byref(sc))
    return Pq, Pk, sc.value


def proxy_scores(cfg: Cfg, Pq, Pk, scale: float, rows=None):
    """O4-O6: (lse [g][Ns], L [g][M][M]).  With ``rows`` only those block rows are computed
    (others stay NaN; lse is valid only for sampled rows inside the listed block rows)."""
    c = _check(cfg)
    Pq = np.ascontiguousarray(Pq, np.float64)
    Pk = np.ascontiguousarray(Pk, np.float64)
    r = _i32(rows)
    lse = np.full((cfg.n_groups, cfg.Ns), np.nan)
    L = np.full((cfg.n_groups, cfg.M, cfg.M), np.nan)
    lib().oracle_proxy_scores(ctypes.byref(c), _ptr(Pq), _ptr(Pk), float(scale), _ptr(r),
                              0 if r is None else len(r), _ptr(lse), _ptr(L))
    return lse, L


def budget_from_mass(a, gamma: float):
    a = np.ascontiguousarray(a, np.float64)
    mg = ctypes.c_double(0.0)
    k = lib().oracle_budget_from_mass(_ptr(a), len(a), float(gamma), ctypes.byref(mg))
    return k, mg.value


def budgets(cfg: Cfg, Q, K, heads=None):
    """O7: (kstar [Hq] int32, budget [Hq], margin [Hq], mass [Hq][M]); unlisted heads = -1/NaN."""
    c = _check(cfg)
    Q, K = _f32(Q), _f32(K)
    hs = _i32(heads)
    H, M = cfg.n_q_heads, cfg.M
    kstar = np.full(H, -1, np.int32)
    budget = np.full(H, np.nan)
    margin = np.full(H, np.nan)
    mass = np.full((H, M), np.nan)
    lib().oracle_budgets(ctypes.byref(c), _ptr(Q), _ptr(K), _ptr(hs), 0 if hs is None else len(hs),
                         _ptr(kstar), _ptr(budget), _ptr(margin), _ptr(mass))
    return kstar, budget, margin, mass


def row_count(cfg: Cfg, kstar: int, m: int) -> int:
    c = _check(cfg)
    return lib().oracle_row_count(ctypes.byref(c), int(kstar), int(m))


def select(cfg: Cfg, L, kstar, rows=None):
    """O9: (block_cnt [Hq][M], block_idx [Hq][M][M] (-1 padded), cut_margin [Hq][M])."""
    c = _check(cfg)
    L = np.ascontiguousarray(L, np.float64)
    ks = _i32(kstar)
    r = _i32(rows)
    H, M = cfg.n_q_heads, cfg.M
    cnt = np.zeros((H, M), np.int32)
    idx = np.full((H, M, M), -1, np.int32)
    mg = np.full((H, M), np.nan)
    lib().oracle_select(ctypes.byref(c), _ptr(L), _ptr(ks), _ptr(r), 0 if r is None else len(r),
                        _ptr(cnt), _ptr(idx), _ptr(mg))
    return cnt, idx, mg


def attention(cfg: Cfg, Q, K, V, block_cnt, block_idx, items=None):
    """O10: block-sparse causal attention; O [Hq][N][d] float64 (NaN for rows not listed)."""
    c = _check(cfg)
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    cnt = _i32(block_cnt)
    idx = _i32(block_idx)
    it = _items(items)
    O = np.full((cfg.n_q_heads, cfg.seq_len, cfg.head_dim), np.nan)
    lib().oracle_attention(ctypes.byref(c), _ptr(Q), _ptr(K), _ptr(V), _ptr(cnt), _ptr(idx),
                           _ptr(it), 0 if it is None else len(it), _ptr(O))
    return O


def dense(cfg: Cfg, Q, K, V, items=None):
    """Dense causal attention = O10 with every causal block."""
    c = _check(cfg)
    Q, K, V = _f32(Q), _f32(K), _f32(V)
    it = _items(items)
    O = np.full((cfg.n_q_heads, cfg.seq_len, cfg.head_dim), np.nan)
    lib().oracle_dense(ctypes.byref(c), _ptr(Q), _ptr(K), _ptr(V), _ptr(it),
                       0 if it is None else len(it), _ptr(O))
    return O


def cost_ratio(cfg: Cfg) -> float:
    c = _check(cfg)
    return lib().oracle_cost_ratio(ctypes.byref(c))


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def seq_avgpool_scores(cfg: Cfg, Q, K):
    """O11: the seq-avgpool comparator's per-head log-domain block scores S [Hq][M][M]
    (SPEC S:365-373), -inf above the diagonal."""
    c = _check(cfg)
    Q, K = _f32(Q), _f32(K)
    S = np.full((cfg.n_q_heads, cfg.M, cfg.M), np.nan)
    lib().oracle_seq_avgpool_scores(ctypes.byref(c), _ptr(Q), _ptr(K), _ptr(S))
    return S


def select_heads(cfg: Cfg, S, kstar):
    """O9 on per-head maps S [Hq][M][M]: (block_cnt, block_idx (-1 padded), cut_margin)."""
    c = _check(cfg)
    S = np.ascontiguousarray(S, np.float64)
    ks = _i32(kstar)
    H, M = cfg.n_q_heads, cfg.M
    cnt = np.zeros((H, M), np.int32)
    idx = np.full((H, M, M), -1, np.int32)
    mg = np.full((H, M), np.nan)
    lib().oracle_select_heads(ctypes.byref(c), _ptr(S), _ptr(ks), _ptr(cnt), _ptr(idx), _ptr(mg))
    return cnt, idx, mg


def avgpool_estimate(cfg: Cfg, Q, K):
    """The comparator end to end: O7 budgets (as the proxy path) + O11 scores + per-head O9."""
    S = seq_avgpool_scores(cfg, Q, K)
    kstar, budget, bmargin, mass = budgets(cfg, Q, K)
    cnt, idx, cmargin = select_heads(cfg, S, kstar)
    return dict(S=S, kstar=kstar, budget=budget, budget_margin=bmargin, block_cnt=cnt,
                block_idx=idx, cut_margin=cmargin)


def estimate(cfg: Cfg, Q, K):
    """O1-O9 end to end: dict with Pq, Pk, scale, lse, L, kstar, budget, budget_margin,
    block_cnt, block_idx, cut_margin."""
    Pq, Pk, scale = pool(cfg, Q, K)
    lse, L = proxy_scores(cfg, Pq, Pk, scale)
    kstar, budget, bmargin, mass = budgets(cfg, Q, K)
    cnt, idx, cmargin = select(cfg, L, kstar)
    return dict(Pq=Pq, Pk=Pk, scale=scale, lse=lse, L=L, kstar=kstar, budget=budget,
                budget_margin=bmargin, mass=mass, block_cnt=cnt, block_idx=idx,
                cut_margin=cmargin)


def pipeline(cfg: Cfg, Q, K, V):
    """O1-O10: the estimate plus the block-sparse output O."""
    est = estimate(cfg, Q, K)
    est["O"] = attention(cfg, Q, K, V, est["block_cnt"], est["block_idx"])
    return est


def sparsity(cfg: Cfg, block_cnt) -> float:
    """Block sparsity 1 - selected / causally valid, averaged over heads (Z20)."""
    M = cfg.M
    valid = M * (M + 1) / 2
    per_head = 1.0 - np.asarray(block_cnt).sum(axis=1) / valid
    return float(per_head.mean())
