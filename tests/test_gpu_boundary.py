"""GPU: the C-ABI's validation contract.  PROXYATTN_FLAG_CHECK_FINITE ("all values
finite"; S:49 / S:319 "non-finite input -> validation error") returns E_NONFINITE (-6) for a
NaN or Inf anywhere in Q, K or V, in both layouts, before anything else is enqueued; clean
inputs give the unflagged results bit for bit.  The binding rejects wrong dtypes, devices
and token strides (no silent misreads)."""
import pytest
import torch

import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


def inputs(N=2048, d=128, seed=31):
    Q, K, V, _ = workloads.structured(8, 2, N, d, seed=seed, device=DEV)
    return Q, K, V


@pytest.mark.parametrize("fp32", [False, True])
def test_check_finite_rejects_nan_and_inf(fp32):
    cfg = pa.Config(8, 2, 128, 2048, 128, 4, 1, 0.9, fp32_debug=fp32, check_finite=True)
    Q, K, V = inputs()
    if fp32:
        Q, K, V = Q.float(), K.float(), V.float()
    kstar, _, cnt, idx = pa.estimate(cfg, Q, K)                       # clean: accepted
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
    plain = cfg.replace(check_finite=False)
    k0, _, c0, i0 = pa.estimate(plain, Q, K)
    assert torch.equal(kstar, k0) and torch.equal(cnt, c0)
    assert torch.equal(O, pa.prefill(plain, Q, K, V, c0, i0))
    for name, t, pos, val in (("Q", Q, (3, 1000, 5), float("nan")), ("K", K, (1, 2047, 127), float("nan")),
                              ("K", K, (0, 0, 0), float("inf")), ("V", V, (1, 77, 64), float("-inf"))):
        bad = t.clone()
        bad[pos] = val
        args = dict(Q=Q, K=K, V=V)
        args[name] = bad
        if name != "V":
            for fn in (lambda: pa.estimate(cfg, args["Q"], args["K"]),
                       lambda: pa.budgets(cfg, args["Q"], args["K"]),
                       lambda: pa.pool(cfg, args["Q"], args["K"])):
                with pytest.raises(pa.ProxyAttnError) as ei:
                    fn()
                assert ei.value.code == pa._lib.E_NONFINITE == -6, name
        for fn in (lambda: pa.prefill(cfg, args["Q"], args["K"], args["V"], cnt, idx),
                   lambda: pa.dense_prefill(cfg, args["Q"], args["K"], args["V"])):
            with pytest.raises(pa.ProxyAttnError) as ei:
                fn()
            assert ei.value.code == -6, name
        assert "non-finite" in str(ei.value)


def test_check_finite_token_major_and_unflagged_is_silent():
    cfg = pa.Config(8, 2, 128, 1024 + 64, 128, 4, 1, 0.9)
    Q, K, V = inputs(N=1024 + 64)
    Qt, Kt, Vt = (x.transpose(0, 1).contiguous() for x in (Q, K, V))
    tcfg = pa.with_strides(cfg, Qt, Kt).replace(check_finite=True)
    pa.estimate(tcfg, Qt, Kt)
    bad = Kt.clone()
    bad[1087, 1, 3] = float("nan")                                  # last token, second kv head
    with pytest.raises(pa.ProxyAttnError) as ei:
        pa.estimate(tcfg, Qt, bad)
    assert ei.value.code == -6
    pa.estimate(tcfg.replace(check_finite=False), Qt, bad)           # unflagged: no validation


def test_binding_rejects_wrong_dtype_device_and_strides():
    cfg = pa.Config(8, 2, 128, 1024, 128, 4, 1, 0.9)
    Q, K, V = inputs(N=1024)
    with pytest.raises(ValueError):
        pa.estimate(cfg, Q.float(), K)                               # fp32 into a bf16 config
    with pytest.raises(ValueError):
        pa.estimate(cfg, Q.cpu(), K)                                 # host tensor
    # a head slice of a packed [N][H][d] activation passed without with_strides()
    packed = torch.cat([Q, Q], 0).transpose(0, 1).contiguous()       # [N][16][d] activation
    Qs = packed[:, :8]
    Kt = K.transpose(0, 1).contiguous()
    with pytest.raises(ValueError):
        pa.estimate(cfg.replace(token_major=True), Qs, Kt)
    pa.estimate(pa.with_strides(cfg, Qs, Kt), Qs, Kt)                # with the strides: fine
    out = (torch.empty(8, dtype=torch.int64, device=DEV), torch.empty(8, device=DEV),
           torch.empty(8, 8, dtype=torch.int32, device=DEV), torch.empty(8, 8, 8, dtype=torch.int32, device=DEV))
    with pytest.raises(ValueError):
        pa.estimate(cfg, Q, K, out=out)                              # wrong output dtype


def test_forward_host_rejects_check_finite():
    cfg = pa.Config(8, 2, 128, 1024, 128, 4, 1, 0.9, check_finite=True)
    Q, K, V = (x.cpu().pin_memory() for x in inputs(N=1024))
    ws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=DEV)
    with pytest.raises(pa.ProxyAttnError) as ei:
        pa.forward_host(cfg, Q, K, V, torch.empty_like(Q).pin_memory(), ws)
    assert ei.value.code == pa._lib.E_CONFIG
