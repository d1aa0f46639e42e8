"""Small cases covering every kernel of the library, for compute-sanitizer.

    compute-sanitizer --tool memcheck|synccheck|racecheck|initcheck python scripts/sanitize_cases.py

Each case runs the estimate (A1-A6), the block-sparse prefill (A7) and the dense prefill (A8)
on a short ragged sequence and synchronises, so an error is attributed to its case.  Covered:
the fp32 debug path, the bf16 tensor-core shapes d x b in {64, 128}^2, GQA ratios with an
odd head count (b = 64 pairs with one head), token-major layouts, a zig-zag row range with
kstar given, scores-only + select_ws, method variants, the varlen packed launch and the
pipelined host path, the seq-avgpool comparator and the CHECK_FINITE scan.  No oracle: this checks memory safety, not values (the parity tests do).
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2509_24745_b200 as pa  # noqa: E402
import workloads  # noqa: E402

DEV = torch.device("cuda:0")


def tok(t):
    return t.transpose(0, 1).contiguous()


def layer(cfg, Q, K, V):
    ks, bu, cnt, idx = pa.estimate(cfg, Q, K)
    O = pa.prefill(cfg, Q, K, V, cnt, idx)
    Od = pa.dense_prefill(cfg, Q, K, V)
    torch.cuda.synchronize()
    return ks, cnt, idx, O, Od


def case(name, fn):
    fn()
    torch.cuda.synchronize()
    print("ok", name, flush=True)


def main():
    N = 777                                                     # ragged: partial last block
    for d, b in [(128, 128), (64, 128), (128, 64), (64, 64)]:
        for Hq, Hkv, g in [(8, 2, 1), (7, 1, 1), (8, 4, 2)]:
            def f(d=d, b=b, Hq=Hq, Hkv=Hkv, g=g):
                Q, K, V, _ = workloads.structured(Hq, Hkv, N, d, seed=d + b + Hq, device=DEV)
                layer(pa.Config(Hq, Hkv, d, N, b, 4, g, 0.9), Q, K, V)
            case(f"bf16 d={d} b={b} heads={Hq}/{Hkv} g={g}", f)

    def fp32():
        Q, K, V = (t.to(DEV) for t in workloads.iid(8, 2, 300, 64, seed=1))
        layer(pa.Config(8, 2, 64, 300, 64, 4, 2, 0.9, fp32_debug=True), Q, K, V)
    case("fp32 debug", fp32)

    def token_major():
        Q, K, V, _ = workloads.structured(8, 2, N, 128, seed=3, device=DEV)
        layer(pa.Config(8, 2, 128, N, 128, 4, 1, 0.9, token_major=True), tok(Q), tok(K), tok(V))
    case("token-major", token_major)

    def row_range():
        from paper_2509_24745_b200 import shard
        Q, K, V, _ = workloads.structured(8, 2, 1500, 128, seed=4, device=DEV)
        cfg = pa.Config(8, 2, 128, 1500, 128, 4, 1, 0.9)
        ks, bu, cnt, idx = pa.estimate(cfg, Q, K)
        rows = shard.zigzag_rows(cfg.M, 3, 1)
        wss = [pa.alloc_workspace(cfg, DEV), pa.alloc_workspace(cfg, DEV)]
        out = (ks.clone(), bu.clone(), torch.zeros_like(cnt), torch.zeros_like(idx))
        shard.estimate_rows(cfg, Q, K, rows, out=out, kstar_given=True, scores_only=True,
                            streams=[torch.cuda.Stream(), torch.cuda.Stream()], workspaces=wss)
        torch.cuda.synchronize()
        shard.select_rows(cfg, rows, wss, out[0], (out[2], out[3]))
        for r0, r1 in rows:
            pa.prefill(cfg.replace(row_begin=r0, row_end=r1), Q, K, V, out[2], out[3])
    case("row ranges: scores only, select_ws, row-range prefill", row_range)

    for v in [dict(force_sink=True), dict(constant_k=True), dict(designated_head=True),
              dict(static_kstar=3)]:
        def f(v=v):
            Q, K, V, _ = workloads.structured(8, 2, N, 128, seed=6, device=DEV)
            layer(pa.Config(8, 2, 128, N, 128, 4, 1, 0.9, **v), Q, K, V)
        case(f"variant {v}", f)

    def varlen():
        lens = [300, 0, 1100, 64]
        seqs = [workloads.structured(8, 2, n, 128, seed=7 + i, device=DEV) for i, n in enumerate(lens) if n]
        packed = [torch.cat([tok(s[j]) for s in seqs], 0) for j in range(3)]
        cu = [0]
        for n in lens:
            cu.append(cu[-1] + n)
        pa.forward_varlen(pa.Config(8, 2, 128, 1, 128, 4, 1, 0.9, token_major=True), cu, *packed)
    case("varlen packed", varlen)

    def avgpool():                                              # the seq-avgpool comparator (round 2)
        for d, b in [(128, 128), (64, 64)]:
            Q, K, V, _ = workloads.structured(8, 2, N, d, seed=9 + d, device=DEV)
            cfg = pa.Config(8, 2, d, N, b, 4, 1, 0.9)
            pa.avgpool_scores(cfg, Q, K)
            pa.avgpool_estimate(cfg, Q, K)
    case("seq-avgpool comparator scores + estimate", avgpool)

    def check_finite():                                         # CHECK_FINITE scan, then a NaN (round 2)
        Q, K, V, _ = workloads.structured(8, 2, N, 128, seed=10, device=DEV)
        cfg = pa.Config(8, 2, 128, N, 128, 4, 1, 0.9, check_finite=True)
        layer(cfg, Q, K, V)
        Q[3, 100, 5] = float("nan")
        try:
            pa.estimate(cfg, Q, K)
        except Exception:
            pass
        else:
            raise AssertionError("NaN input not rejected")
    case("CHECK_FINITE scan and rejection", check_finite)

    def host():
        cfg = pa.Config(8, 2, 128, 1000, 128, 4, 1, 0.9)
        Q, K, V, _ = workloads.structured(8, 2, 1000, 128, seed=8, device=DEV)
        Qh, Kh, Vh = (t.cpu().pin_memory() for t in (Q, K, V))
        Oh = torch.empty_like(Qh).pin_memory()
        ws = torch.empty(pa.forward_host_workspace_bytes(cfg), dtype=torch.uint8, device=DEV)
        pa.forward_host(cfg, Qh, Kh, Vh, Oh, ws)
    case("forward_host", host)
    print("all cases ok")


if __name__ == "__main__":
    main()
