"""GPU: the estimate + prefill step (and the packed varlen forward) captured into CUDA graphs
and replayed on NEW input values — the way bench.py times the step and a serving loop would
run it.  The calls are asynchronous and capturable once warmed up on the capture stream
(include/proxyattn.h: the first call on a stream allocates its scheduler buffers); a replay
must equal the eager calls on the same values bit for bit."""
import pytest
import torch

import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


@pytest.mark.parametrize("d,b", [(128, 128), (128, 64), (64, 128)])
def test_graph_replay_equals_eager(d, b):
    N = 4096 + 77
    cfg = pa.Config(8, 2, d, N, b, 4, 1, 0.9)
    ws = pa.alloc_workspace(cfg, DEV)
    inputs = [workloads.structured(8, 2, N, d, seed=500 + k, device=DEV)[:3] for k in range(3)]
    Q, K, V = (t.clone() for t in inputs[0])                   # the graph's static inputs
    out = (torch.empty(8, dtype=torch.int32, device=DEV), torch.empty(8, device=DEV),
           torch.empty(8, cfg.M, dtype=torch.int32, device=DEV),
           torch.empty(8, cfg.M, cfg.M, dtype=torch.int32, device=DEV))
    O = torch.empty_like(Q)

    def step():
        pa.estimate(cfg, Q, K, workspace=ws, out=out)
        pa.prefill(cfg, Q, K, V, out[2], out[3], O)
    s = torch.cuda.Stream(DEV)
    s.wait_stream(torch.cuda.current_stream(DEV))
    with torch.cuda.stream(s):
        step()                                                  # warm-up on the capture stream
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
    torch.cuda.synchronize()
    for Qn, Kn, Vn in inputs[1:] + inputs[:1]:
        Q.copy_(Qn), K.copy_(Kn), V.copy_(Vn)
        g.replay()
        torch.cuda.synchronize()
        kstar, _, cnt, idx = pa.estimate(cfg, Qn, Kn)
        Oe = pa.prefill(cfg, Qn, Kn, Vn, cnt, idx)
        assert torch.equal(out[0], kstar) and torch.equal(out[2], cnt)
        for h in range(8):
            for m in range(cfg.M):
                c = int(cnt[h, m])
                assert torch.equal(out[3][h, m, :c], idx[h, m, :c]), (h, m)
        assert torch.equal(O, Oe)


def test_graph_replay_varlen():
    lens = [1500, 0, 2300, 640]
    cu = [0, 1500, 1500, 3800, 4440]
    cfg = pa.Config(8, 2, 128, 1, 128, 4, 1, 0.9, token_major=True)
    total = cu[-1]

    def packed(seed):
        seqs = [workloads.structured(8, 2, n, 128, seed=seed + i, device=DEV) for i, n in enumerate(lens) if n]
        return [torch.cat([x[j].transpose(0, 1) for x in seqs], 0).contiguous() for j in range(3)]
    Q, K, V = packed(600)
    ws = torch.empty(pa.varlen_workspace_bytes(cfg, cu), dtype=torch.uint8, device=DEV)
    O = torch.empty_like(Q)
    kstar = torch.zeros(len(lens), 8, dtype=torch.int32, device=DEV)
    s = torch.cuda.Stream(DEV)
    s.wait_stream(torch.cuda.current_stream(DEV))
    with torch.cuda.stream(s):
        pa.forward_varlen(cfg, cu, Q, K, V, O, ws, kstar)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            pa.forward_varlen(cfg, cu, Q, K, V, O, ws, kstar)
    torch.cuda.synchronize()
    Qn, Kn, Vn = packed(700)
    assert Qn.shape[0] == total
    Q.copy_(Qn), K.copy_(Kn), V.copy_(Vn)
    g.replay()
    torch.cuda.synchronize()
    Oe, ke = pa.forward_varlen(cfg, cu, Qn, Kn, Vn)
    assert torch.equal(kstar, ke) and torch.equal(O, Oe)


@pytest.mark.parametrize("b", [128, 64])
def test_graph_survives_a_larger_launch_on_its_stream(b):
    # a graph captured at a small size keeps the scheduler arrays of its
    # stream in its kernel parameters; a later, LARGER eager launch on the same stream must
    # not free them (the library retires, never frees, superseded arrays).  Capture small,
    # run large eagerly on the capture stream, replay small: equal to eager small.
    d = 128
    small = pa.Config(8, 2, d, 2048 + 77, b, 4, 1, 0.9)
    large = pa.Config(8, 2, d, 16384, b, 4, 1, 0.9)
    Qs, Ks, Vs, _ = workloads.structured(8, 2, small.seq_len, d, seed=801, device=DEV)
    Ql, Kl, Vl, _ = workloads.structured(8, 2, large.seq_len, d, seed=802, device=DEV)
    ws = pa.alloc_workspace(small, DEV)
    out = (torch.empty(8, dtype=torch.int32, device=DEV), torch.empty(8, device=DEV),
           torch.empty(8, small.M, dtype=torch.int32, device=DEV),
           torch.empty(8, small.M, small.M, dtype=torch.int32, device=DEV))
    O = torch.empty_like(Qs)
    s = torch.cuda.Stream(DEV)
    s.wait_stream(torch.cuda.current_stream(DEV))

    def step():
        pa.estimate(small, Qs, Ks, workspace=ws, out=out)
        pa.prefill(small, Qs, Ks, Vs, out[2], out[3], O)
    with torch.cuda.stream(s):
        step()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        kl, _, cl, il = pa.estimate(large, Ql, Kl)          # grows the stream's arrays
        Ol = pa.prefill(large, Ql, Kl, Vl, cl, il)
        junk = torch.full((64 << 20,), -1, dtype=torch.int32, device=DEV)   # reuse freed memory
        O.zero_()
        g.replay()
    torch.cuda.synchronize()
    del junk
    kstar, _, cnt, idx = pa.estimate(small, Qs, Ks)
    Oe = pa.prefill(small, Qs, Ks, Vs, cnt, idx)
    torch.cuda.synchronize()
    assert torch.equal(out[0], kstar) and torch.equal(out[2], cnt)
    assert torch.equal(O, Oe)
    assert torch.isfinite(Ol.float()).all()


def test_capture_while_another_thread_runs_eagerly():
    # library helper streams are per (device, caller stream), so an eager call on
    # another thread's stream is never recorded into this thread's capture
    import threading
    cfg = pa.Config(8, 2, 128, 4096, 128, 4, 1, 0.9)
    Q, K, V, _ = workloads.structured(8, 2, 4096, 128, seed=811, device=DEV)
    Q2, K2, V2, _ = workloads.structured(8, 2, 4096, 128, seed=812, device=DEV)
    ref2 = pa.prefill(cfg, Q2, K2, V2, *pa.estimate(cfg, Q2, K2)[2:])
    ws, ws2 = pa.alloc_workspace(cfg, DEV), pa.alloc_workspace(cfg, DEV)
    out = (torch.empty(8, dtype=torch.int32, device=DEV), torch.empty(8, device=DEV),
           torch.empty(8, cfg.M, dtype=torch.int32, device=DEV),
           torch.empty(8, cfg.M, cfg.M, dtype=torch.int32, device=DEV))
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    with torch.cuda.stream(s2):                              # warm both streams' library state
        pa.prefill(cfg, Q2, K2, V2, *pa.estimate(cfg, Q2, K2, workspace=ws2)[2:])
    with torch.cuda.stream(s1):
        pa.estimate(cfg, Q, K, workspace=ws, out=out)
    torch.cuda.synchronize()
    got, errs = [], []
    go = threading.Event()

    def eager():
        try:
            with torch.cuda.stream(s2):
                go.wait()
                for _ in range(20):
                    k2, _, c2, i2 = pa.estimate(cfg, Q2, K2, workspace=ws2)
                    got.append(pa.prefill(cfg, Q2, K2, V2, c2, i2))
            s2.synchronize()
        except Exception as e:
            errs.append(e)
    th = threading.Thread(target=eager)
    th.start()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s1):
        with torch.cuda.graph(g, stream=s1, capture_error_mode="thread_local"):
            go.set()
            for _ in range(5):
                pa.estimate(cfg, Q, K, workspace=ws, out=out)
    th.join()
    assert not errs, errs
    g.replay()
    torch.cuda.synchronize()
    assert all(torch.equal(o, ref2) for o in got)
    assert torch.equal(out[0], pa.estimate(cfg, Q, K)[0])
