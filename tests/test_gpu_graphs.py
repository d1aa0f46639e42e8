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
