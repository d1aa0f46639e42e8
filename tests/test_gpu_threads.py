"""GPU: the C-ABI called from several host threads at once, each on its own CUDA stream with
its own inputs and workspace (a serving process runs layers of different requests
concurrently).  The library's static state — the per-stream scheduler buffers of the
attention launch, the per-device Alg. 1 side stream, the thread-local fork / join events and
error string — must keep every thread's results equal, bit for bit, to the same calls made
sequentially."""
import threading

import pytest
import torch

import paper_2509_24745_b200 as pa
import workloads

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda:0") if torch.cuda.is_available() else None


def layer(cfg, Q, K, V, ws):
    kstar, budget, cnt, idx = pa.estimate(cfg, Q, K, workspace=ws)
    return kstar, cnt, idx, pa.prefill(cfg, Q, K, V, cnt, idx)


def test_concurrent_threads_match_sequential():
    shapes = [(128, 128, 4096 + 77), (64, 128, 3000), (128, 64, 2500), (64, 64, 2049)]
    cases = []
    for t, (d, b, N) in enumerate(shapes):
        cfg = pa.Config(8, 2, d, N, b, 4, 1, 0.9)
        Q, K, V, _ = workloads.structured(8, 2, N, d, seed=400 + t, device=DEV)
        cases.append((cfg, Q, K, V, pa.alloc_workspace(cfg, DEV)))
    ref = [layer(*c) for c in cases]
    torch.cuda.synchronize()
    got = [None] * len(cases)
    errors = []
    barrier = threading.Barrier(len(cases))

    def run(t):
        try:
            s = torch.cuda.Stream(device=DEV)
            with torch.cuda.stream(s):
                barrier.wait()
                for _ in range(3):                  # repeated: interleave with the others
                    got[t] = layer(*cases[t])
            s.synchronize()
        except Exception as e:                      # surfaced below
            errors.append((t, e))
    threads = [threading.Thread(target=run, args=(t,)) for t in range(len(cases))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for t, (r, g) in enumerate(zip(ref, got)):
        kr, cr, ir, Or = r
        kg, cg, ig, Og = g
        assert torch.equal(kr, kg) and torch.equal(cr, cg), t
        M = cases[t][0].M
        for h in range(8):
            for m in range(M):
                c = int(cr[h, m])
                assert torch.equal(ir[h, m, :c], ig[h, m, :c]), (t, h, m)
        assert torch.equal(Or, Og), t
