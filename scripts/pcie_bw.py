"""PCIe copy rates on the box: H2D of the layer's Q/K/V (1.61 GB, pinned), D2H of O (1.07 GB),
alone and concurrently (two streams), and H2D of Q as 2-D per-head chunks (the host path's copies)."""
import json
import time

import torch

dev = torch.device("cuda:0")
Qh = torch.empty(32, 131072, 128, dtype=torch.bfloat16).pin_memory()
Kh = torch.empty(8, 131072, 128, dtype=torch.bfloat16).pin_memory()
Vh = torch.empty_like(Kh).pin_memory()
Oh = torch.empty_like(Qh).pin_memory()
Qd, Kd, Vd, Od = (torch.empty(t.shape, dtype=t.dtype, device=dev) for t in (Qh, Kh, Vh, Qh))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def wall(fn, it=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / it * 1e3


def h2d():
    with torch.cuda.stream(s1):
        Qd.copy_(Qh, non_blocking=True); Kd.copy_(Kh, non_blocking=True); Vd.copy_(Vh, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        Oh.copy_(Od, non_blocking=True)


def both():
    h2d(); d2h()


def h2d_chunks(n=16):
    with torch.cuda.stream(s1):
        Kd.copy_(Kh, non_blocking=True); Vd.copy_(Vh, non_blocking=True)
        c = 131072 // n
        for i in range(n):
            Qd[:, i * c:(i + 1) * c].copy_(Qh[:, i * c:(i + 1) * c], non_blocking=True)


r = {"h2d_1.61GB_ms": wall(h2d), "d2h_1.07GB_ms": wall(d2h), "both_concurrent_ms": wall(both),
     "h2d_2d_chunks16_ms": wall(h2d_chunks)}
r["h2d_GBps"] = 1.61e9 / (r["h2d_1.61GB_ms"] * 1e-3) / 1e9
r["d2h_GBps"] = 1.07e9 / (r["d2h_1.07GB_ms"] * 1e-3) / 1e9
print(json.dumps(r))
