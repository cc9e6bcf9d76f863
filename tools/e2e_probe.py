"""PCIe ceilings vs the host streaming path (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R = C = 16384; P = 3
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
host = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
for h in host: h.uniform_()
d = torch.empty((P, R, C), device="cuda")
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3
h2d = t(lambda: [d[p].copy_(host[p], non_blocking=True) for p in range(P)])
d2h = t(lambda: [host[p].copy_(d[p], non_blocking=True) for p in range(P)])
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
hb = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
def both():
    with torch.cuda.stream(s1):
        for p in range(P): d[p].copy_(host[p], non_blocking=True)
    with torch.cuda.stream(s2):
        for p in range(P): hb[p].copy_(d[p], non_blocking=True)
bidir = t(both)
res = {"h2d_ms": round(h2d, 2), "h2d_GBps": round(P*R*C*4/h2d/1e6, 1), "d2h_ms": round(d2h, 2),
       "d2h_GBps": round(P*R*C*4/d2h/1e6, 1), "bidir_ms": round(bidir, 2)}
for mb in (8, 16, 32, 64, 128, 256):
    os.environ["SC_HOST_CHUNK_MB"] = str(mb)
    res[f"e2e_{mb}MB_ms"] = round(t(lambda: dev.two_pass_host(host, host, w)), 2)
print(json.dumps(res))
