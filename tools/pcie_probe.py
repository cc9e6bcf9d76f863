import time, json, torch
R = C = 16384; P = 3
host = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
hb = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
d = torch.empty((P, R, C), device="cuda"); d2 = torch.empty_like(d)
def t(fn, n=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / n * 1e3, 2)
res = {}
for ns in (1, 2, 4):
    hs = [torch.cuda.Stream() for _ in range(ns)]; ds = [torch.cuda.Stream() for _ in range(ns)]
    CH = 512
    def both():
        k = 0
        for p in range(P):
            for r0 in range(0, R, CH):
                with torch.cuda.stream(hs[k % ns]):
                    d[p, r0:r0+CH].copy_(host[p][r0:r0+CH], non_blocking=True)
                with torch.cuda.stream(ds[k % ns]):
                    hb[p][r0:r0+CH].copy_(d2[p, r0:r0+CH], non_blocking=True)
                k += 1
    def h2d_only():
        k = 0
        for p in range(P):
            for r0 in range(0, R, CH):
                with torch.cuda.stream(hs[k % ns]):
                    d[p, r0:r0+CH].copy_(host[p][r0:r0+CH], non_blocking=True)
                k += 1
    res[f"bidir_{ns}streams_ms"] = t(both)
    res[f"h2d_{ns}streams_ms"] = t(h2d_only)
print(json.dumps(res))
