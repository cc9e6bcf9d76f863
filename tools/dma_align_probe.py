"""Duplex (H2D + D2H at once) DMA rate on page-locked numpy memory vs the alignment of the HOST address (dev tool):
0 / 256 / 2048 bytes past a page boundary 49-50 GB/s each way, 16 / 64 bytes 43.6-44.1 (profiles/r02_dma_align.json)."""
import os, sys, json, time, ctypes
import numpy as np, torch
n = 16384 * 16384
cudart = ctypes.CDLL("libcudart.so.12")
def duplex(h_in, h_out, d_in, d_out, reps=5):
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream(); ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
        s1.synchronize(); s2.synchronize(); ts.append(time.perf_counter() - t0)
    return round(h_in.numel() * 4 / min(ts) / 1e9, 1)
d1 = torch.empty(n, dtype=torch.float32, device="cuda"); d2 = torch.empty(n, dtype=torch.float32, device="cuda")
res = {}
def aligned(off_bytes):
    raw = np.ones(n + (1 << 20), dtype=np.float32)
    base = raw.ctypes.data
    start = ((base + 4095) & ~4095) + off_bytes
    a = raw[(start - base) // 4:(start - base) // 4 + n]
    assert a.ctypes.data == start
    cudart.cudaHostRegister(ctypes.c_void_p(raw.ctypes.data), ctypes.c_size_t(raw.nbytes), ctypes.c_uint(1))
    return raw, a
for off in (0, 16, 64, 256, 2048):
    r1, a1 = aligned(off); r2, a2 = aligned(off)
    res[f"offset_{off}_ptr_mod_4096"] = [a1.ctypes.data % 4096, np.ones(8).ctypes.data % 4096]
    res[f"offset_{off}_duplex"] = duplex(torch.from_numpy(a1), torch.from_numpy(a2), d1, d2)
    cudart.cudaHostUnregister(ctypes.c_void_p(r1.ctypes.data)); cudart.cudaHostUnregister(ctypes.c_void_p(r2.ctypes.data))
    del r1, r2, a1, a2
b = np.ones(n, dtype=np.float32); res["plain_numpy_ptr_mod_4096"] = b.ctypes.data % 4096
print(json.dumps(res))
