"""Fused PPM payload kernel (u8 HWC read -> two-pass -> u8 write) timing (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096,16384").split(",")]:
    x = torch.randint(0, 256, (n, n, 3), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3): dev.two_pass_u8hwc(x, w, y)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): dev.two_pass_u8hwc(x, w, y)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 10
    print(json.dumps({"n": n, "ms": round(ms, 4), "Gpix_s": round(n * n / ms / 1e6, 1), "GBps": round(6 * n * n / ms / 1e6, 1)}))
