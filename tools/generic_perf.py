import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
for (R, C) in ((4096, 4096), (4095, 4095), (4096, 4097), (8191, 8193), (16383, 16383)):
    x = dev.synthetic((3, R, C), 1, 1); y = torch.empty_like(x)
    ms = t(lambda: dev.two_pass(x, w, y))
    print(json.dumps({"R": R, "C": C, "ms": round(ms, 4), "GBps": round(24 * R * C / ms / 1e6, 1)}))
