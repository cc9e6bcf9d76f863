"""Two-pass and single pass at kernel widths 5..63 (dev tool): widths 1..9 run the tuned
row-streaming kernels, wider ones the plain kernels of kern_wide.cu."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R = C = int(os.environ.get("SIZE", 8192))
x = dev.synthetic((3, R, C), 1, 1)
y = torch.empty_like(x)
def t(fn, n=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
FP = 126.7 * 148 * 1.965e9
for W in (5, 9, 11, 13, 15, 21, 25, 31, 33, 63):
    w = np.random.default_rng(W).standard_normal(W).astype(np.float32)
    ms = t(lambda: dev.two_pass(x, w, y))
    ops = 3 * R * C * 2 * (2 * W - 1)
    rec = {"W": W, "two_pass_ms": round(ms, 4), "hbm_floor_ms": round(24 * R * C / 6535.7e6, 4), "fp32_floor_ms": round(ops / FP * 1e3, 4)}
    if W <= 15 or W == 31:
        k = np.outer(w, w).astype(np.float32)
        ms1 = t(lambda: dev.single_pass(x, k, y), n=3)
        rec["single_ms"] = round(ms1, 4)
        rec["single_fp32_floor_ms"] = round(3 * R * C * (2 * W * W - 1) / FP * 1e3, 4)
    print(json.dumps(rec), flush=True)
