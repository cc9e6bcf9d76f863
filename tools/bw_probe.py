"""Bandwidth probes (dev tool): memcpy, torch elementwise, our pipeline at W=1/3/5."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R, C, P = 16384, 16384, 3
x = dev.synthetic((P, R, C), 5, 1)
y = torch.empty_like(x)
alg = 2 * 4 * P * R * C
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts))
res = {}
res["memcpy"] = t(lambda: y.copy_(x))
res["torch_mul"] = t(lambda: torch.mul(x, 1.0, out=y))
w1 = np.array([1.0], np.float32); w3 = np.array([0.25, 0.5, 0.25], np.float32); w5 = np.array([1,4,6,4,1], np.float32) / 16
res["vpass_w1"] = t(lambda: dev.vpass(x, w1, y))
res["hpass_w1"] = t(lambda: dev.hpass(x, w1, y))
res["vpass_w5"] = t(lambda: dev.vpass(x, w5, y))
res["hpass_w5"] = t(lambda: dev.hpass(x, w5, y))
res["fused_w1"] = t(lambda: dev.two_pass(x, w1, y))
res["fused_w5"] = t(lambda: dev.two_pass(x, w5, y))
for k, v in res.items():
    print(json.dumps({"op": k, "ms": round(v, 4), "GBps": round(alg / v / 1e6, 1)}))
