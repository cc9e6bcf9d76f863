"""In-place two-pass (no scratch) and the one-pass split at cfg5 size under planner knobs (dev tool)."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
R = C = int(os.environ.get("SIZE", 16384))
x = dev.synthetic((3, R, C), 1, 1)
scr = torch.zeros_like(x)
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
grid = [{}] + [{"SC_BAND_H": str(b), "SC_BAND_H2": str(b2)} for b, b2 in ((256, 32), (256, 64), (512, 64), (1024, 64))] + \
       [{"SC_NT": "256"}, {"SC_NT": "256", "SC_BAND_H": "256", "SC_BAND_H2": "64"}, {"SC_NS": "3"}, {"SC_NS": "5"}]
for kn in grid:
    for k, v in kn.items(): os.environ[k] = v
    r = {"knobs": kn, "inplace_ms": round(t(lambda: dev.two_pass_inplace(x, w)), 4),
         "split_ms": round(t(lambda: dev.two_pass_split(x, scr, w)), 4)}
    for k in kn: os.environ.pop(k)
    print(json.dumps(r), flush=True)
