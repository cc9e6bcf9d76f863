import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
R = C = 16384
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
base_s = dev.synthetic((3 * R * C + 8,), 1, 1)
base_d = torch.empty_like(base_s)
def view(b, off):
    return b[off:off + 3 * R * C].view(3, R, C)
for so, do in ((0, 0), (1, 0), (0, 1), (1, 1), (2, 2)):
    src, dst = view(base_s, so), view(base_d, do)
    ms = t(lambda: dev.two_pass(src, w, dst))
    print(json.dumps({"src_off": so, "dst_off": do, "ms": round(ms, 4)}))
