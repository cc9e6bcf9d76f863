"""Fused time vs width at fixed rows, in CUDA graphs (partial-strip cost; dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2592
widths = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2048, 2080, 2304, 2592, 2816, 3072]
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
def graph_time(fn, k=20, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(k): fn()
    g.replay(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3 / k)
    return float(np.median(ts))
for c in widths:
    x = dev.synthetic((3, rows, c), 1, 1); y = torch.empty_like(x)
    tf = graph_time(lambda: dev.two_pass(x, w, y)); tc = graph_time(lambda: y.copy_(x))
    print(json.dumps({"rows": rows, "cols": c, "fused_us": round(tf, 2), "copy_us": round(tc, 2),
                      "fused_TBps": round(x.numel() * 8 / tf / 1e6, 2), "copy_TBps": round(x.numel() * 8 / tc / 1e6, 2)}), flush=True)
