"""Floors for a small launch (cfg1 geometry) in a CUDA graph: empty kernel, copy, fused (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
x = dev.synthetic((3, n, n), 1, 1); y = torch.empty_like(x); z = torch.empty(1, device="cuda")
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
def graph_time(fn, k=20, reps=20):
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
    return round(float(np.median(ts)), 2)
res = {"n": n, "empty_us": graph_time(lambda: z.add_(1)), "copy_us": graph_time(lambda: y.copy_(x)),
       "fused_us": graph_time(lambda: dev.two_pass(x, w, y))}
os.environ["SC_DIRECT"] = "1"
res["fused_direct_us"] = graph_time(lambda: dev.two_pass(x, w, y))
os.environ.pop("SC_DIRECT")
res["bytes"] = x.numel() * 8
print(json.dumps(res))
