"""Fused-kernel time vs rows at fixed width, in CUDA graphs (fixed cost vs per-row cost; dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
cols = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
def graph_time(fn, k=20, reps=15):
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
for rows in (16, 64, 256, 1152, 2304, 4608):
    x = dev.synthetic((3, rows, cols), 1, 1); y = torch.empty_like(x)
    out = {"rows": rows, "cols": cols, "copy_us": graph_time(lambda: y.copy_(x)), "fused_us": graph_time(lambda: dev.two_pass(x, w, y))}
    for knob in ("SC_OCC=1", "SC_OCC=2", "SC_NS=3", "SC_IPC=1"):
        k, v = knob.split("="); os.environ[k] = v
        out[knob] = graph_time(lambda: dev.two_pass(x, w, y)); os.environ.pop(k)
    print(json.dumps(out), flush=True)
