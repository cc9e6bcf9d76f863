"""Planner/tuning sweep for the fused kernel (dev tool): env knobs read per launch."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--op", default="fused")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--grid", default="")
ap.add_argument("--graph", action="store_true", help="time 20 launches captured in a CUDA graph (no host overhead)")
ap.add_argument("--size", type=int, default=0, help="override: 3 x size x size, gauss5")
ap.add_argument("--rows", type=int, default=0, help="override rows (with --cols)")
ap.add_argument("--cols", type=int, default=0)
a = ap.parse_args()
wl = CONFIGS[a.cfg]
if a.size or a.rows:
    import dataclasses
    wl = dataclasses.replace(wl, rows=a.rows or a.size, cols=a.cols or a.size, frames=1, planes=3)
w = wl.tap_vector()
shape = (wl.frames, wl.planes, wl.rows, wl.cols) if wl.frames > 1 else (wl.planes, wl.rows, wl.cols)
x = dev.synthetic(shape, wl.seed, wl.kind)
y = torch.empty_like(x)
dense = np.outer(w, w).astype(np.float32)
op = {"fused": lambda: dev.two_pass(x, w, y), "single": lambda: dev.single_pass(x, dense, y),
      "hpass": lambda: dev.hpass(x, w, y), "vpass": lambda: dev.vpass(x, w, y),
      "inplace": lambda: dev.two_pass_inplace(x, w), "split": lambda: dev.two_pass_split(x, y, w)}[a.op]
KEYS = ["SC_NS", "SC_OCC", "SC_NT", "SC_BAND_H", "SC_BAND_H2", "SC_TAIL_WAVES", "SC_EXACT_WAVES", "SC_L2_EVICT_FIRST", "SC_IPC"]
def run(env):
    for k in KEYS: os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    for _ in range(3): op()
    torch.cuda.synchronize()
    if a.graph:
        g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                for _ in range(20): op()
        g.replay(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(a.reps):
            s.record(); g.replay(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) / 20)
        med = float(np.median(ts))
        print(json.dumps({"env": env, "ms": round(med, 5), "GBps": round(wl.alg_bytes / med / 1e6, 1), "graph": True}), flush=True)
        return
    ts = []
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); op(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    med = float(np.median(ts))
    print(json.dumps({"env": env, "ms": round(med, 4), "GBps": round(wl.alg_bytes / med / 1e6, 1)}), flush=True)
grid = [{}]
grid += [{"SC_NS": n} for n in (3, 5, 6, 8)]
grid += [{"SC_OCC": o} for o in (1, 2, 3)]
grid += [{"SC_NT": t} for t in (32, 64, 96, 192, 256)]
grid += [{"SC_BAND_H": b} for b in (64, 128, 256, 512, 1024, 2048)]
grid += [{"SC_L2_EVICT_FIRST": 1}]
grid += [{"SC_NT": 64, "SC_NS": 6}, {"SC_NT": 64, "SC_NS": 8}, {"SC_NT": 256, "SC_NS": 3}]
if a.grid:
    grid = [json.loads(g) for g in a.grid.split(";")]
os.environ["SC_DEBUG_PLAN"] = "1"; run({}); os.environ.pop("SC_DEBUG_PLAN")
for g in grid: run(g)
