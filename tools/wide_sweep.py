"""Planner knobs for the widths 11..21 kernels (dev tool): SIZE, OP=two_pass|single|hpass|vpass."""
import os, sys, json, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R = C = int(os.environ.get("SIZE", 8192))
op = os.environ.get("OP", "two_pass")
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
grid = [{}]
for ns in (5, 6, 8): grid.append({"SC_NS": str(ns)})
for bh, bh2 in ((128, 32), (256, 64)): grid.append({"SC_BAND_H": str(bh), "SC_BAND_H2": str(bh2), "SC_NS": "6"})
for nt in (64, 96): grid.append({"SC_NT": str(nt), "SC_NS": "6", "SC_BAND_H": "128", "SC_BAND_H2": "32"})
for W in [int(v) for v in os.environ.get("WIDTHS", "11,15,21").split(",")]:
    w = np.random.default_rng(W).standard_normal(W).astype(np.float32)
    k = np.outer(w, w).astype(np.float32)
    fn = {"two_pass": lambda: dev.two_pass(x, w, y), "single": lambda: dev.single_pass(x, k, y),
          "hpass": lambda: dev.hpass(x, w, y), "vpass": lambda: dev.vpass(x, w, y)}[op]
    for kn in grid:
        for a, b in kn.items(): os.environ[a] = b
        ms = t(fn, n=3 if op == "single" else 10)
        for a in kn: os.environ.pop(a)
        print(json.dumps({"W": W, "op": op, "knobs": kn, "ms": round(ms, 4)}), flush=True)
