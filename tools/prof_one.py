"""Run one op a few times at a config (for ncu captures; dev tool)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--op", default="fused")
ap.add_argument("--n", type=int, default=3)
a = ap.parse_args()
wl = CONFIGS[a.cfg]
w = wl.tap_vector()
shape = (wl.frames, wl.planes, wl.rows, wl.cols) if wl.frames > 1 else (wl.planes, wl.rows, wl.cols)
x = dev.synthetic(shape, wl.seed, wl.kind)
y = torch.empty_like(x)
dense = np.outer(w, w).astype(np.float32)
for _ in range(a.n):
    if a.op == "fused": dev.two_pass(x, w, y)
    elif a.op == "hpass": dev.hpass(x, w, y)
    elif a.op == "single": dev.single_pass(x, dense, y)
    elif a.op == "single_general": dev.single_pass(x, np.random.default_rng(2).standard_normal((5, 5)).astype(np.float32), y)
    elif a.op == "inplace": dev.two_pass_inplace(x, w)
    elif a.op == "split": dev.two_pass_split(x, y, w)
torch.cuda.synchronize()
print("done")
