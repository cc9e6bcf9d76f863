"""One op at a kernel width on 3 x SIZE^2 for an ncu capture (dev tool): argv = width [op]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
W = int(sys.argv[1]); op = sys.argv[2] if len(sys.argv) > 2 else "two_pass"
R = C = int(os.environ.get("SIZE", 8192))
x = dev.synthetic((3, R, C), 1, 1); y = torch.empty_like(x)
w = np.random.default_rng(W).standard_normal(W).astype(np.float32)
k = np.random.default_rng(W).standard_normal((W, W)).astype(np.float32)
for _ in range(3):
    if op == "two_pass": dev.two_pass(x, w, y)
    elif op == "single": dev.single_pass(x, k, y)
    elif op == "hpass": dev.hpass(x, w, y)
torch.cuda.synchronize(); print("done")
