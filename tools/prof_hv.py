import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
x = dev.synthetic((3, 16384, 16384), 5, 1); y = torch.empty_like(x)
w1 = np.array([1.0], np.float32)
op = sys.argv[1]
for _ in range(3):
    if op == "h": dev.hpass(x, w1, y)
    else: dev.vpass(x, w1, y)
torch.cuda.synchronize(); print("done")
