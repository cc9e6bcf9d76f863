"""One fused two-pass at cfg5 size into a destination view offset by one float
(unaligned destination rows: the staged-store path), for an ncu capture (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R = C = 16384
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
src = dev.synthetic((3, R, C), 1, 1)
base = torch.empty(3 * R * C + 8, device="cuda")
dst = base[1:1 + 3 * R * C].view(3, R, C)
for _ in range(3):
    dev.two_pass(src, w, dst)
torch.cuda.synchronize()
print("done")
