"""One misaligned-view launch sequence for ncu (dev tool): argv = src_off dst_off (floats)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
R = C = 16384
so, do = int(sys.argv[1]), int(sys.argv[2])
base_s = dev.synthetic((3 * R * C + 8,), 1, 1); base_d = torch.empty_like(base_s)
src = base_s[so:so + 3 * R * C].view(3, R, C); dst = base_d[do:do + 3 * R * C].view(3, R, C)
for _ in range(3): dev.two_pass(src, w, dst)
torch.cuda.synchronize(); print("done")
