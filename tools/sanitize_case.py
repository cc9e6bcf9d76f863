"""Small invocations of every kernel family for compute-sanitizer runs (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w5 = np.array([-1, -2, 7, -2, -1], np.float32); w3 = np.array([0.25, 0.5, 0.25], np.float32)
dense = np.outer(w5, w5).astype(np.float32)
for (P, R, C) in ((3, 67, 256), (2, 41, 131), (1, 9, 12)):
    x = dev.synthetic((P, R, C), 3, 2)
    for w in (w5, w3):
        y = dev.two_pass(x, w)
        img, scr = x.clone(), torch.zeros_like(x)
        dev.two_pass_split(img, scr, w)
        d = torch.zeros_like(x)
        dev.hpass(x, w, d); dev.vpass(x, w, d)
    s = torch.zeros_like(x)
    dev.single_pass(x.clone(), dense, s, copy_back=True)
    if R > 20:
        out = torch.empty((P, R - 10, C), device="cuda")
        dev.two_pass_band(x[:, 3:R - 3].contiguous(), w5, out, global_rows=R, src_row0=3, dst_row0=5, out_lo=5,
                          out_hi=R - 5)
u8 = torch.randint(0, 256, (40, 64, 3), dtype=torch.uint8, device="cuda")
dev.two_pass_u8hwc(u8, w5)
dev.planes_to_hwc(dev.hwc_to_planes(u8))
os.makedirs("gpurun_out", exist_ok=True)
host = [np.random.rand(50, 70).astype(np.float32) for _ in range(3)]
dev.two_pass_host(host, host, w5)
torch.cuda.synchronize()
print("sanitize case done")
