"""Per-rank kernel time of an interior row band at N = 1, 2, 4, 8 (cfg5 geometry) on
ONE GPU: the compute part of the N-GPU step, i.e. the strong-scaling ceiling
before any NVLink effect (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.multi import band_plan
R = C = 16384
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
base = None
for n in (1, 2, 4, 8):
    b = band_plan(R, min(1, n - 1), n, 2)  # an interior band when n > 2
    src = dev.synthetic((3, b.in_hi - b.in_lo, C), 5, 1)
    dst = torch.empty((3, b.hi - b.lo, C), device="cuda")
    f = lambda: dev.two_pass_band(src, w, dst, global_rows=R, src_row0=b.in_lo, dst_row0=b.lo, out_lo=b.lo, out_hi=b.hi)
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50): f()
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 50
    base = base or ms
    print(json.dumps({"n": n, "band_rows": b.hi - b.lo, "ms_per_rank": round(ms, 4),
                      "compute_scaling_eff": round(base / (n * ms), 3),
                      "GBps": round(2 * 4 * 3 * (b.hi - b.lo) * C / ms / 1e6, 1)}))
    del src, dst
