"""Quick CUDA-event timing of each kernel family at a config (dev tool)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg5")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--ops", default="fused,split,single,hpass,copy")
a = ap.parse_args()
wl = CONFIGS[a.cfg]
w = wl.tap_vector()
shape = (wl.frames, wl.planes, wl.rows, wl.cols) if wl.frames > 1 else (wl.planes, wl.rows, wl.cols)
x = dev.synthetic(shape, wl.seed, wl.kind)
y = torch.empty_like(x)
z = torch.empty_like(x)
dense = np.outer(w, w).astype(np.float32)
alg = wl.alg_bytes
def timeit(fn):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); ts.append(s.elapsed_time(e))
    return float(np.median(ts)), float(np.min(ts))
ops = {
  "fused": lambda: dev.two_pass(x, w, y),
  "split": lambda: dev.two_pass_split(y, z, w),
  "single": lambda: dev.single_pass(x, dense, y),
  "hpass": lambda: dev.hpass(x, w, y),
  "copy": lambda: y.copy_(x),
}
for name in a.ops.split(","):
    med, mn = timeit(ops[name])
    print(json.dumps({"cfg": a.cfg, "op": name, "ms_med": round(med, 4), "ms_min": round(mn, 4),
                      "alg_GBps_med": round(alg / med / 1e6, 1), "frac_of_6447": round(alg / med / 1e6 / 6447.5, 3)}))
