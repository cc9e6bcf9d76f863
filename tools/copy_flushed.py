"""A plain device copy of each config's image under bench.py's protocol (256 MB
L2 flush before every step, CUDA events around the step only): the same-size
copy floor the small-config bench lines can be compared with (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cfg in ("cfg1", "cfg2", "cfg3"):
    wl = CONFIGS[cfg]
    x = dev.synthetic((wl.planes, wl.rows, wl.cols), wl.seed, wl.kind)
    y = torch.empty_like(x)
    w = wl.tap_vector()
    for name, fn in (("copy", lambda: y.copy_(x)), ("fused", lambda: dev.two_pass(x, w, y))):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        pairs = []
        for _ in range(100):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); fn(); b.record()
            pairs.append((a, b))
        torch.cuda.synchronize()
        ms = float(np.median([a.elapsed_time(b) for a, b in pairs]))
        print(json.dumps({"cfg": cfg, "op": name, "ms_flushed": round(ms, 4)}))
