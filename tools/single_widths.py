"""Single pass at widths 5/7/9, general and mirror-symmetric matrices, aligned kernel vs the lane-strided one (SC_FORCE_GENERIC=1) (dev tool)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
R = C = int(os.environ.get("SIZE", 8192))
x = dev.synthetic((3, R, C), 1, 1); y = torch.empty_like(x)
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): fn()
    e.record(); e.synchronize()
    return s.elapsed_time(e) / n
for W in (5, 7, 9):
    w = np.random.default_rng(W).standard_normal(W).astype(np.float32)
    k = np.random.default_rng(W).standard_normal((W, W)).astype(np.float32)
    half = np.random.default_rng(W).standard_normal(W // 2 + 1).astype(np.float32)
    ws = np.concatenate([half, half[-2::-1]])
    ksym = np.outer(ws, ws).astype(np.float32)
    rec = {"W": W, "lib": os.path.basename(os.environ.get("SEPCONV_B200_LIB", "main"))}
    for g in ("0", "1"):
        os.environ["SC_FORCE_GENERIC"] = g
        rec["gen_g" + g] = round(t(lambda: dev.single_pass(x, k, y)), 4)
        rec["sym_g" + g] = round(t(lambda: dev.single_pass(x, ksym, y)), 4)
    print(json.dumps(rec), flush=True)
