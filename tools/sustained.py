"""An op timed in steady state (N back-to-back launches after a heat-up, NVML SM clock sampled) (dev tool):
argv = op (fused|inplace|split|single|single_general) [n]."""
import os, sys, json, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS
op = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
wl = CONFIGS[os.environ.get("CFG", "cfg5")]
w = wl.tap_vector()
x = dev.synthetic((wl.planes, wl.rows, wl.cols), wl.seed, wl.kind); y = torch.empty_like(x)
dense = np.outer(w, w).astype(np.float32)
gen = np.random.default_rng(2).standard_normal((5, 5)).astype(np.float32)
fn = {"fused": lambda: dev.two_pass(x, w, y), "inplace": lambda: dev.two_pass_inplace(x, w),
      "split": lambda: dev.two_pass_split(x, y, w), "single": lambda: dev.single_pass(x, dense, y),
      "single_general": lambda: dev.single_pass(x, gen, y)}[op]
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk = []; stop = False
def sample():
    while not stop:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.02)
for _ in range(300): fn()
torch.cuda.synchronize()
t = threading.Thread(target=sample); t.start()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(n): fn()
e.record(); e.synchronize()
stop = True; t.join()
print(json.dumps({"op": op, "n": n, "ms": round(s.elapsed_time(e) / n, 4), "sm_mhz_median": float(np.median(clk)) if clk else None}))
