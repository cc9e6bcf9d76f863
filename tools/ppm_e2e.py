"""PPM bytes -> convolved PPM bytes end to end (ppm.convolve_ppm_bytes) at square sizes (dev tool)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import ppm
from paper_1711_09791_b200.kernels import gaussian5
for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2048,4096,8192").split(",")]:
    rng = np.random.default_rng(n)
    data = f"P6\n{n} {n}\n255\n".encode() + rng.integers(0, 256, size=n * n * 3, dtype=np.uint8).tobytes()
    k = gaussian5()
    out = ppm.convolve_ppm_bytes(data, k)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); out = ppm.convolve_ppm_bytes(data, k); ts.append(time.perf_counter() - t0)
    ms = float(np.median(ts)) * 1e3
    print(json.dumps({"n": n, "payload_MB": round(n * n * 3 / 1e6, 1), "ms": round(ms, 2),
                      "GBps_each_way": round(n * n * 3 / ms / 1e6, 2)}), flush=True)
