"""End-to-end host path (sc_two_pass_host_f32) vs host chunk size (dev tool)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
for n in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1152,2592,4096").split(",")]:
    planes = [torch.empty((n, n), dtype=torch.float32, pin_memory=True).uniform_() for _ in range(3)]
    res = {"n": n}
    for mb in (32, 16, 8, 4, 2, 1):
        os.environ["SC_HOST_CHUNK_MB"] = str(mb)
        dev.two_pass_host(planes, planes, w)
        ts = []
        for _ in range(7):
            t0 = time.perf_counter(); dev.two_pass_host(planes, planes, w); ts.append(time.perf_counter() - t0)
        res[f"{mb}MB_ms"] = round(float(np.median(ts)) * 1e3, 3)
    os.environ.pop("SC_HOST_CHUNK_MB")
    res["bytes_each_way_MB"] = round(3 * n * n * 4 / 1e6, 1)
    print(json.dumps(res), flush=True)
