"""Fused two-pass at the reference ladder sizes: host cost, back-to-back and graph time (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
sizes = [int(s) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else "1152,1728,2592,3888".split(","))]
for n in sizes:
    x = dev.synthetic((3, n, n), 42, 1); y = torch.empty_like(x)
    for _ in range(5): dev.two_pass(x, w, y)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); k = 200
    for _ in range(k): dev.two_pass(x, w, y)
    host_us = (time.perf_counter() - t0) / k * 1e6
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k): dev.two_pass(x, w, y)
    e.record(); e.synchronize()
    b2b = s.elapsed_time(e) / k * 1e3
    g = torch.cuda.CUDAGraph(); st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(20): dev.two_pass(x, w, y)
    torch.cuda.synchronize(); g.replay(); torch.cuda.synchronize()
    s.record()
    for _ in range(10): g.replay()
    e.record(); e.synchronize()
    gr = s.elapsed_time(e) / 200 * 1e3
    # single launch, cold-ish (after L2 flush)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(20):
        flush.zero_(); s.record(); dev.two_pass(x, w, y); e.record(); e.synchronize(); ts.append(s.elapsed_time(e) * 1e3)
    byt = 3 * n * n * 8
    print(json.dumps({"n": n, "host_us": round(host_us, 1), "b2b_us": round(b2b, 2), "graph_us": round(gr, 2),
                      "cold_us": round(float(np.median(ts)), 2), "TBps_graph": round(byt / gr / 1e6, 2),
                      "TBps_cold": round(byt / float(np.median(ts)) / 1e6, 2)}))
