"""Launch-overhead study at small configs (dev tool)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev
from paper_1711_09791_b200.configs import CONFIGS
for cfg in ("cfg1", "cfg2"):
    wl = CONFIGS[cfg]; w = wl.tap_vector()
    x = dev.synthetic((wl.planes, wl.rows, wl.cols), wl.seed, wl.kind); y = torch.empty_like(x)
    for _ in range(5): dev.two_pass(x, w, y)
    torch.cuda.synchronize()
    # host wall per call
    t0 = time.perf_counter(); n = 200
    for _ in range(n): dev.two_pass(x, w, y)
    host_us = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    # back-to-back GPU throughput
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n): dev.two_pass(x, w, y)
    e.record(); e.synchronize()
    b2b_us = s.elapsed_time(e) / n * 1e3
    # CUDA graph of 20 launches
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for _ in range(20): dev.two_pass(x, w, y)
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    s.record()
    for _ in range(10): g.replay()
    e.record(); e.synchronize()
    graph_us = s.elapsed_time(e) / 200 * 1e3
    ok = torch.equal(y, dev.two_pass(x, w))
    print(json.dumps({"cfg": cfg, "host_us_per_call": round(host_us, 1), "b2b_us_per_launch": round(b2b_us, 2),
                      "graph_us_per_launch": round(graph_us, 2), "graph_result_ok": bool(ok),
                      "GBps_graph": round(wl.alg_bytes / graph_us / 1e3, 1)}))
