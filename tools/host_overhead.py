"""Host-side cost per call of each layer (dev tool)."""
import os, sys, time, ctypes, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev, _lib
L = _lib.load()
x = dev.synthetic((3, 64, 1024), 1, 1); y = torch.empty_like(x)
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
taps = w.ctypes.data
stream = torch.cuda.current_stream().cuda_stream
def bench(fn, n=2000):
    for _ in range(50): fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    dt = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    return round(dt, 2)
res = {}
res["raw_ctypes_call"] = bench(lambda: L.sc_two_pass_fused_f32(x.data_ptr(), y.data_ptr(), 3, 64, 1024, 64*1024, 64*1024, 1024, 1024, taps, 5, 0, stream))
res["device.two_pass"] = bench(lambda: dev.two_pass(x, w, y))
res["torch_current_stream"] = bench(lambda: torch.cuda.current_stream(x.device).cuda_stream)
res["planes_geom"] = bench(lambda: dev._planes(x, "x"))
res["taps_conv"] = bench(lambda: dev._taps(w))
res["empty_kernel_torch_add"] = bench(lambda: torch.add(x, 1.0, out=y))
print(json.dumps(res))
