#!/bin/bash
timeout -s KILL 600 python -m pytest tests/test_ppm.py -x -q -m gpu 2>&1 | tail -3
python - <<'PY'
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
from paper_1711_09791_b200 import device as dev
for (R, C) in ((16384, 16384), (1080, 1920), (4096, 4096)):
    src = torch.randint(0, 256, (R, C, 3), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(src)
    w = np.array([1, 4, 6, 4, 1], np.float32) / 16
    for _ in range(3): dev.two_pass_u8hwc(src, w, out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20): dev.two_pass_u8hwc(src, w, out)
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 20
    print(json.dumps({"shape": [R, C], "ms": round(ms, 4), "Gpix_s": round(R * C / ms / 1e6, 1), "GBps": round(6 * R * C / ms / 1e6, 1)}))
PY
