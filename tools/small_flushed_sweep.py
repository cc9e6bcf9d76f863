"""Planner knobs at a small config under the bench's protocol (256 MB L2 flush
before every step, CUDA events around the step alone), next to a plain copy of
the same image under the same protocol (dev tool).

    python tools/small_flushed_sweep.py --cfg cfg1 [--grid '{"SC_NT":64};{"SC_IPC":1}']
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1711_09791_b200 import device as dev  # noqa: E402
from paper_1711_09791_b200.configs import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="cfg1")
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--grid", default="")
ap.add_argument("--size", type=int, default=0, help="override: 3 x size x size")
a = ap.parse_args()
wl = CONFIGS[a.cfg]
if a.size:
    import dataclasses

    wl = dataclasses.replace(wl, rows=a.size, cols=a.size, frames=1, planes=3)
w = wl.tap_vector()
x = dev.synthetic((wl.planes, wl.rows, wl.cols), wl.seed, wl.kind)
y = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
KEYS = ["SC_NS", "SC_OCC", "SC_NT", "SC_BAND_H", "SC_BAND_H2", "SC_IPC", "SC_NO_PDL", "SC_TAIL_WAVES", "SC_NO_SMALL",
        "SC_SMALL_MAX_MB"]


def timed(fn):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    pairs = []
    for _ in range(a.reps):
        flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        pairs.append((s, e))
    torch.cuda.synchronize()
    return statistics.median(s.elapsed_time(e) for s, e in pairs) * 1e3


copy_us = timed(lambda: y.copy_(x))
print(json.dumps({"cfg": a.cfg, "shape": [wl.planes, wl.rows, wl.cols], "op": "copy", "us": round(copy_us, 2)}),
      flush=True)
grid = [{}] + [{"SC_IPC": i} for i in (1, 2, 3, 4)] + [{"SC_NT": t} for t in (32, 64, 96, 128)] + \
       [{"SC_NS": n} for n in (3, 6, 8)] + [{"SC_OCC": o} for o in (2, 3)] + [{"SC_NO_PDL": 1}]
if a.grid:
    grid = [json.loads(g) for g in a.grid.split(";")]
for env in grid:
    for k in KEYS:
        os.environ.pop(k, None)
    os.environ.update({k: str(v) for k, v in env.items()})
    us = timed(lambda: dev.two_pass(x, w, y))
    print(json.dumps({"cfg": a.cfg, "env": env, "us": round(us, 2), "frac_of_copy": round(copy_us / us, 3)}),
          flush=True)
