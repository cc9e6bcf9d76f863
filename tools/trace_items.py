"""Per-CTA timeline of one fused launch from an SC_TRACE build (dev tool).

    python -m paper_1711_09791_b200.build -D SC_TRACE --out paper_1711_09791_b200/libsepconv_b200_trace.so
    SEPCONV_B200_LIB=paper_1711_09791_b200/libsepconv_b200_trace.so python tools/trace_items.py 1152 1152
"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1711_09791_b200 import device as dev, _lib
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
cols = int(sys.argv[2]) if len(sys.argv) > 2 else rows
L = _lib.load()
L.sc_trace_copy.argtypes = [ctypes.c_void_p, ctypes.c_longlong]
w = np.array([1, 4, 6, 4, 1], np.float32) / 16
x = dev.synthetic((3, rows, cols), 1, 1); y = torch.empty_like(x)
for _ in range(5): dev.two_pass(x, w, y)
torch.cuda.synchronize()
os.environ["SC_DEBUG_PLAN"] = "1"
dev.two_pass(x, w, y)
torch.cuda.synchronize()
os.environ.pop("SC_DEBUG_PLAN")
S = 64
buf = np.zeros(S * 4096, np.uint64)
assert L.sc_trace_copy(buf.ctypes.data, buf.size) == 0
t = buf.reshape(4096, S).astype(np.int64)
ctas = t[t[:, 0] > 0]
g0 = ctas[:, 0].min()
start = (ctas[:, 0] - g0) / 1e3  # us
end = (ctas[:, 41] - g0) / 1e3
span_cyc = ctas[:, 40] - ctas[:, 1]
span_ns = ctas[:, 41] - ctas[:, 0]
ghz = float(np.median(span_cyc / np.maximum(span_ns, 1)))
out = {"ctas": int(len(ctas)), "ghz": round(ghz, 3), "kernel_span_us": round(float(end.max()), 2),
       "start_us_p50_p90_max": [round(float(np.percentile(start, q)), 2) for q in (50, 90, 100)],
       "end_us_min_p50_max": [round(float(np.min(end)), 2), round(float(np.median(end)), 2), round(float(end.max()), 2)],
       "items_per_cta_mean": round(float(ctas[:, 42].mean()), 2)}
# per-item latencies (cycles -> us)
c2u = lambda c: c / ghz / 1e3
first_claim = c2u(ctas[:, 2] - ctas[:, 1])
out["entry_to_first_claim_us_p50"] = round(float(np.median(first_claim)), 3)
lat, work, gap = [], [], []
for r in ctas:
    n = int(min(r[42], 8))
    for i in range(n):
        if r[20 + i] and r[2 + i]:
            lat.append(c2u(r[20 + i] - r[2 + i]))      # claim -> first stage seen by consumers
            work.append(c2u(r[30 + i] - r[20 + i]))    # first stage -> item done
        if i + 1 < n and r[20 + i + 1]:
            gap.append(c2u(r[20 + i + 1] - r[30 + i]))  # item done -> next item's first stage
    # consumer exit after last item
out["claim_to_first_stage_us_p50_p90"] = [round(float(np.percentile(lat, q)), 3) for q in (50, 90)]
out["item_work_us_p50_p90"] = [round(float(np.percentile(work, q)), 3) for q in (50, 90)]
out["done_to_next_first_stage_us_p50_p90"] = [round(float(np.percentile(gap, q)), 3) for q in (50, 90)] if gap else None
last_done = np.array([c2u(r[30 + min(int(r[42]), 8) - 1] - r[1]) if r[42] else 0 for r in ctas])
exit_after = np.array([c2u(r[40] - r[1]) for r in ctas]) - last_done
out["last_item_done_to_exit_us_p50"] = round(float(np.median(exit_after)), 3)
print(json.dumps(out))
# the latest-finishing CTAs: their items (id, claim, first stage, done) in us from kernel start
if os.environ.get("TRACE_DETAIL"):
    order = np.argsort(-end)[:8]
    for k in list(order) + list(np.argsort(end)[:3]):
        r = ctas[k]; base = (r[0] - g0) / 1e3
        n = int(min(r[42], 8))
        items = [(int(r[10 + i]), round(base + c2u(r[2 + i] - r[1]), 2), round(base + c2u(r[20 + i] - r[1]), 2) if r[20 + i] else None,
                  round(base + c2u(r[30 + i] - r[1]), 2) if r[30 + i] else None) for i in range(n)]
        print(json.dumps({"cta": int(k), "sm": int(r[43]), "end_us": round(float(end[k]), 2), "items": items}))

if os.environ.get("TRACE_STAGES"):
    # stage readiness/done times (us from CTA start) of the first 8 stages for a few CTAs
    for k in range(min(4, len(ctas))):
        r = ctas[k]
        st = [(round(c2u(r[48 + i] - r[1]), 2), round(c2u(r[56 + i] - r[1]), 2)) for i in range(8) if r[48 + i]]
        print(json.dumps({"cta": k, "claim0": round(c2u(r[2] - r[1]), 2), "stages_ready_done": st}))
