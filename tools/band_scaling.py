"""Per-rank step time of an interior row band at N = 1, 2, 4, 8 (cfg5 geometry) on
ONE GPU: the compute part of the N-GPU step, i.e. the strong-scaling ceiling
before any NVLink effect (dev tool).

Two forms per N: the plain band kernel (input rows incl. halo in one buffer),
and the peer transport's actual step -- `sc_two_pass_band_peer_sig_f32` with the
halo rows in separate neighbour buffers and the readiness signalling on (the
neighbours' words pre-published, so no wait: what remains is the step's own
cost). Efficiency = T(N=1) / (N * T(N)).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_09791_b200 import _lib  # noqa: E402
from paper_1711_09791_b200 import device as dev  # noqa: E402
from paper_1711_09791_b200.multi import SIG_WORDS, band_plan  # noqa: E402

R = C = 16384
P = 3
w = np.array([1, 4, 6, 4, 1], np.float32) / np.float32(16)
L = _lib.load()
stream = torch.cuda.current_stream().cuda_stream


def timed(f, n=50):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        f()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / n


base = None
for n in (1, 2, 4, 8):
    b = band_plan(R, min(1, n - 1), n, 2)  # an interior band when n > 2
    src = dev.synthetic((P, b.in_hi - b.in_lo, C), 5, 1)
    dst = torch.empty((P, b.hi - b.lo, C), device="cuda")
    ms = timed(lambda: dev.two_pass_band(src, w, dst, global_rows=R, src_row0=b.in_lo, dst_row0=b.lo, out_lo=b.lo,
                                         out_hi=b.hi))
    base = base or ms
    row = {"n": n, "band_rows": b.hi - b.lo, "ms_per_rank": round(ms, 4),
           "compute_scaling_eff": round(base / (n * ms), 3),
           "GBps": round(2 * 4 * P * (b.hi - b.lo) * C / ms / 1e6, 1)}
    if n > 1:
        own = src[:, b.lo - b.in_lo:b.hi - b.in_lo].contiguous()
        top = src[:, :b.lo - b.in_lo].contiguous() if b.lo > b.in_lo else None
        bot = src[:, b.hi - b.in_lo:].contiguous() if b.in_hi > b.hi else None
        sig = torch.zeros(SIG_WORDS, dtype=torch.int64, device="cuda")
        nbr = torch.full((SIG_WORDS,), 1 << 40, dtype=torch.int64, device="cuda")
        err = torch.zeros(1, dtype=torch.int32).pin_memory()
        epoch = [0]
        rows = b.hi - b.lo

        def peer_step():
            epoch[0] += 1
            _lib.check(L.sc_two_pass_band_peer_sig_f32(
                own.data_ptr(), dst.data_ptr(), P, R, C, rows * C, rows * C, C, C, b.lo, rows,
                top.data_ptr() if top is not None else None, b.in_lo, b.lo - b.in_lo, (b.lo - b.in_lo) * C, C,
                bot.data_ptr() if bot is not None else None, b.hi, b.in_hi - b.hi, (b.in_hi - b.hi) * C, C,
                b.lo, b.lo, b.hi, w.ctypes.data, 5, 0, sig.data_ptr(),
                nbr.data_ptr() if top is not None else None, nbr.data_ptr() if bot is not None else None,
                epoch[0], err.data_ptr(), stream))

        pms = timed(peer_step)
        row.update({"peer_signalled_ms": round(pms, 4), "peer_signalled_eff": round(base / (n * pms), 3)})
        del own, top, bot
    print(json.dumps(row), flush=True)
    del src, dst
