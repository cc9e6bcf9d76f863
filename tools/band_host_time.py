"""Host time per row-band step of the multi-GPU transports ("host time
per step under 20 us in NCCL mode"), on one GPU.

The NCCL plan runs with a one-rank communicator whose band names itself as both
neighbours (the packed halos go through ncclSend/ncclRecv and come back), on the
geometry of one rank of config 5 at N = 8 (3 x 2048 x 16384 owned rows). Host
time = wall time of `steps` step() calls issued back to back, measured BEFORE the
final synchronize (the GPU runs behind); GPU time per step from CUDA events.

    python tools/band_host_time.py [--steps 200]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def measure(step, steps):
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    host_us = (time.perf_counter() - t0) * 1e6 / steps
    b.record()
    torch.cuda.synchronize()
    return host_us, a.elapsed_time(b) * 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    args = ap.parse_args()
    from paper_1711_09791_b200 import _lib
    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.multi import Band, NcclBandStepper, PeerBandStepper, nccl_comm

    torch.cuda.set_device(0)
    P, R, C = 3, 16384, 16384
    lo, hi = 2048 * 3, 2048 * 4  # rank 3 of 8
    w = np.array([1, 4, 6, 4, 1], np.float32) / np.float32(16)
    src = dev.synthetic((P, hi - lo, C), 5, 1)
    dst = torch.empty_like(src)
    band = Band(0, 1, R, 2, lo, hi)
    out = {}
    comm = nccl_comm(None, 0)
    os.environ["SC_BAND_TIMING"] = "1"
    st = NcclBandStepper(src, dst, band, w, use_graph=False, comm=comm, rank_above=0, rank_below=0)
    for _ in range(3):
        st.step()  # phase breakdown on stderr
    torch.cuda.synchronize()
    st.close()
    del os.environ["SC_BAND_TIMING"]
    for graph in (True, False):
        st = NcclBandStepper(src, dst, band, w, use_graph=graph, comm=comm, rank_above=0, rank_below=0)
        host_us, gpu_us = measure(st.step, args.steps)
        out["nccl_graph" if graph else "nccl_eager"] = {"host_us_per_step": round(host_us, 2),
                                                        "gpu_us_per_step": round(gpu_us, 2), "graphed": st.graphed}
        st.close()
    # peer transport, signalled: the neighbours' ready words pre-published in
    # device memory (as if they had started), so the kernel never waits
    L = _lib.load()
    above = dev.synthetic((P, 2, C), 6, 1)
    below = dev.synthetic((P, 2, C), 7, 1)
    from paper_1711_09791_b200.multi import SIG_WORDS

    sig = torch.zeros(SIG_WORDS, dtype=torch.int64, device="cuda")
    nbr = torch.full((SIG_WORDS,), 1 << 40, dtype=torch.int64, device="cuda")  # always "ready"
    err = torch.zeros(1, dtype=torch.int32).pin_memory()
    stream = torch.cuda.current_stream().cuda_stream
    epoch = [0]
    base = (src.data_ptr(), dst.data_ptr(), P, R, C, (hi - lo) * C, (hi - lo) * C, C, C, lo, hi - lo,
            above.data_ptr(), lo - 2, 2, 2 * C, C, below.data_ptr(), hi, 2, 2 * C, C, lo, lo, hi, w.ctypes.data, 5, 0,
            sig.data_ptr(), nbr.data_ptr(), nbr.data_ptr())

    def peer_step():
        epoch[0] += 1
        _lib.check(L.sc_two_pass_band_peer_sig_f32(*base, epoch[0], err.data_ptr(), stream))

    host_us, gpu_us = measure(peer_step, args.steps)
    out["peer_signalled"] = {"host_us_per_step": round(host_us, 2), "gpu_us_per_step": round(gpu_us, 2)}
    # the same without neighbour words (no waits: only the ready store and the done count)
    base_nowait = base[:-2] + (None, None)

    def peer_step_nowait():
        epoch[0] += 1
        _lib.check(L.sc_two_pass_band_peer_sig_f32(*base_nowait, epoch[0], err.data_ptr(), stream))

    host_us, gpu_us = measure(peer_step_nowait, args.steps)
    out["peer_signalled_nowait"] = {"host_us_per_step": round(host_us, 2), "gpu_us_per_step": round(gpu_us, 2)}
    # the plain peer call with the same neighbour rows (no signalling at all)
    base_plain = base[:-3]

    def peer_step_plain():
        _lib.check(L.sc_two_pass_band_peer_f32(*base_plain, stream))

    host_us, gpu_us = measure(peer_step_plain, args.steps)
    out["peer_unsignalled_same_rows"] = {"host_us_per_step": round(host_us, 2), "gpu_us_per_step": round(gpu_us, 2)}
    solo = PeerBandStepper(src, dst, Band(0, 1, hi - lo, 2, 0, hi - lo), w)
    host_us, gpu_us = measure(solo.step, args.steps)
    out["peer_plain_call"] = {"host_us_per_step": round(host_us, 2), "gpu_us_per_step": round(gpu_us, 2)}
    print(json.dumps({"geometry": f"{P}x{hi - lo}x{C} band (config 5, rank 3 of 8)", "steps": args.steps, **out}))


if __name__ == "__main__":
    main()
