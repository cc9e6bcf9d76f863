"""FP32 rate under sustained load: the FP32-bound kernels (single pass, u8
payload) against the FP32 rate the B200 actually holds under its power cap
(dev tool).

1. tools/fp32_burn.cu (the single pass's FMUL2 + FFMA2(x, one, acc) mix) back to
   back for --seconds: lane-ops/s and the SM clock (NVML, sampled every 20 ms).
2. each kernel back to back for --seconds on its cfg5-sized input: time per
   launch (CUDA events), the reference algorithm's FP32 ops per launch
   (single pass 49 per output, two-pass 18 per output), the SM clock.

    python tools/fp32_sustained.py [--seconds 3]
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1711_09791_b200 import device as dev  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_fp32_burn.so")
BURST_FP32 = 148 * 128 * 1.965e9  # lane-ops/s at the maximum SM clock


def build():
    if not os.path.exists(SO):
        subprocess.check_call(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler",
                               "-fPIC", os.path.join(HERE, "fp32_burn.cu"), "-o", SO])
    lib = ctypes.CDLL(SO)
    lib.fp32_burn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return lib


class Clocks:
    def __init__(self):
        import pynvml

        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.samples, self.power, self.run = [], [], True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        while self.run:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000)
            time.sleep(0.02)

    def stop(self):
        self.run = False
        self.t.join()
        tail = self.samples[len(self.samples) // 4:]  # after the ramp
        ptail = self.power[len(self.power) // 4:]
        return statistics.median(tail), max(ptail)


def sustained(fn, seconds):
    """(ms per launch over the run, median SM MHz, max W) of fn back to back."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    clk = Clocks()
    n, t0 = 0, time.time()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < seconds:
        for _ in range(10):
            fn()
        n += 10
        if n % 100 == 0:
            torch.cuda.synchronize()
    e.record()
    e.synchronize()
    mhz, watts = clk.stop()
    return s.elapsed_time(e) / n, mhz, watts


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=3.0)
    a = ap.parse_args()
    lib = build()
    stream = torch.cuda.current_stream().cuda_stream
    out = torch.empty(148 * 8 * 256, device="cuda")
    iters = 2048
    ops = 148 * 8 * 256 * iters * 8 * 2 * 2
    ms, mhz, w = sustained(lambda: lib.fp32_burn(out.data_ptr(), 148 * 8, iters, stream), a.seconds)
    burn_rate = ops / (ms * 1e-3)
    print(json.dumps({"kernel": "fp32_burn (FMUL2 + FFMA2 mix)", "ms": round(ms, 4), "lane_ops_per_s": burn_rate,
                      "frac_of_burst": round(burn_rate / BURST_FP32, 3), "sm_mhz": mhz, "power_w_max": w,
                      "lane_ops_per_cycle_per_sm": round(burn_rate / (148 * mhz * 1e6), 1)}), flush=True)
    R = C = 16384
    x = dev.synthetic((3, R, C), 5, 1)
    y = torch.empty_like(x)
    gauss = np.float32([1, 4, 6, 4, 1]) / np.float32(16)
    m_sym = gauss[:, None] * gauss[None, :]
    rng = np.random.default_rng(2)
    m_gen = rng.standard_normal((5, 5)).astype(np.float32)
    outputs = 3 * (R - 4) * (C - 4)
    cases = [("single pass, general matrix", lambda: dev.single_pass(x, m_gen, y), 49 * outputs),
             ("single pass, mirror-symmetric (outer(gauss5))", lambda: dev.single_pass(x, m_sym, y), 49 * outputs),
             ("fused two-pass", lambda: dev.two_pass(x, gauss, y), 18 * outputs)]
    u8 = torch.randint(0, 256, (R, C, 3), dtype=torch.uint8, device="cuda")
    u8o = torch.empty_like(u8)
    cases.append(("u8 payload (fused read -> two-pass -> write)", lambda: dev.two_pass_u8hwc(u8, gauss, u8o),
                  18 * (R - 4) * (C - 4) * 3))
    for name, fn, alg_ops in cases:
        ms, mhz, w = sustained(fn, a.seconds)
        rate = alg_ops / (ms * 1e-3)
        print(json.dumps({"kernel": name, "ms": round(ms, 4), "alg_lane_ops_per_s": rate,
                          "frac_of_sustained_fp32": round(rate / burn_rate, 3),
                          "frac_of_burst_fp32": round(rate / BURST_FP32, 3), "sm_mhz": mhz, "power_w_max": w,
                          "frac_of_fp32_at_this_clock": round(rate / (148 * 128 * mhz * 1e6), 3)}), flush=True)


if __name__ == "__main__":
    main()
