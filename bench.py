#!/usr/bin/env python3
"""Benchmark of the B200 separable-convolution hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg5]

Workload (BASELINE.json configs[4], the largest single-image config and the one
north_star scores at 1/2/4/8 GPUs): one image of 3 float32 planes x 16384 x 16384,
values U[0,1) from a seed, taps [1,4,6,4,1]/16, faithful two-pass. A "step" is
one fused two-pass over the whole image; N>1 splits it into row bands with a
2-row NCCL halo exchange per step (strong scaling: total work fixed).

metric: Gpixels/s (1 pixel = one (row, col) location across the 3 planes);
value = whole-job pixels / max-over-ranks step time, inputs resident in HBM.
e2e: the same metric through the C-ABI host entry point (sc_two_pass_host_f32):
pinned host planes in, H2D + kernel + D2H inside the timed region.

Inputs are 3.2 GB, far larger than the 126 MB L2, so no flush is needed between
timed steps. --impl reference times the reference's own CPU path on the host
cores: the real sepconv_lab package (baseline/_ref),
convolve_image(TWO_PASS, StaticChunked(os.cpu_count())) on the full workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_1711_09791_b200.configs import CONFIGS  # noqa: E402

METRIC = "Gpixels/s (3-plane fp32) and effective HBM GB/s as % of B200 peak, 1/2/4/8 GPU"
NOMINAL_HBM_GBPS = 8000.0


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0}, "fallback"


def traffic_from_profiles(cfg: str):
    """dram read+write bytes per launch of the fused kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(cfg)
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# clocks sampled during the timed region

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _poll(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:  # noqa: BLE001 - clocks are best-effort evidence
                return
            self._stop.wait(0.05)

    def start(self):
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"], "samples": 0}
        def num(v):
            try:
                return float(v)
            except ValueError:
                return None
        busy = [s for s in self.samples if num(s[7]) and num(s[7]) > 0] or self.samples
        sm = [num(s[0]) for s in busy if num(s[0])]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in busy:
            for name, v in zip(names, s[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(busy[0][1]), "reasons": sorted(reasons), "samples": len(busy)}


# ---------------------------------------------------------------------------
# distributed plumbing

def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_config(wl, world):
    """The `config` object of both arms' JSON lines (identical for the same
    workload and N): what is convolved, how it is split, and the L2 protocol,
    which follows from the largest per-rank input (rank 0's share)."""
    from paper_1711_09791_b200.multi import partition_block

    if wl.frames > 1:
        f0, f1 = partition_block(0, wl.frames, 0, world)
        share_px = (f1 - f0) * wl.rows * wl.cols
    else:
        lo, hi = partition_block(0, wl.rows, 0, world)
        share_px = (hi - lo) * wl.cols
    in_bytes = 4 * wl.planes * share_px
    l2 = ("inputs %.1f GB >> 126 MB L2; no flush needed" % (in_bytes / 1e9) if in_bytes >= (256 << 20) else
          "inputs %.0f MB < 2x L2: a 256 MB L2 flush before every step, outside the step's events" % (in_bytes / 1e6))
    return {"workload": f"{wl.name}: {wl.note}", "frames": wl.frames, "planes": wl.planes, "rows": wl.rows,
            "cols": wl.cols, "taps": [float(v) for v in wl.tap_vector()],
            "parallelism": f"rowband{world}" if wl.frames == 1 else f"frames{world}", "l2": l2}


REF_INSTALL = os.path.join(ROOT, "baseline", "_ref")


def import_reference():
    """The real reference package, sepconv_lab, from baseline/_ref (the pip install
    of /root/reference/pkg that travels with the repo), or None."""
    if os.path.isdir(REF_INSTALL) and REF_INSTALL not in sys.path:
        sys.path.append(REF_INSTALL)
    try:
        import sepconv_lab
    except ImportError:
        return None
    return sepconv_lab


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ReferenceRun:
    """One step of the workload through the reference's own CPU path:
    sepconv_lab.convolve_image(image, kernel, TWO_PASS, StaticChunked(cores),
    workspace=..., pool=...) (S/executors.py:269-405) on the FULL image of the
    configuration (every frame for a batch), vectorised, with one worker pool
    reused across steps as the reference's time_variant does (S/bench.py:134-179).
    The input samples are the bench's own (the same seeded splitmix64 stream,
    generated by the oracle's C generator so the two arms convolve identical data)."""

    def __init__(self, sl, wl, cores):
        from oracle import oracle as orc

        self.sl, self.wl = sl, wl
        P, R, C = wl.planes, wl.rows, wl.cols
        self.buf = orc.synthetic(wl.frames * P * R * C, wl.seed, wl.kind).reshape(wl.frames, P, R, C)
        # zero-copy Images over the (F, P, R, C) buffer (Plane keeps float32 C-contiguous views, S/image.py:37-39)
        self.images = [sl.Image([sl.Plane(self.buf[f, p]) for p in range(P)]) for f in range(wl.frames)]
        self.workspace = sl.Image.zeros(R, C, P)
        self.kernel = sl.SeparableKernel(wl.tap_vector())
        self.variant = sl.ConvVariant(sl.Algorithm.TWO_PASS)
        self.plan = sl.StaticChunked(workers=cores)
        self.pool = sl.WorkerPool(cores)

    def __call__(self):
        for img in self.images:
            self.sl.convolve_image(img, self.kernel, self.variant, self.plan, workspace=self.workspace,
                                   pool=self.pool)

    def close(self):
        self.pool.close()


def _port_run(wl, cores, rows):
    """Fallback when sepconv_lab is not installed: the oracle's numpy port of the
    same StaticChunked two-pass on a row slice (kind "port")."""
    from oracle import oracle as orc

    w = wl.tap_vector()
    planes = [orc.synthetic(rows * wl.cols, wl.seed, wl.kind, offset=p * wl.rows * wl.cols).reshape(rows, wl.cols)
              for p in range(wl.planes)]
    scratch = [np.zeros_like(p) for p in planes]
    run = orc.NumpyTwoPass(cores)
    return (lambda: run(planes, scratch, w)), run.close


def reference_arm(args, wl):
    """The reference's own CPU implementation of the path on the host cores (rank 0
    only; other ranks exit without work): the real sepconv_lab package on the FULL
    configured workload, same steps and warm-up as our arm."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    sl = import_reference()
    if sl is not None:
        run = ReferenceRun(sl, wl, cores)
        fn, close = run, run.close
        px = wl.pixels
        kind = "reference"
        sample = (f"the full workload per step ({wl.frames} x {wl.planes}x{wl.rows}x{wl.cols}): sepconv_lab "
                  f"{sl.__version__} (baseline/_ref) convolve_image(TWO_PASS, StaticChunked({cores})), vectorised, "
                  f"one WorkerPool reused (S/executors.py:269-405, S/bench.py:134-179)")
    else:
        rows = max(64, min(wl.rows, args.ref_rows))
        fn, close = _port_run(wl, cores, rows)
        px = rows * wl.cols
        kind = "port"
        sample = (f"{wl.planes}x{rows}x{wl.cols} slice of {wl.name} per step (sepconv_lab not installed: numpy "
                  f"port of the reference's vectorised two-pass, StaticChunked({cores}) threads)")
    times = []
    try:
        for _ in range(args.warmup):
            fn()
        for _ in range(args.steps):
            t0 = time.perf_counter()
            fn()
            times.append(time.perf_counter() - t0)
    finally:
        close()
    dt = sum(times) / len(times)
    value = px / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gpix/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak" if wl.frames > 1 else "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": workload_config(wl, world),
        "cpu_baseline": {"value": round(value, 6), "unit": "Gpix/s", "cores": cores, "kind": kind,
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "Gpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(wl):
    """Bounded sample of the same workload on the reference's own CPU path (the
    real sepconv_lab when installed): 1 warm-up, then steps until ~10 s of CPU
    work (at least 2). Reported baseline, not the target."""
    cores = os.cpu_count() or 1
    sl = import_reference()
    if sl is not None:
        run = ReferenceRun(sl, wl, cores)
        fn, close, px, kind = run, run.close, wl.pixels, "reference"
        what = (f"full {wl.name} workload per step, sepconv_lab {sl.__version__} convolve_image(TWO_PASS, "
                f"StaticChunked({cores}))")
    else:
        rows = min(wl.rows, 2048)
        fn, close = _port_run(wl, cores, rows)
        px, kind = rows * wl.cols, "port"
        what = f"{wl.planes}x{rows}x{wl.cols} slice of {wl.name}, numpy port, StaticChunked({cores})"
    try:
        fn()  # warm-up (S/bench.py:158-159)
        reps, t0 = 0, time.perf_counter()
        while True:
            fn()
            reps += 1
            el = time.perf_counter() - t0
            if (el > 10.0 and reps >= 2) or reps >= 200:
                break
    finally:
        close()
    return {"value": round(px * reps / el / 1e9, 6), "unit": "Gpix/s", "cores": cores, "kind": kind,
            "cpu_model": cpu_model(), "sample": f"{what}; {reps} steps after 1 warm-up"}


def host_chunk_bytes(rows, cols, planes, r, band_lo, band_hi, in_lo, in_hi, call_planes=None):
    """Bytes the host path moves per step (mirrors csrc/stream.cu chunking: ~1/24 of
    the call's planes per chunk, clamped to [4, 32] MiB; halo rows re-read per chunk)."""
    total = (call_planes or planes) * (band_hi - band_lo) * cols * 4
    chunk_bytes = min(max(total // 24, 4 << 20), 32 << 20)
    ch = max(16, min(band_hi - band_lo, chunk_bytes // (cols * 4)))
    h2d = d2h = 0
    for lo in range(band_lo, band_hi, ch):
        hi = min(lo + ch, band_hi)
        a, b = max(lo - r, in_lo), min(hi + r, in_hi)
        h2d += (b - a) * cols * 4
        d2h += (hi - lo) * cols * 4
    return h2d * planes, d2h * planes


def halo_mode(choice: str, world: int) -> str:
    """Row-band halo transport for N>1: 'peer' needs peer access between every
    pair of local GPUs (NVLink/NVSwitch) -- or, in the one-GPU multi-rank debug
    mode, IPC on the same device."""
    import torch

    if choice != "auto":
        return choice
    n = torch.cuda.device_count()
    if n < 2:
        return "peer"  # ranks share the one device: IPC within a device needs no peer access
    ok = all(torch.cuda.can_device_access_peer(a, b) for a in range(n) for b in range(n) if a != b)
    return "peer" if ok else "nccl"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg5", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-rows", type=int, default=512)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--halo", default="auto", choices=["auto", "peer", "nccl"],
                    help="N>1 row bands: halo rows read in-kernel from the neighbours' memory (peer, "
                         "CUDA IPC over NVLink) or exchanged with NCCL send/recv (nccl); auto = peer when "
                         "every pair of local GPUs has peer access")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    wl = CONFIGS[args.config]

    if args.impl == "reference":
        return reference_arm(args, wl)

    import torch
    import torch.distributed as dist

    from paper_1711_09791_b200 import _lib
    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.multi import BandStepper, NcclBandStepper, PeerBandStepper, band_plan, frame_shard

    world, rank, local = dist_env()
    backend = os.environ.get("SEPCONV_BENCH_BACKEND", "nccl")  # gloo: orchestration check on one GPU
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
        dist.barrier()  # all ranks join the communicator before the first P2P group
    w = wl.tap_vector()
    r = len(w) // 2
    P, R, C = wl.planes, wl.rows, wl.cols
    per_frame = P * R * C

    # ---- inputs resident in HBM (generated in place: counter-based, no scatter)
    halo = "none"
    if wl.frames > 1:
        f0, f1 = frame_shard(wl.frames, rank, world)
        src = torch.empty((f1 - f0, P, R, C), dtype=torch.float32, device=device)
        dev.fill_synthetic(src, wl.seed, wl.kind, offset=f0 * per_frame)
        dst = torch.empty_like(src)
        band = None
        units_px = (f1 - f0) * R * C

        def step():
            dev.two_pass(src, w, dst)
    else:
        band = band_plan(R, rank, world, r)
        halo = halo_mode(args.halo, world) if world > 1 else "none"
        if halo == "peer" and args.halo == "auto":
            from paper_1711_09791_b200.multi import peer_transport_works

            if not peer_transport_works():  # one-time probe: both transports, same bits on every rank
                halo = "nccl"
        # owned rows only for the peer transport and the library's NCCL plan; the
        # torch P2P stepper (gloo orchestration checks) holds the halo rows too
        own_only = halo == "peer" or (halo == "nccl" and backend == "nccl")
        rows_held = (band.lo, band.hi) if own_only else (band.in_lo, band.in_hi)
        src = torch.empty((P, rows_held[1] - rows_held[0], C), dtype=torch.float32, device=device)
        for p in range(P):
            # peer: owned rows only (the kernel reads the halo rows from the neighbours);
            # nccl: owned rows plus the halo rows (refreshed by the exchange each step)
            dev.fill_synthetic(src[p], wl.seed, wl.kind, offset=p * R * C + rows_held[0] * C)
        dst = torch.empty((P, band.hi - band.lo, C), dtype=torch.float32, device=device)
        units_px = (band.hi - band.lo) * C
        stepper = None
        # device-side readiness signals order every peer step (no host barrier per
        # step) -- except when ranks share a GPU (one-GPU orchestration checks):
        # kernels that wait on one another must not share a device
        peer_signal = torch.cuda.device_count() >= world
        if halo == "peer":
            stepper = PeerBandStepper(src, dst, band, w, signal=peer_signal)
            if not peer_signal:
                stepper.sync()  # every band written before any kernel reads a neighbour's rows
        elif halo == "nccl" and backend == "nccl":
            stepper = NcclBandStepper(src, dst, band, w)  # packed halos, one graph launch per step
        elif halo == "nccl":
            stepper = BandStepper(src, dst, band, w)

        def step():
            if world == 1:
                dev.two_pass(src, w, dst)
            else:
                stepper.step()

    total_px = wl.frames * R * C
    # inputs smaller than 2x the 126 MB L2 (config 1) would be timed L2-resident:
    # flush L2 before every timed step instead and time the steps one by one
    in_bytes = 4 * P * units_px
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device) if in_bytes < (256 << 20) else None
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(local)
    sampler.start()
    stream = torch.cuda.current_stream()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    if flush is None:
        t_start.record(stream)
        for _ in range(args.steps):
            step()
        t_end.record(stream)
        torch.cuda.synchronize()
        ms = t_start.elapsed_time(t_end) / args.steps
    else:
        pairs = []
        for _ in range(args.steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b.record(stream)
            pairs.append((a, b))
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    sampler.stop()
    local_ms = ms  # this rank's own per-step time (its kernels only)
    if world > 1:
        t = torch.tensor([ms], device=device if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = total_px / (ms / 1e3) / 1e9

    # ---- dominant-kernel roofline: the fused kernel's own launch time (events on its stream)
    # (10 back-to-back launches per sample so the host launch gap is hidden)
    kev = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(10):
            if band is not None and world > 1:
                stepper.kernel_only()
            else:
                dev.two_pass(src, w, dst)
        b.record(stream)
        b.synchronize()
        kev.append(a.elapsed_time(b) / 10)
    kms_b2b = statistics.median(kev)
    if world > 1:
        # peer transport: those launches read the neighbours' buffers; nobody goes on
        # (and later frees or unmaps anything) before every rank's reads are done
        torch.cuda.synchronize()
        dist.barrier()
    # When a step IS one launch of the kernel (N=1, or N>1 with in-kernel peer halo
    # reads), its duration is read from the timed region itself (CUDA events on the
    # launching stream, this rank); otherwise (NCCL transport: two launches and an
    # exchange per step) from the back-to-back kernel-only launches above.
    one_launch = launches == args.steps
    kms = local_ms if one_launch else kms_b2b
    kernel_px = units_px
    if band is not None and world > 1 and hasattr(stepper, "kernel_rows"):
        kernel_px = (stepper.kernel_rows[1] - stepper.kernel_rows[0]) * C  # NCCL plan: the interior launch
    kernel_bytes = 2 * 4 * P * kernel_px  # algorithmic: one read + one write of the samples one launch produces
    peaks, peak_kind = measured_peaks()
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = kernel_bytes / (kms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4),
                "traffic": traffic_from_profiles(args.config) if world == 1 else None,
                "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                "kernel": "sepconv_rows_kernel<MODE_FUSED, r=2, TMA>", "kernel_ms": round(kms, 4),
                "kernel_timing": ("timed region, 1 launch per step" if one_launch else
                                  "10 back-to-back kernel-only launches after the timed region"),
                "kernel_ms_back_to_back": round(kms_b2b, 4),
                "alg_bytes_per_launch": kernel_bytes}
    if flush is not None and world == 1:
        # small inputs: a plain copy of the same image under the same protocol (L2
        # flushed before every step) -- the floor launch latency and DRAM ramp set
        # at this size, next to the big-transfer peak above
        dst_copy = torch.empty_like(src)
        cpairs = []
        for _ in range(min(args.steps, 100)):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            dst_copy.copy_(src)
            b.record(stream)
            cpairs.append((a, b))
        torch.cuda.synchronize()
        copy_ms = statistics.median(a.elapsed_time(b) for a, b in cpairs)
        roofline["same_size_copy_ms"] = round(copy_ms, 4)
        roofline["frac_of_same_size_copy"] = round(copy_ms / ms, 4)
        del dst_copy

    # ---- N=1: the drop-in call on HBM-resident planes, as a sepconv_lab user's
    # convolve_image(image, kernel, TWO_PASS, Cuda()) runs it -- in place, without a
    # workspace (one pass, no scratch) and with one (the reference's scratch end
    # state too: one read, two writes)
    dropin = None
    if band is not None and world == 1 and args.e2e_steps > 0:
        img = src.clone()
        scr = torch.empty_like(src)

        def ev_ms(fn, n=20):
            for _ in range(3):  # plan, snapshot pool and clocks settled
                fn()
            torch.cuda.synchronize()
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            for _ in range(n):
                fn()
            b_ev.record(stream)
            torch.cuda.synchronize()
            return a_ev.elapsed_time(b_ev) / n

        ip_ms = ev_ms(lambda: dev.two_pass_inplace(img, w))
        sp_ms = ev_ms(lambda: dev.two_pass_split(img, scr, w))
        dropin = {"no_workspace": {"ms": round(ip_ms, 4), "value": round(total_px / (ip_ms / 1e3) / 1e9, 3),
                                   "path": "sc_two_pass_inplace_f32: in place, one pass + halo snapshot"},
                  "workspace": {"ms": round(sp_ms, 4), "value": round(total_px / (sp_ms / 1e3) / 1e9, 3),
                                "path": "sc_two_pass_split_f32: image and scratch (H0), one pass + halo snapshot"}}
        del img, scr

    # ---- config 2 also names the single pass (copy-back on / off): the FP32-bound
    # kernel next to the reference algorithm's FP32 floor (49 ops per sample at 126.7
    # lane-ops per cycle per SM x 148 SMs x the maximum SM clock; tools/fp2_rate.cu),
    # device-resident under the same L2-flush protocol, and end to end through
    # convolve_image on numpy planes (streamed, sc_single_pass_host_f32)
    single = None
    if args.config == "cfg2" and world == 1 and band is not None:
        dense = np.ascontiguousarray(np.multiply.outer(w, w), dtype=np.float32)
        ws_t = torch.zeros_like(src)
        img_t = src.clone()
        W = len(w)
        valid = P * (R - 2 * r) * (C - 2 * r)
        fp_floor_ms = valid * (2 * W * W - 1) / (126.7 * 148 * 1.965e9) * 1e3

        def flushed(fn, n=50):
            for _ in range(3):
                fn()
            ps = []
            for _ in range(n):
                if flush is not None:
                    flush.fill_(1)
                a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_ev.record(stream)
                fn()
                b_ev.record(stream)
                ps.append((a_ev, b_ev))
            torch.cuda.synchronize()
            return statistics.median(a.elapsed_time(b) for a, b in ps)

        nc_ms = flushed(lambda: dev.single_pass(src, dense, ws_t))
        cb_ms = flushed(lambda: dev.single_pass(img_t, dense, ws_t, copy_back=True))
        single = {"fp32_floor_ms": round(fp_floor_ms, 4),
                  "no_copy": {"ms": round(nc_ms, 4), "value": round(total_px / (nc_ms / 1e3) / 1e9, 3),
                              "frac_of_fp32_floor": round(fp_floor_ms / nc_ms, 3)},
                  "copy_back": {"ms": round(cb_ms, 4), "value": round(total_px / (cb_ms / 1e3) / 1e9, 3),
                                "path": "one pass: workspace and image in place"}}
        if args.e2e_steps > 0:
            import time as _time

            from paper_1711_09791_b200 import Algorithm, ConvVariant, Cuda, Image, Plane, SeparableKernel
            from paper_1711_09791_b200 import convolve_image as _convolve

            host = src.cpu().numpy()
            image = Image([Plane(np.ascontiguousarray(pl)) for pl in host])
            wsi = Image([Plane(np.zeros_like(pl)) for pl in host])
            kern = SeparableKernel(w)
            for cb in (False, True):
                var = ConvVariant(Algorithm.SINGLE_PASS_GENERIC, cb)
                _convolve(image, kern, var, Cuda(), workspace=wsi)  # first call: page-locking
                ts = []
                for _ in range(max(args.e2e_steps, 3)):
                    t0 = _time.perf_counter()
                    _convolve(image, kern, var, Cuda(), workspace=wsi)
                    ts.append(_time.perf_counter() - t0)
                ems = min(ts) * 1e3
                single["e2e_copy_back" if cb else "e2e_no_copy"] = {
                    "ms": round(ems, 3), "value": round(total_px / (ems / 1e3) / 1e9, 3),
                    "path": "convolve_image(image, kernel, SINGLE_PASS_GENERIC, Cuda(), workspace=ws) on numpy planes"}
            del host, image, wsi
        del ws_t, img_t
        # the reference package's own single pass on the host cores (config 2
        # also times SINGLE_PASS_UNROLLED5 without copy-back), same image
        sl = import_reference() if not args.no_cpu_baseline else None
        if sl is not None:
            from oracle import oracle as orc

            cores = os.cpu_count() or 1
            hostx = orc.synthetic(P * R * C, wl.seed, wl.kind).reshape(P, R, C)
            rimg = sl.Image([sl.Plane(hostx[pl]) for pl in range(P)])
            rws = sl.Image.zeros(R, C, P)
            rk = sl.SeparableKernel(w)
            rvar = sl.ConvVariant(sl.Algorithm.SINGLE_PASS_UNROLLED5, False)
            rpool = sl.WorkerPool(cores)
            try:
                rplan = sl.StaticChunked(workers=cores)
                sl.convolve_image(rimg, rk, rvar, rplan, workspace=rws, pool=rpool)
                rts = []
                for _ in range(3):
                    t0 = time.perf_counter()
                    sl.convolve_image(rimg, rk, rvar, rplan, workspace=rws, pool=rpool)
                    rts.append(time.perf_counter() - t0)
            finally:
                rpool.close()
            rms = min(rts) * 1e3
            single["cpu_reference"] = {
                "ms": round(rms, 2), "value": round(total_px / (rms / 1e3) / 1e9, 4), "cores": cores,
                "cpu_model": cpu_model(),
                "path": f"sepconv_lab {sl.__version__} convolve_image(SINGLE_PASS_UNROLLED5, no copy-back, "
                        f"StaticChunked({cores})), vectorised"}
            del hostx, rimg, rws

    # ---- N>1 row bands: the same steps with the OTHER halo transport (secondary)
    # (only when the peer transport is the timed one: the NCCL plan then always
    # exists, while a peer stepper built where peer access failed could leave the
    # ranks out of step in its collectives)
    halo_alt = None
    if band is not None and world > 1 and backend == "nccl" and halo == "peer":
        other = "nccl"
        alt = None
        try:
            alt = NcclBandStepper(src, dst, band, w)
            for _ in range(args.warmup):
                alt.step()
            torch.cuda.synchronize()
            dist.barrier()
            a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_ev.record(stream)
            for _ in range(args.steps):
                alt.step()
            b_ev.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([a_ev.elapsed_time(b_ev) / args.steps], device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            alt_ms = float(t.item())
            halo_alt = {"halo": other, "ms_per_step": round(alt_ms, 4),
                        "value": round(total_px / (alt_ms / 1e3) / 1e9, 3)}
        except Exception as exc:  # noqa: BLE001 - secondary evidence only
            halo_alt = {"halo": other, "error": str(exc)[:200]}
        finally:
            if alt is not None:
                alt.close()

    # ---- N>1 row bands: bit-exactness spot check of the timed transport's output
    # against the single-GPU band kernel on the same rows (each rank regenerates its
    # input rows plus halo from the counter-based generator; no data moves)
    band_check = None
    if band is not None and world > 1:
        stepper.step()
        torch.cuda.synchronize()
        ref_in = torch.empty((P, band.in_hi - band.in_lo, C), dtype=torch.float32, device=device)
        for p in range(P):
            dev.fill_synthetic(ref_in[p], wl.seed, wl.kind, offset=p * R * C + band.in_lo * C)
        ref_out = torch.empty_like(dst)
        dev.two_pass_band(ref_in, w, ref_out, global_rows=R, src_row0=band.in_lo, dst_row0=band.lo,
                          out_lo=band.lo, out_hi=band.hi)
        same = torch.equal(ref_out.view(torch.int32), dst.view(torch.int32))
        flag = torch.tensor([1 if same else 0], device=device if backend == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        band_check = ("bit-exact on every rank vs the single-GPU band kernel" if int(flag.item()) == 1
                      else "MISMATCH")
        del ref_in, ref_out
        dist.barrier()

    # ---- end to end through the C-ABI host entry point (pinned host planes)
    e2e = None
    if args.e2e_steps > 0:
        # host planes hold this rank's rows (N=1: the whole image); in place like conv_two_pass
        if band is not None and world == 1:
            host = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
            for p in range(P):
                host[p].copy_(src[p].cpu())
            h2d, d2h = host_chunk_bytes(R, C, P, r, 0, R, 0, R)
            planes = [h for h in host]

            def e2e_step():
                dev.two_pass_host(planes, planes, w, device=local)
        elif band is not None:
            # N>1: each rank streams ITS row band end to end through the C-ABI host
            # entry point: its pinned host copy holds rows [in_lo, in_hi) (owned +
            # halo), so the halo comes from host memory and no GPU exchange is needed
            hrows = torch.empty((P, band.in_hi - band.in_lo, C), dtype=torch.float32, device=device)
            for p in range(P):
                dev.fill_synthetic(hrows[p], wl.seed, wl.kind, offset=p * R * C + band.in_lo * C)
            hb = [torch.empty((band.in_hi - band.in_lo, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
            for p in range(P):
                hb[p].copy_(hrows[p].cpu())
            del hrows
            h2d, d2h = host_chunk_bytes(R, C, P, r, band.lo, band.hi, band.in_lo, band.in_hi)

            def e2e_step():
                dev.two_pass_host_band(hb, hb, w, global_rows=R, row0=band.in_lo, out_lo=band.lo, out_hi=band.hi,
                                       device=local)
        else:
            # frame batch: every frame-plane is one host plane of the reference's
            # Image; the C-ABI host entry point streams them all (in place)
            hb = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
            hb.copy_(src)
            planes = list(hb.view(-1, R, C).unbind(0))
            h2d = d2h = 0
            for _p in planes:
                a_, b_ = host_chunk_bytes(R, C, 1, r, 0, R, 0, R, call_planes=len(planes))
                h2d += a_
                d2h += b_

            def e2e_step():
                dev.two_pass_host(planes, planes, w, device=local)
        e2e_step()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        e_ms = (time.perf_counter() - t0) * 1e3 / args.e2e_steps
        if world > 1:
            t = torch.tensor([e_ms], device=device if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
            # bytes over PCIe per step for the whole job (every rank's own copies)
            tb = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64,
                              device=device if backend == "nccl" else "cpu")
            dist.all_reduce(tb, op=dist.ReduceOp.SUM)
            h2d, d2h = int(tb[0].item()), int(tb[1].item())
        e2e = {"value": round(total_px / (e_ms / 1e3) / 1e9, 4), "unit": "Gpix/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e_ms, 3),
               "path": "sc_two_pass_host_f32 (pinned host planes, chunked H2D/kernel/D2H on 3 streams)"
               if (world == 1 or band is None) else
               "sc_two_pass_host_band_f32 per rank (its row band + halo rows from its pinned host copy, chunked "
               "H2D/kernel/D2H on 3 streams)"}
        if band is not None and world == 1:
            # the PCIe floor of this step on this box: the same planes' plain pinned
            # H2D alone and D2H alone (one cudaMemcpyAsync per plane, CUDA events);
            # the duplex step cannot beat the slower direction
            def copy_ms(fn):
                fn()
                torch.cuda.synchronize()
                a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_ev.record(stream)
                fn()
                b_ev.record(stream)
                torch.cuda.synchronize()
                return a_ev.elapsed_time(b_ev)

            scratch_dev = torch.empty_like(src)
            h2d_ms = copy_ms(lambda: [scratch_dev[p].copy_(host[p], non_blocking=True) for p in range(P)])
            d2h_ms = copy_ms(lambda: [host[p].copy_(scratch_dev[p], non_blocking=True) for p in range(P)])
            # both directions at once (the step's real floor: the link is not fully duplex)
            back = [torch.empty((R, C), dtype=torch.float32, pin_memory=True) for _ in range(P)]
            s_up, s_down = torch.cuda.Stream(), torch.cuda.Stream()

            def duplex():
                for p in range(P):
                    with torch.cuda.stream(s_up):
                        scratch_dev[p].copy_(host[p], non_blocking=True)
                    with torch.cuda.stream(s_down):
                        back[p].copy_(src[p], non_blocking=True)

            duplex()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            duplex()
            torch.cuda.synchronize()
            dup_ms = (time.perf_counter() - t0) * 1e3
            del scratch_dev, back
            e2e.update({"pcie_h2d_alone_ms": round(h2d_ms, 3), "pcie_d2h_alone_ms": round(d2h_ms, 3),
                        "pcie_duplex_ms": round(dup_ms, 3), "frac_of_pcie_duplex": round(dup_ms / e_ms, 4)})

    # ---- end to end as a sepconv_lab user makes the call: the reference's own
    # convolve_image with the Cuda plan (plugin.py) on its numpy (PAGEABLE) planes,
    # no workspace (the reference's internal one is unobservable: fused path), in
    # place; the library stages pageable rows through its pinned ring
    e2e_pageable = None
    if args.e2e_steps > 0 and band is not None and world == 1:
        if "host" in locals():
            del host, planes  # noqa: F821 - release the pinned copies first
        sl = import_reference()
        from paper_1711_09791_b200 import plugin
        from paper_1711_09791_b200.executors import Cuda

        pg = np.empty((P, R, C), dtype=np.float32)
        for p in range(P):
            pg[p] = src[p].cpu().numpy()
        if sl is not None:
            plugin.install(sl)
            img = sl.Image([sl.Plane(pg[p]) for p in range(P)])
            kern, var = sl.SeparableKernel(w), sl.ConvVariant(sl.Algorithm.TWO_PASS)
            call = "sepconv_lab.convolve_image(image, kernel, TWO_PASS, Cuda()) with the plugin installed"
        else:
            import paper_1711_09791_b200 as pkg

            img = pkg.Image([pkg.Plane(pg[p]) for p in range(P)])
            kern, var = pkg.SeparableKernel(w), pkg.ConvVariant(pkg.Algorithm.TWO_PASS)
            call = "paper_1711_09791_b200.convolve_image(image, kernel, TWO_PASS, Cuda())"
        conv = sl.convolve_image if sl is not None else pkg.convolve_image
        h2d, d2h = host_chunk_bytes(R, C, P, r, 0, R, 0, R)

        def timed(plan, n):
            t0 = time.perf_counter()
            for _ in range(n):
                conv(img, kern, var, plan)
            return (time.perf_counter() - t0) * 1e3 / n

        # (a) the default plan: the image's buffer is page-locked on the first call
        # (timed on its own) and stays registered while it lives, so later calls DMA
        # straight from it
        first_ms = timed(Cuda(device=local), 1)
        # (buffers below 64 MB are staged on first use and page-locked when they come
        # back: the second call pays it, also untimed)
        second_ms = timed(Cuda(device=local), 1)
        reg_ms = timed(Cuda(device=local), args.e2e_steps)
        # (b) never registered: every call stages through the pinned ring
        from paper_1711_09791_b200.device import host_registry

        host_registry.clear()
        staged = Cuda(device=local, register_host=False)
        timed(staged, 1)
        st_ms = timed(staged, args.e2e_steps)
        e2e_pageable = {"value": round(total_px / (reg_ms / 1e3) / 1e9, 4), "unit": "Gpix/s",
                        "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(reg_ms, 3),
                        "first_call_ms": round(first_ms, 3), "second_call_ms": round(second_ms, 3),
                        "path": call + " on pageable numpy planes; the buffer is page-locked on the first call "
                                       "(64 MB and more; smaller ones on the second) and kept registered while it lives",
                        "staged": {"value": round(total_px / (st_ms / 1e3) / 1e9, 4), "ms_per_step": round(st_ms, 3),
                                   "path": "Cuda(register_host=False): every call through the library's pinned "
                                           "staging ring (host copy threads, non-temporal stores)"}}
        if e2e:
            e2e_pageable["frac_of_pinned"] = round(e2e_pageable["value"] / e2e["value"], 4)
            e2e_pageable["staged"]["frac_of_pinned"] = round(e2e_pageable["staged"]["value"] / e2e["value"], 4)
        ndev = torch.cuda.device_count()
        if ndev > 1:
            # one process driving every visible GPU (the reference's plans are
            # single-process): row bands streamed through each GPU's own PCIe link
            multi_plan = Cuda(devices=tuple(range(ndev)))
            timed(multi_plan, 1)
            m_ms = timed(multi_plan, args.e2e_steps)
            e2e_pageable["devices"] = {"n": ndev, "value": round(total_px / (m_ms / 1e3) / 1e9, 4),
                                       "ms_per_step": round(m_ms, 3),
                                       "path": f"Cuda(devices=range({ndev})): sc_two_pass_host_multi_f32"}
        del img, pg
        if sl is not None:
            plugin.uninstall()  # the CPU baseline below runs the unmodified reference

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl)

    if rank == 0:
        eff = 2 * 4 * P * total_px / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Gpix/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak" if wl.frames > 1 else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": workload_config(wl, world),
            **({"halo": halo} if band is not None and world > 1 else {}),
            **({"halo_alt": halo_alt} if halo_alt is not None else {}),
            **({"band_check": band_check} if band_check is not None else {}),
            **({"dropin_device": dropin} if dropin is not None else {}),
            **({"single_pass": single} if single is not None else {}),
            "effective_GBps": round(eff, 1), "pct_of_8TBps": round(100 * eff / NOMINAL_HBM_GBPS, 2),
            "pct_of_measured_copy": round(100 * eff / peak, 2),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "e2e_pageable": e2e_pageable,
            "gpu_launches": int(launches),
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        if band is not None and stepper is not None and hasattr(stepper, "close"):
            stepper.close()  # barriers before unmapping: exporters outlive importers
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
