"""In-kernel halo reads from neighbouring bands (multi-GPU without an exchange
step): the band kernel fetches the r halo rows straight from the adjacent bands'
memory. Bit-identical to the whole-image two-pass.

On this one-GPU pool the neighbours are (a) other tensors in the same process
and (b) another PROCESS's buffers mapped with CUDA IPC (the same mechanism as
across GPUs, minus NVLink). The bands are written and synchronised before any
kernel runs, so no kernel ever waits on another."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device

    return device


@pytest.mark.parametrize("R,C,world,taps,extended", [
    (300, 1000, 3, [1, 4, 6, 4, 1], False),
    (301, 999, 4, [-1, -2, 7, -2, -1], True),     # unaligned rows (generic producer)
    (64, 256, 8, [0.25, 0.5, 0.25], False),
    (97, 130, 5, [1, 2, 3, 4, 5, 4, 3, 2, 1], False),
    (40, 64, 2, [0.1, 0.2, 0.4, 0.2, 0.1, 0.3, 0.7], True),
])
def test_peer_bands_match_whole_image(dev, R, C, world, taps, extended):
    from paper_1711_09791_b200.multi import band_plan

    w = np.asarray(taps, dtype=np.float32)
    w /= w.sum()
    x = dev.synthetic((3, R, C), 11, 1)
    want = dev.two_pass(x, w, extended=extended).cpu().numpy()
    r = len(w) // 2
    bands = [band_plan(R, k, world, r) for k in range(world)]
    owned = [x[:, b.lo:b.hi].clone() for b in bands]  # each band its own buffer, owned rows only
    got = np.empty_like(want)
    for k, b in enumerate(bands):
        out = torch.full((3, b.hi - b.lo, C), float("nan"), device="cuda")
        above = dev.PeerRows.of(owned[k - 1], bands[k - 1].lo) if k > 0 else None
        below = dev.PeerRows.of(owned[k + 1], bands[k + 1].lo) if k < world - 1 else None
        dev.two_pass_band_peer(owned[k], w, out, global_rows=R, src_row0=b.lo, dst_row0=b.lo, out_lo=b.lo,
                               out_hi=b.hi, above=above, below=below, extended=extended)
        got[:, b.lo:b.hi] = out.cpu().numpy()
    assert np.array_equal(_bits(got), _bits(want))


def test_peer_band_validation(dev):
    from paper_1711_09791_b200.errors import InvalidArgumentError

    w = np.array([1, 4, 6, 4, 1], np.float32) / 16
    x = dev.synthetic((3, 60, 64), 1, 1)
    top, mid = x[:, :20].clone(), x[:, 20:40].clone()
    out = torch.empty((3, 20, 64), device="cuda")
    with pytest.raises(InvalidArgumentError):  # no halo source for rows 18, 19
        dev.two_pass_band_peer(mid, w, out, global_rows=60, src_row0=20, dst_row0=20, out_lo=20, out_hi=40)
    with pytest.raises(InvalidArgumentError):  # the band above must end at src_row0
        dev.two_pass_band_peer(mid, w, out, global_rows=60, src_row0=20, dst_row0=20, out_lo=20, out_hi=40,
                               above=dev.PeerRows.of(top[:, :18], 0))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ipc_worker(rank, world, port, R, C, q):
    import torch.distributed as dist

    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.multi import PeerBandStepper, band_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        w = np.array([-1, -2, 7, -2, -1], np.float32)
        x = dev.synthetic((3, R, C), 5, 2)  # every rank can regenerate the image: check its own band
        want = dev.two_pass(x, w).cpu().numpy()
        band = band_plan(R, rank, world, 2)
        src = x[:, band.lo:band.hi].clone()
        dst = torch.full_like(src, float("nan"))
        del x
        # ranks share the one GPU here: no device-side waits between their kernels
        # (B200_PROFILING.md: kernels that wait on one another must not share a GPU)
        stepper = PeerBandStepper(src, dst, band, w, signal=False)
        stepper.sync()          # every band written before any kernel reads a neighbour
        for _ in range(3):
            stepper.step()      # inputs fixed across steps: no per-step synchronisation needed
        torch.cuda.synchronize()
        ok = np.array_equal(_bits(dst.cpu().numpy()), _bits(want[:, band.lo:band.hi]))
        dist.barrier()          # neighbours stop reading before anyone unmaps / frees
        stepper.close()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_stepper_over_cuda_ipc(world):
    """Each process maps its neighbours' band buffers with CUDA IPC; one launch per
    step reads the halo rows from them. Result: the whole-image bits."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, 203, 1024, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(results[r] for r in range(world)), results


@pytest.mark.parametrize("halo", ["peer", "nccl"])
def test_bench_two_ranks_on_one_gpu(halo):
    """bench.py's N>1 row-band step, both halo transports, as 2 torchrun ranks
    sharing this GPU (gloo for the host-side collectives; NCCL mode stages the
    halo through host memory). It must print one well-formed JSON line."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import json
    import subprocess
    import sys

    from conftest import ROOT

    port = _free_port()
    env = dict(os.environ, SEPCONV_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
           "cfg3", "--steps", "5", "--warmup", "3", "--e2e-steps", "1", "--halo", halo]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["halo"] == halo and line["value"] > 0
    assert line["gpu_launches"] >= 5 and line["e2e"]["value"] > 0
    assert line["band_check"].startswith("bit-exact"), line["band_check"]
    assert line["config"]["parallelism"] == "rowband2"


@pytest.mark.parametrize("world,extended", [(3, False), (4, True)])
def test_band_split_mode_on_gpu(dev, oracle, world, extended):
    """band_two_pass_split with the CUDA row/column passes on every band of one
    image (halo rows pre-filled, as the exchange would): owned image and scratch
    rows equal the reference's end state."""
    from paper_1711_09791_b200.multi import band_plan, band_two_pass_split

    R, C = 203, 517
    w = np.array([-1, -2, 7, -2, -1], np.float32)
    full = dev.synthetic((3, R, C), 3, 2)
    fh = full.cpu().numpy()
    want_img = oracle.two_pass(fh, w, extended=extended)
    want_scr = oracle.two_pass_scratch(fh, w, extended=extended)
    for k in range(world):
        b = band_plan(R, k, world, 2)
        local = full[:, b.in_lo:b.in_hi].clone()
        scratch = torch.full_like(local, float("nan"))  # zero fill must overwrite everything
        band_two_pass_split(local, scratch, b, w, extended=extended, exchange=False)
        own = slice(b.lo - b.in_lo, b.hi - b.in_lo)
        assert np.array_equal(_bits(local[:, own].cpu().numpy()), _bits(want_img[:, b.lo:b.hi]))
        assert np.array_equal(_bits(scratch[:, own].cpu().numpy()), _bits(want_scr[:, b.lo:b.hi]))


def _probe_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1711_09791_b200.multi import peer_transport_works

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        q.put((rank, peer_transport_works()))
    finally:
        dist.destroy_process_group()


def test_peer_transport_probe_agrees():
    """bench.py's one-time probe (peer halo reads vs send/recv exchange on a tiny
    banded image) returns True on every rank when the IPC mapping works."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_probe_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    results = dict(q.get(timeout=5) for _ in range(3))
    assert all(results.values()), results


def test_peer_rows_in_host_mapped_memory(dev):
    """The halo rows' bulk copies also work when the neighbouring bands live in
    pinned HOST memory (mapped into the device address space over PCIe): the TMA
    engine reading non-local memory through the fabric, as it does for a peer
    GPU's HBM over NVLink."""
    from paper_1711_09791_b200.multi import band_plan

    R, C, world = 120, 1024, 3
    w = np.array([-1, -2, 7, -2, -1], np.float32)
    x = dev.synthetic((3, R, C), 21, 2)
    want = dev.two_pass(x, w).cpu().numpy()
    bands = [band_plan(R, k, world, 2) for k in range(world)]
    host = [x[:, b.lo:b.hi].cpu().pin_memory() for b in bands]  # every band in pinned host memory
    b = bands[1]
    own = x[:, b.lo:b.hi].clone()
    out = torch.full_like(own, float("nan"))
    above = dev.PeerRows(host[0].data_ptr(), bands[0].lo, bands[0].hi - bands[0].lo, host[0].stride(0),
                         host[0].stride(1), keep=host[0])
    below = dev.PeerRows(host[2].data_ptr(), bands[2].lo, bands[2].hi - bands[2].lo, host[2].stride(0),
                         host[2].stride(1), keep=host[2])
    dev.two_pass_band_peer(own, w, out, global_rows=R, src_row0=b.lo, dst_row0=b.lo, out_lo=b.lo, out_hi=b.hi,
                           above=above, below=below)
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(want[:, b.lo:b.hi]))


@pytest.mark.parametrize("world,R,C", [(3, 301, 999), (4, 200, 1024)])
def test_host_band_streaming(dev, oracle, world, R, C):
    """sc_two_pass_host_band_f32: each rank's band streamed from ITS host copy of
    rows [in_lo, in_hi) (in place), 16-row chunks; stitched == the whole image."""
    from paper_1711_09791_b200.multi import band_plan

    w = np.array([1, 4, 6, 4, 1], np.float32) / 16
    rng = np.random.default_rng(R)
    x = rng.uniform(-50, 50, size=(3, R, C)).astype(np.float32)
    want = oracle.two_pass(x, w)
    got = np.empty_like(want)
    os.environ["SC_HOST_CHUNK_MB"] = "0"  # 16-row chunks: many seams inside each band
    try:
        for k in range(world):
            b = band_plan(R, k, world, 2)
            hb = [torch.from_numpy(np.ascontiguousarray(x[p, b.in_lo:b.in_hi])).pin_memory() for p in range(3)]
            dev.two_pass_host_band(hb, hb, w, global_rows=R, row0=b.in_lo, out_lo=b.lo, out_hi=b.hi)
            for p in range(3):
                got[p, b.lo:b.hi] = hb[p].numpy()[b.lo - b.in_lo:b.hi - b.in_lo]
    finally:
        del os.environ["SC_HOST_CHUNK_MB"]
    assert np.array_equal(_bits(got), _bits(want))
