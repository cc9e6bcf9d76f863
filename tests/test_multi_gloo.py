"""Multi-rank row-band path on CPU: world_size 2/3/4 processes over gloo, the
real halo exchange (torch.distributed batch_isend_irecv) and the band
orchestration of paper_1711_09791_b200.multi, with the C oracle's band function
standing in for the GPU kernel. The banded result must equal the whole-image
reference bits."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, R, C, P, taps, extended, overlap, q):
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1711_09791_b200.multi import band_plan, band_two_pass

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = np.asarray(taps, dtype=np.float32)
        full = orc.synthetic(P * R * C, 99, kind=2).reshape(P, R, C)
        band = band_plan(R, rank, world, len(w) // 2)
        local = torch.full((P, band.local_rows, C), float("nan"))
        local[:, band.owned] = torch.from_numpy(full[:, band.lo:band.hi])
        out = torch.zeros((P, band.hi - band.lo, C))
        band_two_pass(local, out, band, w, extended=extended, band_fn=orc.two_pass_band, overlap=overlap)
        want = orc.two_pass(full, w, extended=extended)[:, band.lo:band.hi]
        ok = np.array_equal(out.numpy().view(np.uint32), want.view(np.uint32))
        # a prepared op list is reused every step (BandStepper): exchange twice more
        from paper_1711_09791_b200.multi import halo_ops

        ops = halo_ops(local, band)
        for _ in range(2):
            local[:, : band.owned.start] = float("nan")
            local[:, band.owned.stop :] = float("nan")
            if ops:
                for wk in dist.batch_isend_irecv(ops):
                    wk.wait()
            ok = ok and np.array_equal(local.numpy(), full[:, band.in_lo : band.in_hi])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,R,extended,overlap", [
    (2, 37, False, True), (3, 41, True, True), (4, 23, False, False), (2, 9, False, True),
])
def test_band_exchange_matches_whole_image(world, R, extended, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    taps = [-1.0, -2.0, 7.0, -2.0, -1.0]
    procs = [ctx.Process(target=_worker, args=(r, world, port, R, 29, 3, taps, extended, overlap, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results


def test_band_plan_rules():
    from paper_1711_09791_b200.errors import InvalidArgumentError
    from paper_1711_09791_b200.multi import band_plan, frame_shard

    b = band_plan(16384, 3, 8, 2)
    assert (b.lo, b.hi, b.in_lo, b.in_hi) == (6144, 8192, 6142, 8194)
    assert b.local_rows == 2052 and b.owned == slice(2, 2050)
    first, last = band_plan(16384, 0, 8, 2), band_plan(16384, 7, 8, 2)
    assert first.in_lo == 0 and last.in_hi == 16384
    # every row is owned exactly once
    owned = np.zeros(1001, dtype=int)
    for r in range(7):
        bb = band_plan(1001, r, 7, 2)
        owned[bb.lo:bb.hi] += 1
    assert (owned == 1).all()
    with pytest.raises(InvalidArgumentError):
        band_plan(10, 0, 8, 2)  # bands shorter than the radius
    assert [frame_shard(512, r, 8) for r in (0, 7)] == [(0, 64), (448, 512)]
    assert sum(b - a for a, b in (frame_shard(513, r, 4) for r in range(4))) == 513
