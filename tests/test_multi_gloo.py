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


def _meta_worker(rank, world, port, R, q):
    import torch.distributed as dist

    from paper_1711_09791_b200.multi import PeerMeta, band_plan, peer_neighbours, publish_peer_meta

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        band = band_plan(R, rank, world, 2)
        handle = bytes([rank]) * 64  # stands in for the CUDA IPC handle
        me = PeerMeta(rank, band.lo, band.hi, handle, 128 * rank, 7 * R, 7, 7, 3)
        above, below = peer_neighbours(publish_peer_meta(me, band), band)
        ok = (above is None) == (rank == 0) and (below is None) == (rank == world - 1)
        if above is not None:
            ok = ok and above.rank == rank - 1 and above.hi == band.lo and above.handle == bytes([rank - 1]) * 64
            ok = ok and above.offset == 128 * (rank - 1)
        if below is not None:
            ok = ok and below.rank == rank + 1 and below.lo == band.hi and below.handle == bytes([rank + 1]) * 64
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_metadata_exchange(world):
    """The peer (in-kernel halo) path's only host collective: every rank publishes
    its band buffer's IPC handle + geometry and picks its two neighbours."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_meta_worker, args=(r, world, port, 41, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results


def test_peer_neighbour_validation():
    from paper_1711_09791_b200.errors import InvalidArgumentError
    from paper_1711_09791_b200.multi import PeerMeta, band_plan, peer_neighbours

    R, world = 30, 3
    bands = [band_plan(R, r, world, 2) for r in range(world)]
    metas = [PeerMeta(b.rank, b.lo, b.hi, b"\0" * 64, 0, 100, 10, 10, 3) for b in bands]
    above, below = peer_neighbours(metas, bands[1])
    assert (above.rank, below.rank) == (0, 2)
    assert peer_neighbours(metas, bands[0])[0] is None and peer_neighbours(metas, bands[2])[1] is None
    with pytest.raises(InvalidArgumentError):  # a gap between bands
        peer_neighbours([metas[0], PeerMeta(1, 11, 20, b"\0" * 64, 0, 100, 10, 10, 3), metas[2]], bands[1])
    with pytest.raises(InvalidArgumentError):  # width mismatch
        peer_neighbours([metas[0], metas[1], PeerMeta(2, 20, 30, b"\0" * 64, 0, 100, 10, 11, 3)], bands[1])
    with pytest.raises(InvalidArgumentError):  # missing neighbour
        peer_neighbours([metas[1], metas[2]], bands[1])


def _split_worker(rank, world, port, R, C, P, taps, extended, q):
    import torch.distributed as dist

    from oracle import oracle as orc
    from paper_1711_09791_b200.multi import band_plan, band_two_pass_split

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = np.asarray(taps, dtype=np.float32)
        full = orc.synthetic(P * R * C, 17, kind=2).reshape(P, R, C)
        band = band_plan(R, rank, world, len(w) // 2)
        local = torch.full((P, band.local_rows, C), float("nan"))
        local[:, band.owned] = torch.from_numpy(full[:, band.lo:band.hi])
        scratch = torch.zeros((P, band.local_rows, C))  # the reference's zero workspace

        def hp(s, d, lo, hi):
            for p in range(P):
                orc.horizontal_rows(s[p].numpy(), d[p].numpy(), w, lo, hi)

        def vp(s, d, lo, hi):
            for p in range(P):
                orc.vertical_rows(s[p].numpy(), d[p].numpy(), w, lo, hi)

        band_two_pass_split(local, scratch, band, w, extended=extended, hpass_fn=hp, vpass_fn=vp)
        own = slice(band.lo - band.in_lo, band.hi - band.in_lo)
        want_img = orc.two_pass(full, w, extended=extended)[:, band.lo:band.hi]
        want_scr = orc.two_pass_scratch(full, w, extended=extended)[:, band.lo:band.hi]
        ok = np.array_equal(local[:, own].numpy().view(np.uint32), want_img.view(np.uint32))
        ok = ok and np.array_equal(scratch[:, own].numpy().view(np.uint32), want_scr.view(np.uint32))
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,R,extended", [(2, 37, False), (3, 41, True), (4, 23, False)])
def test_band_split_mode_matches_reference_state(world, R, extended):
    """Split two-pass (K2 + K3) on row bands: owned image rows AND owned scratch
    rows equal the reference's end state bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    taps = [-1.0, -2.0, 7.0, -2.0, -1.0]
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, R, 29, 3, taps, extended, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(results[r] for r in range(world)), results
