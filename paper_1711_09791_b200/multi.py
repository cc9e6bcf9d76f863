"""Multi-GPU partitioner: one process per GPU.

Row bands (configs 3 and 5). Rank g owns output rows
partition_block(0, R, g, n) of every plane and holds input rows
[lo - r, hi + r) clipped to the image. Output row y needs row-pass rows y-r..y+r
and the row pass is row-local, so the only exchange is r input rows with each
neighbour: ONE batched NCCL send/recv group per step (torch.distributed P2P over
NVLink/NVSwitch). The interior rows [lo + r, hi - r) depend on owned rows only and
run while the halos are in flight; the 2r boundary rows run after they land. The
faithful zero-row rule and the ring use GLOBAL row indices, so the banded result
is bit-identical to the single-GPU one.

Frame batches (config 4): frames are independent; partition_block shards them
with no communication at all.

The exchange and the orchestration are backend-agnostic (NCCL on GPUs, gloo on
CPU tensors for the world_size-2 tests); the per-band compute is a callable,
by default the fused kernel's band entry point.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch

from .errors import InvalidArgumentError


def partition_block(lo: int, hi: int, index: int, cutoff: int) -> tuple[int, int]:
    """The index-th of `cutoff` near-equal contiguous chunks of [lo, hi).

    Restates the reference's balanced split (S/executors.py:121-139): the first
    (n mod cutoff) chunks get one extra element; sizes differ by at most one.
    """
    if lo > hi:
        raise InvalidArgumentError(f"range bounds out of order: [{lo}, {hi})")
    if cutoff < 1:
        raise InvalidArgumentError(f"cutoff must be >= 1, got {cutoff}")
    if not 0 <= index < cutoff:
        raise InvalidArgumentError(f"chunk index {index} outside [0, {cutoff})")
    q, s = divmod(hi - lo, cutoff)
    if index < s:
        start = lo + index * (q + 1)
        return start, start + q + 1
    start = lo + s * (q + 1) + (index - s) * q
    return start, start + q


@dataclass(frozen=True)
class Band:
    """Rank `rank` of `world`: owned output rows [lo, hi) of a `rows`-tall image,
    held input rows [in_lo, in_hi) (owned rows plus up to `radius` halo rows)."""

    rank: int
    world: int
    rows: int
    radius: int
    lo: int
    hi: int

    @property
    def in_lo(self) -> int:
        return max(self.lo - self.radius, 0)

    @property
    def in_hi(self) -> int:
        return min(self.hi + self.radius, self.rows)

    @property
    def local_rows(self) -> int:
        return self.in_hi - self.in_lo

    @property
    def owned(self) -> slice:
        """Owned rows inside the local (held-rows) buffer."""
        return slice(self.lo - self.in_lo, self.hi - self.in_lo)

    @property
    def halo_bytes_per_plane_col(self) -> int:
        """float32 bytes received per plane per column per step."""
        return 4 * ((self.lo - self.in_lo) + (self.in_hi - self.hi))


def band_plan(rows: int, rank: int, world: int, radius: int) -> Band:
    """Row band of `rank`; every band must be at least `radius` rows tall so that a
    halo comes from the adjacent rank only."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgumentError(f"rank {rank} outside world of {world}")
    lo, hi = partition_block(0, rows, rank, world)
    smallest = rows // world
    if world > 1 and smallest < max(radius, 1):
        raise InvalidArgumentError(
            f"{rows} rows over {world} ranks gives bands of {smallest} rows; need >= {max(radius, 1)}"
        )
    return Band(rank, world, rows, radius, lo, hi)


def frame_shard(frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [f0, f1) of a batch handled by `rank` (config 4; no communication)."""
    return partition_block(0, frames, rank, world)


def halo_ops(local, band: Band, group=None):
    """The P2P operations of one halo exchange for the held-rows buffer `local`
    ((P, band.local_rows, C)): send the first/last r owned rows of every plane to
    the neighbours, receive theirs into the halo rows. Reusable across steps."""
    import torch.distributed as dist

    if band.world == 1:
        return []
    ops = []
    top = band.lo - band.in_lo      # halo rows above (0 for rank 0)
    bot = band.in_hi - band.hi      # halo rows below (0 for the last rank)
    o0, o1 = band.owned.start, band.owned.stop
    for p in range(local.shape[0]):
        if band.rank > 0 and top > 0:
            ops.append(dist.P2POp(dist.isend, local[p, o0 : o0 + top], band.rank - 1, group=group))
            ops.append(dist.P2POp(dist.irecv, local[p, 0:top], band.rank - 1, group=group))
        if band.rank < band.world - 1 and bot > 0:
            ops.append(dist.P2POp(dist.isend, local[p, o1 - bot : o1], band.rank + 1, group=group))
            ops.append(dist.P2POp(dist.irecv, local[p, o1 : o1 + bot], band.rank + 1, group=group))
    return ops


def exchange_halos(local, band: Band, group=None):
    """Fill the halo rows of `local` from the neighbours' owned rows with ONE
    batched send/recv group (NCCL: one grouped launch over NVLink). Returns the
    async works (wait on them before reading the halo rows)."""
    import torch.distributed as dist

    ops = halo_ops(local, band, group)
    return dist.batch_isend_irecv(ops) if ops else []


BandFn = Callable[..., object]


def _default_band_fn(src, dst, *, global_rows, src_row0, dst_row0, out_lo, out_hi, taps, extended,
                     out_lo2=0, out_hi2=0):
    from . import device

    return device.two_pass_band(src, taps, dst, global_rows=global_rows, src_row0=src_row0, dst_row0=dst_row0,
                                out_lo=out_lo, out_hi=out_hi, extended=extended, out_lo2=out_lo2, out_hi2=out_hi2)


def band_two_pass(local_src, local_dst, band: Band, taps, *, extended: bool = False, group=None,
                  band_fn: BandFn | None = None, overlap: bool = True) -> None:
    """One step of the banded fused two-pass.

    local_src: (P, band.local_rows, C) held input rows (owned rows filled, halo
    rows overwritten by the exchange). local_dst: (P, hi - lo, C) owned output rows.
    """
    fn = band_fn or _default_band_fn
    r = band.radius
    common = dict(global_rows=band.rows, src_row0=band.in_lo, dst_row0=band.lo, taps=taps, extended=extended)
    works = exchange_halos(local_src, band, group)
    # interior output rows read owned input rows only: run them while halos fly
    i_lo = band.lo + (r if band.rank > 0 else 0)
    i_hi = band.hi - (r if band.rank < band.world - 1 else 0)
    if not overlap or i_lo >= i_hi:
        for w in works:
            w.wait()
        fn(local_src, local_dst, out_lo=band.lo, out_hi=band.hi, **common)
        return
    fn(local_src, local_dst, out_lo=i_lo, out_hi=i_hi, **common)
    for w in works:
        w.wait()
    # both boundary strips (top r rows, bottom r rows) in ONE launch
    if band_fn is None:
        fn(local_src, local_dst, out_lo=band.lo, out_hi=i_lo, out_lo2=i_hi, out_hi2=band.hi, **common)
        return
    if i_lo > band.lo:
        fn(local_src, local_dst, out_lo=band.lo, out_hi=i_lo, **common)
    if i_hi < band.hi:
        fn(local_src, local_dst, out_lo=i_hi, out_hi=band.hi, **common)


def band_two_pass_split(local, scratch, band: Band, taps, *, extended: bool = False, group=None,
                        exchange: bool = True, hpass_fn=None, vpass_fn=None) -> None:
    """The two-pass SPLIT mode (K2 + K3) on a row band, in place, with the
    reference's buffer end state (third row; conv_two_pass,
    S/conv.py:392-421): after the halo exchange, the row pass fills the band's
    scratch with H0 (zero outside the live rows and on the column ring; the halo
    rows' H0 is recomputed locally -- the row pass is row-local), then the column
    pass writes V(H0) into the owned rows of `local`. Owned rows of `local` end as
    the reference's image, owned rows of `scratch` as its workspace.

    local, scratch: (P, band.local_rows, C). hpass_fn(src, dst, row_lo, row_hi) /
    vpass_fn(src, dst, row_lo, row_hi) work on band-local rows (defaults: the
    CUDA row and column passes; the CPU tests pass the oracle's)."""
    r = band.radius
    if hpass_fn is None or vpass_fn is None:
        from . import device

        hpass_fn = hpass_fn or (lambda s, d, lo, hi: device.hpass(s, taps, d, lo, hi, zero_fill=True))
        vpass_fn = vpass_fn or (lambda s, d, lo, hi: device.vpass(s, taps, d, lo, hi))
    if exchange:
        for w in exchange_halos(local, band, group):
            w.wait()
    live_lo, live_hi = (0, band.rows) if extended else (r, band.rows - r)
    h_lo = max(live_lo, band.in_lo) - band.in_lo
    h_hi = min(live_hi, band.in_hi) - band.in_lo
    hpass_fn(local, scratch, h_lo, max(h_lo, h_hi))
    v_lo = max(band.lo, r) - band.in_lo
    v_hi = min(band.hi, band.rows - r) - band.in_lo
    if v_hi > v_lo:
        vpass_fn(scratch, local, v_lo, v_hi)


class BandStepper:
    """Prepared banded two-pass step for a fixed pair of band buffers.

    Same work as `band_two_pass` (one batched halo exchange, the interior rows
    overlapped with it, then both boundary strips in one launch) with the
    per-step host work cut to the bare C-ABI calls: the ctypes argument tuples,
    the P2P op list and the stream handle are built once. At 8 GPUs a config-5
    step is ~0.13 ms of GPU time, so host overhead per step matters.
    """

    def __init__(self, local_src, local_dst, band: Band, taps, *, extended: bool = False, group=None,
                 host_staged: bool | None = None):
        from . import _lib
        from . import device as dev

        self.band = band
        self.src, self.dst = local_src, local_dst
        self._lib = _lib.load()
        self._check = _lib.check
        w = dev._taps(taps)
        self._w = w  # keep alive
        wp = w.ctypes.data  # const float* taps (kept alive by self._w)
        n, Rs, C, sps, srs = dev._planes(local_src, "local_src")
        n2, Rd, C2, dps, drs = dev._planes(local_dst, "local_dst")
        if n2 != n or C2 != C or Rd != band.hi - band.lo or Rs != band.local_rows:
            raise InvalidArgumentError("band buffers do not match the band plan")
        r = band.radius
        i_lo = band.lo + (r if band.rank > 0 else 0)
        i_hi = band.hi - (r if band.rank < band.world - 1 else 0)
        if i_lo >= i_hi:  # tiny band: everything after the exchange
            i_lo = i_hi = band.lo
        stream = torch.cuda.current_stream(local_src.device).cuda_stream
        flags = _lib.SC_EXTENDED if extended else 0
        head = (local_src.data_ptr(), local_dst.data_ptr(), n, band.rows, C, sps, dps, srs, drs, band.in_lo, Rs,
                band.lo)
        tail = (wp, w.size, flags, stream)
        self._interior = head + (i_lo, i_hi, 0, 0) + tail if i_hi > i_lo else None
        if i_hi > i_lo:
            self._boundary = head + (band.lo, i_lo, i_hi, band.hi) + tail
        else:
            self._boundary = head + (band.lo, band.hi, 0, 0) + tail
        # Backends that cannot move CUDA tensors (gloo: used to exercise the
        # multi-rank orchestration on one GPU / in CI) stage the halo rows
        # through host memory; NCCL exchanges device rows directly.
        if host_staged is None:
            import torch.distributed as dist

            host_staged = dist.is_initialized() and dist.get_backend(group) != "nccl" and local_src.is_cuda
        self._staged = host_staged
        if host_staged:
            self._host = torch.empty(local_src.shape, dtype=local_src.dtype, pin_memory=True)
            self._ops = halo_ops(self._host, band, group)
        else:
            self._ops = halo_ops(local_src, band, group)

    def _exchange(self):
        import torch.distributed as dist

        if not self._ops:
            return []
        if not self._staged:
            return dist.batch_isend_irecv(self._ops)
        b = self.band
        o0, o1 = b.owned.start, b.owned.stop
        top, bot = b.lo - b.in_lo, b.in_hi - b.hi
        # owned boundary rows down, exchange on the host, halo rows back up
        self._host[:, o0:o0 + top].copy_(self.src[:, o0:o0 + top])
        self._host[:, o1 - bot:o1].copy_(self.src[:, o1 - bot:o1])
        torch.cuda.current_stream().synchronize()
        for wk in dist.batch_isend_irecv(self._ops):
            wk.wait()
        if top:
            self.src[:, 0:top].copy_(self._host[:, 0:top], non_blocking=True)
        if bot:
            self.src[:, o1:o1 + bot].copy_(self._host[:, o1:o1 + bot], non_blocking=True)
        return []

    def step(self):
        L = self._lib
        works = self._exchange()
        if self._interior is not None:
            self._check(L.sc_two_pass_band2_f32(*self._interior))
        for w in works:
            w.wait()
        self._check(L.sc_two_pass_band2_f32(*self._boundary))

    def kernel_only(self):
        """The whole band in one launch (no exchange): the dominant kernel for the roofline."""
        b = self.band
        args = self._boundary[:12] + (b.lo, b.hi, 0, 0) + self._boundary[16:]
        self._check(self._lib.sc_two_pass_band2_f32(*args))


_COMMS: dict = {}
SIG_WORDS = 8  # the band signal block (csrc/kernels.cuh SIG_WORDS)


def nccl_comm(group=None, device: int | None = None) -> int:
    """The library's own NCCL communicator over the ranks of `group` (cached): rank 0
    draws the unique id (sc_nccl_unique_id), torch.distributed broadcasts it, every
    rank calls sc_nccl_comm_init on its device. A world of one needs no process
    group (the one-GPU tests)."""
    import ctypes

    import torch.distributed as dist

    from . import _lib

    L = _lib.load()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev_index = torch.cuda.current_device() if device is None else int(device)
    key = (id(group), world, rank, dev_index)
    if key in _COMMS:
        return _COMMS[key]
    uid = ctypes.create_string_buffer(128)
    if rank == 0:
        _lib.check(L.sc_nccl_unique_id(uid))
    if world > 1:
        box = [uid.raw if rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
    comm = ctypes.c_void_p(0)
    _lib.check(L.sc_nccl_comm_init(uid, world, rank, dev_index, ctypes.byref(comm)))
    _COMMS[key] = int(comm.value)
    return _COMMS[key]


class NcclBandStepper:
    """The row-band step with the halo exchange in the library (csrc/nccl_band.cu).

    Each rank holds its OWNED rows only, (P, hi - lo, C). Per step: the r boundary
    rows of every plane are packed into ONE buffer per neighbour and exchanged by
    ncclSend/ncclRecv in one group on a communication stream while the interior
    rows compute; then ONE launch produces both boundary strips, reading the halo
    rows from the receive buffers. use_graph=True captures the step
    into a CUDA graph instead of issuing it eagerly (measured: more host time per
    step with NCCL nodes in the graph, so it is off by default)."""

    def __init__(self, local_src, local_dst, band: Band, taps, *, extended: bool = False, group=None,
                 use_graph: bool = False, comm: int | None = None, rank_above: int | None = None,
                 rank_below: int | None = None):
        import ctypes

        from . import _lib
        from . import device as dev

        self.band = band
        self.src, self.dst = local_src, local_dst
        n, Rs, C, sps, srs = dev._planes(local_src, "local_src")
        n2, Rd, C2, dps, drs = dev._planes(local_dst, "local_dst")
        if Rs != band.hi - band.lo or Rd != band.hi - band.lo or n2 != n or C2 != C:
            raise InvalidArgumentError("NCCL band buffers must hold exactly the owned rows")
        if rank_above is None:
            rank_above = band.rank - 1 if band.rank > 0 else -1
        if rank_below is None:
            rank_below = band.rank + 1 if band.rank < band.world - 1 else -1
        self._lib = _lib.load()
        self._check = _lib.check
        w = dev._taps(taps)
        self._w = w
        with torch.cuda.device(local_src.device):
            if comm is None and (rank_above >= 0 or rank_below >= 0):
                comm = nccl_comm(group, local_src.device.index)
            plan = ctypes.c_void_p(0)
            _lib.check(self._lib.sc_band_plan_create(comm or None, local_src.data_ptr(), local_dst.data_ptr(), n,
                                                     band.rows, C, sps, dps, srs, drs, band.lo, band.hi, rank_above,
                                                     rank_below, w.ctypes.data, w.size,
                                                     _lib.SC_EXTENDED if extended else 0, int(bool(use_graph)),
                                                     ctypes.byref(plan)))
        self._plan = plan.value
        self.graphed = bool(self._lib.sc_band_plan_graphed(self._plan))
        self._stream = torch.cuda.current_stream(local_src.device).cuda_stream
        r = band.radius
        i_lo = band.lo + (r if rank_above >= 0 else 0)
        i_hi = band.hi - (r if rank_below >= 0 else 0)
        # the dominant kernel alone (roofline): the interior rows, which need no halo
        self.kernel_rows = (i_lo, i_hi) if i_hi > i_lo else (band.lo, band.lo)
        self._kernel_args = (local_src.data_ptr(), local_dst.data_ptr(), n, band.rows, C, sps, dps, srs, drs,
                             band.lo, Rs, band.lo, i_lo, max(i_lo, i_hi), 0, 0, w.ctypes.data, w.size,
                             _lib.SC_EXTENDED if extended else 0, self._stream)

    def step(self):
        self._check(self._lib.sc_band_plan_step(self._plan, self._stream))

    def kernel_only(self):
        self._check(self._lib.sc_two_pass_band2_f32(*self._kernel_args))

    def close(self):
        if self._plan:
            torch.cuda.current_stream(self.src.device).synchronize()
            self._check(self._lib.sc_band_plan_destroy(self._plan))
            self._plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


@dataclass(frozen=True)
class PeerMeta:
    """What a rank publishes about its band buffer: owned rows [lo, hi) of every
    plane, at (IPC handle, byte offset) with strides in floats."""

    rank: int
    lo: int
    hi: int
    handle: bytes
    offset: int
    plane_stride: int
    row_stride: int
    cols: int
    planes: int
    sig_handle: bytes = b""  # IPC handle + offset of the band's signal words (empty: no signalling)
    sig_offset: int = 0


def peer_neighbours(metas, band: Band) -> tuple[PeerMeta | None, PeerMeta | None]:
    """The metas of the bands directly above and below `band` (None at the image
    edges), checked to be the adjacent, same-geometry bands the kernel expects."""
    by_rank = {m.rank: m for m in metas}
    me = by_rank.get(band.rank)
    if me is None or (me.lo, me.hi) != (band.lo, band.hi):
        raise InvalidArgumentError("own band missing from the published metadata")
    above = by_rank.get(band.rank - 1) if band.rank > 0 else None
    below = by_rank.get(band.rank + 1) if band.rank < band.world - 1 else None
    if band.rank > 0 and (above is None or above.hi != band.lo):
        raise InvalidArgumentError(f"rank {band.rank}: the band above does not end at row {band.lo}")
    if band.rank < band.world - 1 and (below is None or below.lo != band.hi):
        raise InvalidArgumentError(f"rank {band.rank}: the band below does not start at row {band.hi}")
    for nb in (above, below):
        if nb is not None and (nb.cols != me.cols or nb.planes != me.planes):
            raise InvalidArgumentError("neighbouring bands differ in width or plane count")
        if nb is not None and nb.hi - nb.lo < band.radius:
            raise InvalidArgumentError("a neighbouring band is shorter than the kernel radius")
    return above, below


def publish_peer_meta(me: PeerMeta, band: Band, group=None) -> list:
    """Every rank's PeerMeta, in rank order (one all_gather_object)."""
    import torch.distributed as dist

    if band.world == 1:
        return [me]
    metas = [None] * band.world
    dist.all_gather_object(metas, me, group=group)
    return metas


class PeerBandStepper:
    """Banded two-pass with the halo exchange folded into the kernel.

    Each rank keeps only its OWNED input rows (P, hi - lo, C). At construction
    the ranks publish CUDA IPC handles of their band buffers and of three u64
    signal words (one all_gather_object over the process group) and map their two
    neighbours' buffers and words into their own device's address space (peer
    access over NVLink/NVSwitch). A step is then ONE launch: the producer warp's
    TMA row copies read the r halo rows directly from the neighbours' memory,
    tile by tile, as the interior streams -- no send/recv, no staging buffer, no
    second launch for the boundary rows.

    Ordering is device-side (signal=True, the default with neighbours): step e
    is epoch e; every CTA publishes ready = e when it starts and waits for both
    neighbours' ready >= e before it reads or writes, and the last CTA publishes
    done = e (csrc/kernels.cuh wait_signal). So a step on FRESH inputs needs no
    host barrier: a caller that refills its band in place between steps first
    calls `wait_consumed()` (a stream-ordered wait for the neighbours' done), and
    ping-pong buffers (step e writes what the neighbours read in step e-1) need
    nothing at all. `check()` raises if a wait timed out (SC_PEER_TIMEOUT_MS).
    signal=False keeps the old contract: `sync()` is a process-group barrier.
    """

    def __init__(self, local_src, local_dst, band: Band, taps, *, extended: bool = False, group=None,
                 signal: bool = True):
        from . import _lib
        from . import device as dev

        self.band, self.group = band, group
        self.src, self.dst = local_src, local_dst
        n, Rs, C, sps, srs = dev._planes(local_src, "local_src")
        n2, Rd, C2, dps, drs = dev._planes(local_dst, "local_dst")
        if Rs != band.hi - band.lo or Rd != band.hi - band.lo or n2 != n or C2 != C:
            raise InvalidArgumentError("peer band buffers must hold exactly the owned rows")
        self.signal = bool(signal) and band.world > 1
        # signal words (kernels.cuh: [0] ready, [2]/[3] done counts of the items
        # that read the band above/below, [4]/[5] their per-launch targets) in this
        # device's memory; the error word in pinned host memory (read by the host
        # without a sync)
        self.sig = torch.zeros(SIG_WORDS, dtype=torch.int64, device=local_src.device)
        self.err = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.epoch = 0
        if band.world > 1:
            handle, offset = dev.ipc_export(local_src)
            sh, so = dev.ipc_export(self.sig) if self.signal else (b"", 0)
        else:
            handle, offset, sh, so = b"\0" * 64, 0, b"", 0
        me = PeerMeta(band.rank, band.lo, band.hi, handle, offset, sps, srs, C, n, sh, so)
        above, below = peer_neighbours(publish_peer_meta(me, band, group), band)
        self._opened = []
        rows, sigs = {}, {}
        for side, m in (("above", above), ("below", below)):
            rows[side] = sigs[side] = None
            if m is None:
                continue
            ptr = dev.ipc_open(m.handle, m.offset, local_src.device.index)
            self._opened.append((ptr, m.offset))
            rows[side] = dev.PeerRows(ptr, m.lo, m.hi - m.lo, m.plane_stride, m.row_stride)
            if self.signal:
                if not m.sig_handle:
                    raise InvalidArgumentError("a neighbour published no signal words")
                sp = dev.ipc_open(m.sig_handle, m.sig_offset, local_src.device.index)
                self._opened.append((sp, m.sig_offset))
                sigs[side] = sp
        self.above, self.below = rows["above"], rows["below"]
        self._sig_above, self._sig_below = sigs["above"], sigs["below"]
        self._lib = _lib.load()
        self._check = _lib.check
        w = dev._taps(taps)
        self._w = w
        a = self.above or dev.PeerRows(0, 0, 0, 0, 0)
        b = self.below or dev.PeerRows(0, 0, 0, 0, 0)
        self._stream = torch.cuda.current_stream(local_src.device).cuda_stream
        self._args = (local_src.data_ptr(), local_dst.data_ptr(), n, band.rows, C, sps, dps, srs, drs, band.lo, Rs,
                      a.ptr or None, a.row0, a.rows, a.plane_stride, a.row_stride,
                      b.ptr or None, b.row0, b.rows, b.plane_stride, b.row_stride,
                      band.lo, band.lo, band.hi, w.ctypes.data, w.size, _lib.SC_EXTENDED if extended else 0)
        self._sig_args = (self.sig.data_ptr(), self._sig_above, self._sig_below)

    def sync(self):
        """Process-group barrier (all ranks' prior band writes complete)."""
        import torch.distributed as dist

        torch.cuda.current_stream(self.src.device).synchronize()
        if self.band.world > 1:
            dist.barrier(group=self.group)

    def step(self):
        if self.signal:
            self.epoch += 1
            self._check(self._lib.sc_two_pass_band_peer_sig_f32(*self._args, *self._sig_args, self.epoch,
                                                                self.err.data_ptr(), self._stream))
        else:
            self._check(self._lib.sc_two_pass_band_peer_f32(*self._args, self._stream))

    kernel_only = step  # the step IS the dominant kernel

    def wait_consumed(self):
        """Stream-ordered: the neighbours have finished the current epoch (they no
        longer read this band's rows), so the caller may overwrite them."""
        if self.signal and self.epoch:
            self._check(self._lib.sc_band_signal_wait(self._sig_above, self._sig_below, 1, self.epoch,
                                                      self.err.data_ptr(), self._stream))

    def check(self):
        """Raise if a neighbour wait timed out (the step's output is then invalid)."""
        from .errors import ExecutionError

        if int(self.err.item()) != 0:
            raise ExecutionError([(self.band.rank, RuntimeError("row-band neighbour signal wait timed out"))])

    def close(self):
        """Unmap the neighbours' buffers after EVERY rank has finished reading
        (a barrier first: exporters outlive importers)."""
        from . import device as dev

        torch.cuda.current_stream(self.src.device).synchronize()
        if self.band.world > 1:
            import torch.distributed as dist

            if dist.is_initialized():
                dist.barrier(group=self.group)
        for ptr, off in self._opened:
            dev.ipc_close(ptr, off)
        self._opened = []


def peer_transport_works(group=None, device=None) -> bool:
    """One-time probe run by every rank before choosing the peer transport: a tiny
    banded image is convolved twice, with the halo read in-kernel from the
    neighbours' IPC-mapped buffers and with a send/recv halo exchange
    (BandStepper); True only if every rank got identical bits from both and no
    step failed. Every rank takes part in every collective whatever happens
    locally, so a failure anywhere cannot hang the others."""
    import torch.distributed as dist

    from . import device as dev

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return True
    rank = dist.get_rank(group)
    dev_t = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    R, C, P = 8 * world, 256, 2
    w = (torch.tensor([1, 4, 6, 4, 1], dtype=torch.float32) / 16).numpy()
    band = band_plan(R, rank, world, 2)
    full = dev.synthetic((P, R, C), 97, 1, device=dev_t)
    own = full[:, band.lo:band.hi].clone()
    out_peer = torch.full((P, band.hi - band.lo, C), float("nan"), device=dev_t)
    held = torch.full((P, band.local_rows, C), float("nan"), device=dev_t)
    held[:, band.owned] = own
    out_ref = torch.full_like(out_peer, float("nan"))
    n, Rs, _, sps, srs = dev._planes(own, "own")

    ok = True
    try:
        handle, offset = dev.ipc_export(own)
    except Exception:  # noqa: BLE001 -- any failure means: do not use the peer path
        ok, handle, offset = False, b"\0" * 64, 0
    torch.cuda.synchronize(dev_t)
    metas = publish_peer_meta(PeerMeta(rank, band.lo, band.hi, handle, offset, sps, srs, C, n), band, group)
    everyone = [None] * world
    dist.all_gather_object(everyone, ok, group=group)
    opened = []
    if all(everyone):
        try:
            above, below = peer_neighbours(metas, band)
            rows = []
            for m in (above, below):
                if m is None:
                    rows.append(None)
                    continue
                ptr = dev.ipc_open(m.handle, m.offset, dev_t.index)
                opened.append((ptr, m.offset))
                rows.append(dev.PeerRows(ptr, m.lo, m.hi - m.lo, m.plane_stride, m.row_stride))
            dev.two_pass_band_peer(own, w, out_peer, global_rows=R, src_row0=band.lo, dst_row0=band.lo,
                                   out_lo=band.lo, out_hi=band.hi, above=rows[0], below=rows[1])
            torch.cuda.synchronize(dev_t)
        except Exception:  # noqa: BLE001
            ok = False
    else:
        ok = False
    try:
        BandStepper(held, out_ref, band, w, group=group).step()  # collective P2P: every rank runs it
        torch.cuda.synchronize(dev_t)
    except Exception:  # noqa: BLE001
        ok = False
    ok = ok and bool(torch.equal(out_peer, out_ref))
    flag = torch.tensor([1 if ok else 0], device=dev_t if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    dist.barrier(group=group)  # nobody unmaps / frees while a neighbour may still read
    for ptr, off in opened:
        try:
            dev.ipc_close(ptr, off)
        except Exception:  # noqa: BLE001
            pass
    return bool(flag.item() == 1)
