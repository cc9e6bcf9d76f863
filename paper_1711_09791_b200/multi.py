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


def exchange_halos(local, band: Band, group=None):
    """Fill the halo rows of `local` ((P, band.local_rows, C), held rows) from the
    neighbours' owned rows with one batched send/recv group. Returns the list of
    async works (wait on them before reading the halo rows)."""
    import torch.distributed as dist

    if band.world == 1:
        return []
    r = band.radius
    ops = []
    P = local.shape[0]
    top = band.lo - band.in_lo      # halo rows above (0 for rank 0)
    bot = band.in_hi - band.hi      # halo rows below (0 for the last rank)
    o0 = band.owned.start
    o1 = band.owned.stop
    if band.rank > 0 and top > 0:
        peer = band.rank - 1
        for p in range(P):
            ops.append(dist.P2POp(dist.isend, local[p, o0 : o0 + top], peer, group=group))
            ops.append(dist.P2POp(dist.irecv, local[p, 0:top], peer, group=group))
    if band.rank < band.world - 1 and bot > 0:
        peer = band.rank + 1
        for p in range(P):
            ops.append(dist.P2POp(dist.isend, local[p, o1 - bot : o1], peer, group=group))
            ops.append(dist.P2POp(dist.irecv, local[p, o1 : o1 + bot], peer, group=group))
    assert r >= 0
    if not ops:
        return []
    return dist.batch_isend_irecv(ops)


BandFn = Callable[..., object]


def _default_band_fn(src, dst, *, global_rows, src_row0, dst_row0, out_lo, out_hi, taps, extended):
    from . import device

    return device.two_pass_band(src, taps, dst, global_rows=global_rows, src_row0=src_row0, dst_row0=dst_row0,
                                out_lo=out_lo, out_hi=out_hi, extended=extended)


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
    if i_lo > band.lo:
        fn(local_src, local_dst, out_lo=band.lo, out_hi=i_lo, **common)
    if i_hi < band.hi:
        fn(local_src, local_dst, out_lo=i_hi, out_hi=band.hi, **common)
