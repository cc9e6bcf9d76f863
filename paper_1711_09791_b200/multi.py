"""Multi-GPU partitioner.

Row bands: rank g owns output rows partition_block(0, R, g, n) of every plane
and holds input rows [lo - r, hi + r) clipped to the image; the 2r halo rows are
exchanged with the neighbours by NCCL send/recv. Frame batches: frames are
sharded with the same rule and need no communication.
"""

from __future__ import annotations

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
