"""Drop-in whole-plane operations with the reference's names, signatures and
error behaviour (S/conv.py:29-476), executed by libsepconv_b200.so.

Planes may hold host numpy arrays (staged through HBM; the call blocks, like
the reference) or CUDA tensors (launched on the current stream, no host copy).
Results are bit-identical to the reference on the same inputs: every op is a
float32 multiply or add in the reference's order, never fused into an FMA.

`vectorized` is accepted for signature compatibility and ignored: the
reference's two backends produce identical bits and so does the GPU.
`counter` receives the exact operation counts of the launched work (the GPU
kernels execute precisely the reference's multiplies and adds).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import InvalidArgumentError, InvalidDimensionError, UnsupportedWidthError
from .image import Plane, ValidRegion, valid_region
from .kernels import DenseKernel, SeparableKernel


class Algorithm(str, Enum):
    SINGLE_PASS_GENERIC = "single-generic"
    SINGLE_PASS_UNROLLED5 = "single-unrolled"
    TWO_PASS = "two-pass"


@dataclass(frozen=True)
class ConvVariant:
    """Algorithm plus copy-back; copy_back is normalised to False for two-pass (S/conv.py:35-49)."""

    algorithm: Algorithm
    copy_back: bool = False

    def __post_init__(self):
        if self.algorithm is Algorithm.TWO_PASS and self.copy_back:
            object.__setattr__(self, "copy_back", False)


@dataclass
class OpCounter:
    """Tally of float multiply and add events (S/conv.py:52-57)."""

    multiplications: int = 0
    additions: int = 0


@dataclass(frozen=True)
class ArithCount:
    multiplications: int
    additions: int


# ---------------------------------------------------------------------------
# buffers: host numpy <-> device tensors

def _torch():
    import torch

    return torch


def _is_dev(p: Plane) -> bool:
    # duck-typed: the reference's Plane (numpy data) works too
    return bool(getattr(p.data, "is_cuda", False))


def _shares(a: Plane, b: Plane) -> bool:
    if _is_dev(a) != _is_dev(b):
        return False
    if not _is_dev(a):
        return bool(np.shares_memory(a.data, b.data))
    ta, tb = a.data, b.data
    if ta.device != tb.device:
        return False
    na = ((ta.shape[0] - 1) * ta.stride(0) + ta.shape[1]) * 4
    nb = ((tb.shape[0] - 1) * tb.stride(0) + tb.shape[1]) * 4
    pa, pb = ta.data_ptr(), tb.data_ptr()
    return pa < pb + nb and pb < pa + na


def _check_pair(src: Plane, dst: Plane, width: int) -> None:
    """S/conv.py:68-79: shapes, aliasing, minimum size."""
    if src.rows != dst.rows or src.cols != dst.cols:
        raise InvalidArgumentError(
            f"source and destination dimensions differ: ({src.rows}, {src.cols}) vs ({dst.rows}, {dst.cols})"
        )
    if _shares(src, dst):
        raise InvalidArgumentError("source and destination must be distinct buffers")
    if src.rows < width or src.cols < width:
        raise InvalidDimensionError(f"plane {src.rows}x{src.cols} smaller than kernel width {width}")
    if _is_dev(src) != _is_dev(dst) or (_is_dev(src) and src.data.device != dst.data.device):
        raise InvalidArgumentError("planes must both be host arrays or both live on the same CUDA device")


class _Staged:
    """Device views of a group of planes; host planes are uploaded and, on exit,
    the named regions are written back (only those the reference writes)."""

    def __init__(self, planes, write_only=()):
        """write_only: indices of planes whose device copy is only written (and
        partly written back): allocated on the device, not uploaded."""
        torch = _torch()
        self.planes = planes
        self.host = not _is_dev(planes[0])
        if self.host:
            dev = torch.device("cuda", torch.cuda.current_device())
            self.t = [(torch.empty(p.data.shape, dtype=torch.float32, device=dev) if i in write_only
                       else torch.from_numpy(p.data).to(dev, non_blocking=False)).unsqueeze(0)
                      for i, p in enumerate(planes)]
        else:
            self.t = [p.data.unsqueeze(0) for p in planes]

    def write_back(self, idx: int, rows: tuple[int, int] | None = None, cols: tuple[int, int] | None = None):
        if not self.host:
            return
        torch = _torch()
        t = self.t[idx][0]
        a = self.planes[idx].data
        r0, r1 = rows if rows else (0, a.shape[0])
        c0, c1 = cols if cols else (0, a.shape[1])
        if r1 <= r0 or c1 <= c0:
            return
        torch.from_numpy(a)[r0:r1, c0:c1].copy_(t[r0:r1, c0:c1])

    def finish(self):
        """Host planes: wait for the write-backs (the reference's calls block);
        device planes stay stream-ordered like any CUDA op."""
        if self.host:
            _torch().cuda.current_stream().synchronize()


def _streamable(*planes: Plane) -> bool:
    """Host planes the streamed entry points take as they are (the reference's Plane
    keeps a C-contiguous 2-D float32 numpy array, S/image.py:37-39)."""
    for p in planes:
        a = p.data
        if not isinstance(a, np.ndarray) or a.dtype != np.float32 or a.ndim != 2 or not a.flags.c_contiguous:
            return False
    return True


def _count(counter: OpCounter | None, mults: int, adds: int) -> None:
    if counter is not None:
        counter.multiplications += mults
        counter.additions += adds


# ---------------------------------------------------------------------------
# public ops (S/conv.py:324-440)

def conv_single_pass_generic(src: Plane, kernel: DenseKernel, dst: Plane, *, vectorized: bool = True,
                             counter: OpCounter | None = None) -> None:
    """Direct convolution of src's valid region into dst; dst elsewhere untouched (S/conv.py:324-338)."""
    from . import device

    _check_pair(src, dst, kernel.width)
    region = valid_region(src.rows, src.cols, kernel.radius)
    if _streamable(src, dst):
        # host planes: chunked H2D / kernel / D2H of the valid region (sc_single_pass_host_f32)
        device.single_pass_host([src.data], [dst.data], kernel.matrix)
    else:
        st = _Staged([src, dst])
        device.single_pass(st.t[0], kernel.matrix, st.t[1])
        st.write_back(1, (region.row_lo, region.row_hi), (region.col_lo, region.col_hi))
        st.finish()
    n = (region.row_hi - region.row_lo) * (region.col_hi - region.col_lo)
    _count(counter, kernel.width**2 * n, (kernel.width**2 - 1) * n)


def conv_single_pass_unrolled5(src: Plane, kernel: DenseKernel, dst: Plane, *, vectorized: bool = True,
                               counter: OpCounter | None = None) -> None:
    """The width-5 single pass; bitwise equal to the generic one (S/conv.py:341-359)."""
    if kernel.width != 5:
        raise UnsupportedWidthError(f"unrolled variant needs width 5, got {kernel.width}")
    conv_single_pass_generic(src, kernel, dst, vectorized=vectorized, counter=counter)


def _one_pass(which: str, src: Plane, kernel: SeparableKernel, dst: Plane, counter) -> None:
    from . import device

    _check_pair(src, dst, kernel.width)
    region = valid_region(src.rows, src.cols, kernel.radius)
    if _streamable(src, dst):
        device.pass_host([src.data], [dst.data], kernel.weights, vertical=(which == "v"))
    else:
        st = _Staged([src, dst], write_only=(1,))
        fn = device.hpass if which == "h" else device.vpass
        fn(st.t[0], kernel.weights, st.t[1], region.row_lo, region.row_hi)
        st.write_back(1, (region.row_lo, region.row_hi), (region.col_lo, region.col_hi))
        st.finish()
    n = (region.row_hi - region.row_lo) * (region.col_hi - region.col_lo)
    _count(counter, kernel.width * n, (kernel.width - 1) * n)


def horizontal_pass(src: Plane, kernel: SeparableKernel, dst: Plane, *, vectorized: bool = True,
                    counter: OpCounter | None = None) -> None:
    """1-D convolution along each valid row into dst; dst elsewhere untouched (S/conv.py:362-375)."""
    _one_pass("h", src, kernel, dst, counter)


def vertical_pass(src: Plane, kernel: SeparableKernel, dst: Plane, *, vectorized: bool = True,
                  counter: OpCounter | None = None) -> None:
    """1-D convolution along each valid column into dst; dst elsewhere untouched (S/conv.py:378-389)."""
    _one_pass("v", src, kernel, dst, counter)


def conv_two_pass(plane: Plane, kernel: SeparableKernel, scratch: Plane, *, vectorized: bool = True,
                  counter: OpCounter | None = None, extended: bool = False) -> None:
    """Row pass into scratch, column pass back into `plane` (S/conv.py:392-421).

    End state is the reference's bit for bit, scratch included: scratch holds
    H0 (zero outside the row-pass region) and plane's valid region holds V(H0).
    Runs as the split K2+K3 pair because the reference's scratch is observable.
    """
    from . import device

    _check_pair(plane, scratch, kernel.width)
    r = kernel.radius
    if _streamable(plane, scratch):
        # host planes: streamed, both buffers' end state (sc_two_pass_host_split_f32)
        device.two_pass_host_split([plane.data], [scratch.data], kernel.weights, extended=extended)
    else:
        st = _Staged([plane, scratch])
        device.two_pass_split(st.t[0], st.t[1], kernel.weights, extended=extended)
        st.write_back(0, (r, plane.rows - r), (r, plane.cols - r))
        st.write_back(1)
        st.finish()
    span = plane.cols - 2 * r
    h_rows = plane.rows if extended else plane.rows - 2 * r
    v_rows = plane.rows - 2 * r
    w = kernel.width
    _count(counter, w * span * (h_rows + v_rows), (w - 1) * span * (h_rows + v_rows))


def copy_back(src: Plane, dst: Plane, region: ValidRegion) -> None:
    """dst[region] := src[region]; dst elsewhere untouched (S/conv.py:424-440)."""
    from . import device

    if src.rows != dst.rows or src.cols != dst.cols:
        raise InvalidArgumentError(
            f"source and destination dimensions differ: ({src.rows}, {src.cols}) vs ({dst.rows}, {dst.cols})"
        )
    if _shares(src, dst):
        raise InvalidArgumentError("source and destination must be distinct buffers")
    if not (0 <= region.row_lo <= region.row_hi <= src.rows and 0 <= region.col_lo <= region.col_hi <= src.cols):
        raise InvalidArgumentError(f"region {region} out of bounds for {src.rows}x{src.cols}")
    if _is_dev(src) != _is_dev(dst):
        raise InvalidArgumentError("planes must both be host arrays or both live on the same CUDA device")
    st = _Staged([src, dst], write_only=(1,))
    device.copy_region(st.t[0], st.t[1], region.row_lo, region.row_hi, region.col_lo, region.col_hi)
    st.write_back(1, (region.row_lo, region.row_hi), (region.col_lo, region.col_hi))
    st.finish()


def doubly_interior_region(rows: int, cols: int, radius: int) -> ValidRegion:
    """Rows whose vertical window reads only rows the row pass wrote (S/conv.py:452-459)."""
    region = ValidRegion(2 * radius, rows - 2 * radius, radius, cols - radius)
    if region.row_lo >= region.row_hi or region.col_lo >= region.col_hi:
        raise InvalidDimensionError(f"image {rows}x{cols} has no doubly-interior region for radius {radius}")
    return region


def arith_count(variant: ConvVariant, rows: int, cols: int, width: int) -> ArithCount:
    """Closed-form per-plane multiply/add counts (S/conv.py:462-476)."""
    if rows < width or cols < width:
        raise InvalidDimensionError(f"plane {rows}x{cols} smaller than kernel width {width}")
    r = width // 2
    valid = (rows - 2 * r) * (cols - 2 * r)
    if variant.algorithm is Algorithm.TWO_PASS:
        return ArithCount(multiplications=2 * width * valid, additions=2 * (width - 1) * valid)
    terms = width * width
    return ArithCount(multiplications=terms * valid, additions=(terms - 1) * valid)

