"""Device API: the hot path on torch CUDA tensors (PyTorch is plumbing here --
device memory and streams; every sample is computed by libsepconv_b200.so).

Tensors are float32 stacks of planes, shape (P, R, C) or (N, P, R, C) (any
leading dims that collapse to a uniform plane stride), unit column stride.
Launches go on the current torch stream of the tensor's device and are
asynchronous, like any CUDA op.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import InvalidArgumentError


def _taps(taps) -> np.ndarray:
    w = getattr(taps, "weights", taps)  # SeparableKernel or array-like
    if type(w) is np.ndarray and w.dtype == np.float32 and w.ndim == 1 and w.flags.c_contiguous:
        return w
    if isinstance(w, torch.Tensor):
        w = w.detach().cpu().numpy()
    w = np.ascontiguousarray(w, dtype=np.float32).reshape(-1)
    return w


def _dense(dense) -> np.ndarray:
    m = getattr(dense, "matrix", dense)
    if isinstance(m, torch.Tensor):
        m = m.detach().cpu().numpy()
    m = np.ascontiguousarray(m, dtype=np.float32)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise InvalidArgumentError(f"dense kernel must be square, got shape {m.shape}")
    return m


def _fp(a: np.ndarray) -> int:
    """Address of a float32 host array (the caller keeps `a` alive across the call)."""
    return a.ctypes.data


def _planes(t: torch.Tensor, what: str):
    """(nplanes, R, C, plane_stride, row_stride) of a CUDA float32 plane stack."""
    if type(t) is torch.Tensor and t.is_cuda and t.dtype == torch.float32 and t.dim() >= 2 and t.is_contiguous():
        R, C = t.shape[-2], t.shape[-1]  # fast path: dense stack
        return t.numel() // (R * C) if R * C else 0, R, C, R * C, C
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgumentError(f"{what} must be a CUDA tensor")
    if t.dtype != torch.float32:
        raise InvalidArgumentError(f"{what} must be float32, got {t.dtype}")
    if t.dim() < 2:
        raise InvalidArgumentError(f"{what} must have at least 2 dims (rows, cols)")
    R, C = t.shape[-2], t.shape[-1]
    if t.stride(-1) != 1 and C > 1:
        raise InvalidArgumentError(f"{what} needs unit column stride")
    try:
        v = t.view(-1, R, C)
    except RuntimeError as exc:
        raise InvalidArgumentError(f"{what}: leading dims do not collapse to one plane stride") from exc
    ps = v.stride(0) if v.shape[0] > 1 else R * max(v.stride(1), C)
    return v.shape[0], R, C, ps, v.stride(1)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(t: torch.Tensor) -> int:
    """cudaStream_t of torch's current stream on t's device."""
    if _raw_stream is not None:
        return _raw_stream(t.device.index)
    return torch.cuda.current_stream(t.device).cuda_stream


def _same_geometry(a: torch.Tensor, b: torch.Tensor):
    if a.shape != b.shape:
        raise InvalidArgumentError(
            f"source and destination dimensions differ: {tuple(a.shape)} vs {tuple(b.shape)}"
        )
    if a.device != b.device:
        raise InvalidArgumentError("source and destination live on different devices")


def two_pass(src: torch.Tensor, taps, out: torch.Tensor | None = None, *, extended: bool = False,
             ring: bool = True) -> torch.Tensor:
    """Fused single-read/single-write two-pass, out of place (K1).

    Returns the image the reference leaves in `image` after conv_two_pass
    (S/conv.py:392-421): ring = src, valid region = V(H0). ring=False leaves
    out's ring untouched.
    """
    w = _taps(taps)
    if out is None:
        out = torch.empty_like(src)
    _same_geometry(src, out)
    n, R, C, sps, srs = _planes(src, "src")
    _, _, _, dps, drs = _planes(out, "out")
    flags = (_lib.SC_EXTENDED if extended else 0) | (0 if ring else _lib.SC_NO_RING)
    L = _lib.load()
    _lib.check(L.sc_two_pass_fused_f32(src.data_ptr(), out.data_ptr(), n, R, C, sps, dps, srs, drs,
                                       _fp(w), w.size, flags, _stream(src)))
    return out


def two_pass_band(src: torch.Tensor, taps, out: torch.Tensor, *, global_rows: int, src_row0: int,
                  dst_row0: int, out_lo: int, out_hi: int, extended: bool = False, out_lo2: int = 0,
                  out_hi2: int = 0) -> torch.Tensor:
    """Row band of the fused two-pass (multi-GPU partitioner): src holds global rows
    [src_row0, src_row0 + src.shape[-2]), out row 0 is global row dst_row0. An
    optional second segment [out_lo2, out_hi2) runs in the same launch."""
    w = _taps(taps)
    n, Rs, C, sps, srs = _planes(src, "src")
    n2, Rd, C2, dps, drs = _planes(out, "out")
    if n2 != n or C2 != C:
        raise InvalidArgumentError("band source and destination plane counts / widths differ")
    if max(out_hi, out_hi2) - dst_row0 > Rd:
        raise InvalidArgumentError("destination band too short for the output rows")
    flags = _lib.SC_EXTENDED if extended else 0
    L = _lib.load()
    _lib.check(L.sc_two_pass_band2_f32(src.data_ptr(), out.data_ptr(), n, global_rows, C, sps, dps, srs, drs,
                                       src_row0, Rs, dst_row0, out_lo, out_hi, out_lo2, out_hi2, _fp(w), w.size,
                                       flags, _stream(src)))
    return out


class PeerRows:
    """Rows [row0, row0 + rows) of every plane of a neighbouring band, at a device
    address valid in this process (a local tensor, or another process's buffer
    mapped with ipc_open). Strides in floats."""

    __slots__ = ("ptr", "row0", "rows", "plane_stride", "row_stride", "keep")

    def __init__(self, ptr: int, row0: int, rows: int, plane_stride: int, row_stride: int, keep=None):
        self.ptr, self.row0, self.rows = int(ptr), int(row0), int(rows)
        self.plane_stride, self.row_stride = int(plane_stride), int(row_stride)
        self.keep = keep  # object owning the memory (kept alive)

    @classmethod
    def of(cls, t: torch.Tensor, row0: int) -> "PeerRows":
        _, R, _, ps, rs = _planes(t, "neighbour band")
        return cls(t.data_ptr(), row0, R, ps, rs, keep=t)


def two_pass_band_peer(src: torch.Tensor, taps, out: torch.Tensor, *, global_rows: int, src_row0: int,
                       dst_row0: int, out_lo: int, out_hi: int, above: PeerRows | None = None,
                       below: PeerRows | None = None, extended: bool = False) -> torch.Tensor:
    """Row band whose halo rows come straight from the neighbouring bands' memory
    (no exchange step): src holds global rows [src_row0, src_row0 + src.shape[-2])."""
    w = _taps(taps)
    n, Rs, C, sps, srs = _planes(src, "src")
    n2, Rd, C2, dps, drs = _planes(out, "out")
    if n2 != n or C2 != C:
        raise InvalidArgumentError("band source and destination plane counts / widths differ")
    if out_hi - dst_row0 > Rd:
        raise InvalidArgumentError("destination band too short for the output rows")
    a = above or PeerRows(0, 0, 0, 0, 0)
    b = below or PeerRows(0, 0, 0, 0, 0)
    L = _lib.load()
    _lib.check(L.sc_two_pass_band_peer_f32(
        src.data_ptr(), out.data_ptr(), n, global_rows, C, sps, dps, srs, drs, src_row0, Rs,
        a.ptr or None, a.row0, a.rows, a.plane_stride, a.row_stride,
        b.ptr or None, b.row0, b.rows, b.plane_stride, b.row_stride,
        dst_row0, out_lo, out_hi, _fp(w), w.size, _lib.SC_EXTENDED if extended else 0, _stream(src)))
    return out


def ipc_export(t: torch.Tensor) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of t's allocation, byte offset of t in it)."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise InvalidArgumentError("ipc_export needs a CUDA tensor")
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    L = _lib.load()
    _lib.check(L.sc_ipc_export(t.data_ptr(), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_open(handle: bytes, offset: int, device: int | None = None) -> int:
    """Map another process's exported buffer for `device` (default: torch's current
    device); returns its address in this process."""
    if len(handle) != 64:
        raise InvalidArgumentError("an IPC handle is 64 bytes")
    if device is None:
        device = torch.cuda.current_device()
    ptr = ctypes.c_void_p(0)
    L = _lib.load()
    _lib.check(L.sc_ipc_open(handle, int(offset), int(device), ctypes.byref(ptr)))
    return int(ptr.value)


def ipc_close(ptr: int, offset: int) -> None:
    L = _lib.load()
    _lib.check(L.sc_ipc_close(ptr, int(offset)))


def hpass(src: torch.Tensor, taps, out: torch.Tensor, row_lo: int | None = None, row_hi: int | None = None,
          *, zero_fill: bool = False) -> torch.Tensor:
    """horizontal_rows_vec (S/conv.py:215-240) over rows [row_lo, row_hi) (default: valid rows)."""
    w = _taps(taps)
    _same_geometry(src, out)
    n, R, C, sps, srs = _planes(src, "src")
    _, _, _, dps, drs = _planes(out, "out")
    r = w.size // 2
    lo = r if row_lo is None else row_lo
    hi = R - r if row_hi is None else row_hi
    L = _lib.load()
    _lib.check(L.sc_hpass_f32(src.data_ptr(), out.data_ptr(), n, R, C, sps, dps, srs, drs, lo, hi, _fp(w),
                              w.size, _lib.SC_ZERO_FILL if zero_fill else 0, _stream(src)))
    return out


def vpass(src: torch.Tensor, taps, out: torch.Tensor, row_lo: int | None = None,
          row_hi: int | None = None) -> torch.Tensor:
    """vertical_rows_vec (S/conv.py:269-293) over rows [row_lo, row_hi) inside [r, R-r)."""
    w = _taps(taps)
    _same_geometry(src, out)
    n, R, C, sps, srs = _planes(src, "src")
    _, _, _, dps, drs = _planes(out, "out")
    r = w.size // 2
    lo = r if row_lo is None else row_lo
    hi = R - r if row_hi is None else row_hi
    L = _lib.load()
    _lib.check(L.sc_vpass_f32(src.data_ptr(), out.data_ptr(), n, R, C, sps, dps, srs, drs, lo, hi, _fp(w),
                              w.size, 0, _stream(src)))
    return out


def two_pass_split(image: torch.Tensor, scratch: torch.Tensor, taps, *, extended: bool = False) -> torch.Tensor:
    """The reference two-pass with its buffer semantics (K2 + K3): scratch := H0,
    image[valid] := V(scratch); image ring untouched. Returns image."""
    w = _taps(taps)
    _same_geometry(image, scratch)
    n, R, C, ips, irs = _planes(image, "image")
    _, _, _, sps, srs = _planes(scratch, "scratch")
    L = _lib.load()
    _lib.check(L.sc_two_pass_split_f32(image.data_ptr(), scratch.data_ptr(), n, R, C, ips, sps, irs, srs,
                                       _fp(w), w.size, _lib.SC_EXTENDED if extended else 0, _stream(image)))
    return image


def two_pass_inplace(image: torch.Tensor, taps, *, extended: bool = False) -> torch.Tensor:
    """The two-pass in place with no observable scratch (convolve_image without a
    workspace): image[valid] := V(H0), ring untouched. One pass over the image
    (plus a small halo snapshot) on 16-B aligned rows. Returns image."""
    w = _taps(taps)
    n, R, C, ps, rs = _planes(image, "image")
    L = _lib.load()
    _lib.check(L.sc_two_pass_inplace_f32(image.data_ptr(), n, R, C, ps, rs, _fp(w), w.size,
                                         _lib.SC_EXTENDED if extended else 0, _stream(image)))
    return image


def single_pass(src: torch.Tensor, dense, out: torch.Tensor, *, copy_back: bool = False) -> torch.Tensor:
    """single_pass_rows_vec (S/conv.py:86-114) with the dense matrix; out's ring untouched.
    copy_back additionally writes the valid region into src (S/executors.py:330-331)."""
    m = _dense(dense)
    _same_geometry(src, out)
    n, R, C, sps, srs = _planes(src, "src")
    _, _, _, dps, drs = _planes(out, "out")
    L = _lib.load()
    _lib.check(L.sc_single_pass_f32(src.data_ptr(), out.data_ptr(), n, R, C, sps, dps, srs, drs, _fp(m),
                                    m.shape[0], _lib.SC_COPY_BACK if copy_back else 0, _stream(src)))
    return out


def copy_region(src: torch.Tensor, dst: torch.Tensor, row_lo: int, row_hi: int, col_lo: int,
                col_hi: int) -> torch.Tensor:
    """copy_back (S/conv.py:424-440) on device planes."""
    _same_geometry(src, dst)
    n, R, C, sps, srs = _planes(src, "src")
    _, _, _, dps, drs = _planes(dst, "dst")
    L = _lib.load()
    _lib.check(L.sc_copy_region_f32(src.data_ptr(), dst.data_ptr(), n, R, C, sps, dps, srs, drs, row_lo, row_hi,
                                    col_lo, col_hi, _stream(src)))
    return dst


def fill_synthetic(t: torch.Tensor, seed: int, kind: int, offset: int = 0) -> torch.Tensor:
    """Fill a contiguous CUDA float32 tensor with splitmix64 draws offset.. (S/image.py:131-162)."""
    if not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous():
        raise InvalidArgumentError("fill_synthetic needs a contiguous CUDA float32 tensor")
    L = _lib.load()
    _lib.check(L.sc_fill_synthetic_f32(t.data_ptr(), t.numel(), seed & (2**64 - 1), offset, kind, _stream(t)))
    return t


def synthetic(shape, seed: int, kind: int, device="cuda", offset: int = 0) -> torch.Tensor:
    t = torch.empty(tuple(shape), dtype=torch.float32, device=device)
    return fill_synthetic(t, seed, kind, offset)


class HostRegistry:
    """Page-locked registration of callers' numpy buffers, cached for the buffer's
    lifetime, so repeated end-to-end calls on the same pageable image (a reps
    loop, a video buffer reused frame after frame) DMA straight from and into it
    instead of going through the library's pinned staging ring, whose two host
    copies make the pageable path host-memory-bound.

    * registers the ROOT buffer that owns the data (views of one (P, R, C) array
      share pages; one registration covers all of them) when it holds at least
      `min_bytes` (SC_HOST_REGISTER_MIN_MB, default 64) and owns its memory;
      a smaller buffer of at least `reuse_min_bytes` (SC_HOST_REGISTER_REUSE_MIN_MB,
      default 1) is registered when it is seen a SECOND time (a reps loop, a
      reused frame buffer): one-shot callers never pay the page-locking, repeated
      calls on a 3 x 1152^2 image go from 1.98 ms (staging ring) to the DMA path;
    * releases it when the buffer is garbage-collected (weakref.finalize runs
      before numpy frees the data) or when the total registered exceeds
      `max_bytes` (SC_HOST_REGISTER_MAX_GB, default half of physical memory;
      least recently used first);
    * any failure (e.g. pages already registered elsewhere) leaves the buffer
      unregistered: the staging ring handles it with the same bits.
    The first call on a buffer pays the page-locking (measured ~0.1 s per GB on
    the B200 box, profiles/r02_host_mem_probe.txt); later calls do not."""

    def __init__(self):
        import os
        from collections import OrderedDict

        import threading

        self._regs = OrderedDict()  # root address -> (nbytes, finalizer)
        self._lock = threading.RLock()  # finalizers may run on any thread (garbage collection)
        self.min_bytes = int(float(os.environ.get("SC_HOST_REGISTER_MIN_MB", "64")) * (1 << 20))
        self.reuse_min_bytes = int(float(os.environ.get("SC_HOST_REGISTER_REUSE_MIN_MB", "1")) * (1 << 20))
        self._seen = {}  # root address -> (finalizer, call): smaller buffers seen in one call so far
        self._call = 0   # the entry points count their calls (new_call): all planes of one call are ONE sighting
        try:
            phys = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        except (ValueError, OSError):
            phys = 64 << 30
        self.max_bytes = int(float(os.environ.get("SC_HOST_REGISTER_MAX_GB", str(phys / 2 / 2**30))) * 2**30)
        self.total = 0

    @staticmethod
    def _root(arr):
        root = arr
        while isinstance(root.base, np.ndarray):
            root = root.base
        return root

    def pin(self, arr) -> bool:
        if not isinstance(arr, np.ndarray):
            return False
        root = self._root(arr)
        if not root.flags.owndata or root.base is not None or root.nbytes < min(self.min_bytes, self.reuse_min_bytes):
            return False
        with self._lock:
            key = root.ctypes.data
            if root.nbytes < self.min_bytes and key not in self._regs:
                if key not in self._seen:  # first sighting: remember it, stage this call
                    import weakref

                    if len(self._seen) > 4096:
                        for fin, _ in self._seen.values():
                            fin.detach()
                        self._seen.clear()
                    self._seen[key] = (weakref.finalize(root, self._forget, key), self._call)
                    return False
                if self._seen[key][1] == self._call:  # another plane of the same call
                    return False
                self._seen.pop(key)[0].detach()
            return self._pin_locked(root)

    def new_call(self):
        """One end-to-end call begins: its planes' sightings count once."""
        with self._lock:
            self._call += 1

    def _forget(self, key):
        with self._lock:
            self._seen.pop(key, None)

    def _pin_locked(self, root) -> bool:
        key = root.ctypes.data
        if key in self._regs:
            self._regs.move_to_end(key)
            return True
        while self._regs and self.total + root.nbytes > self.max_bytes:
            old_key, (old_n, fin) = self._regs.popitem(last=False)
            fin.detach()
            self._release(old_key, old_n)
        if self.total + root.nbytes > self.max_bytes:
            return False
        L = _lib.load()
        if L.sc_host_register(key, root.nbytes) != _lib.SC_OK:
            return False
        import weakref

        fin = weakref.finalize(root, self._on_free, key)
        self._regs[key] = (root.nbytes, fin)
        self.total += root.nbytes
        return True

    def _release(self, key, nbytes):
        self.total -= nbytes
        _lib.load().sc_host_unregister(key)

    def _on_free(self, key):
        with self._lock:
            item = self._regs.pop(key, None)
            if item is not None:
                self._release(key, item[0])

    def registered(self, arr) -> bool:
        with self._lock:
            return isinstance(arr, np.ndarray) and self._root(arr).ctypes.data in self._regs

    def clear(self):
        with self._lock:
            for key, (n, fin) in list(self._regs.items()):
                fin.detach()
                self._release(key, n)
            self._regs.clear()
            for fin, _ in self._seen.values():
                fin.detach()
            self._seen.clear()


host_registry = HostRegistry()


def _host_ptrs(planes, shape=None):
    """Addresses of C-contiguous float32 host planes (numpy arrays or CPU tensors,
    pinned or pageable) sharing one 2-D shape."""
    ptrs = []
    for arr in planes:
        if isinstance(arr, torch.Tensor):
            if arr.is_cuda or arr.dtype != torch.float32 or not arr.is_contiguous():
                raise InvalidArgumentError("host planes must be contiguous CPU float32")
            shp = tuple(arr.shape)
            ptrs.append(arr.data_ptr())
        else:
            if not isinstance(arr, np.ndarray) or arr.dtype != np.float32 or not arr.flags.c_contiguous:
                raise InvalidArgumentError("host planes must be C-contiguous float32")
            if not arr.flags.writeable:
                raise InvalidArgumentError("host planes must be writeable")
            shp = arr.shape
            ptrs.append(arr.ctypes.data)
        if len(shp) != 2 or (shape is not None and tuple(shp) != tuple(shape)):
            raise InvalidArgumentError("host planes must be 2-D and share one shape")
        shape = tuple(shp)
    return ptrs, shape


def _ptr_array(ptrs):
    return ctypes.cast((ctypes.c_void_p * len(ptrs))(*ptrs), ctypes.c_void_p)


def two_pass_host(src_planes, dst_planes, taps, *, extended: bool = False, ring: bool = True,
                  device: int = 0, devices=None, register: bool = True) -> None:
    """End-to-end two-pass on HOST planes (numpy arrays or CPU tensors; pinned planes
    are copied by DMA directly, pageable ones through the library's pinned staging
    ring): streamed H2D -> fused kernel -> D2H inside the library; blocks until done.
    dst_planes may be src_planes (in place, as conv_two_pass). devices (a list of
    device indices, one process): row bands streamed through every listed GPU
    concurrently (sc_two_pass_host_multi_f32), same bits. register: large numpy
    buffers are page-locked once and kept registered while they live
    (HostRegistry), so repeated calls DMA directly."""
    w = _taps(taps)
    src_planes, dst_planes = list(src_planes), list(dst_planes)
    if register:
        host_registry.new_call()
        for a in src_planes + dst_planes:
            host_registry.pin(a)
    ptrs_in, shape = _host_ptrs(src_planes)
    ptrs_out, _ = _host_ptrs(dst_planes, shape)
    if not ptrs_in or len(ptrs_in) != len(ptrs_out):
        raise InvalidArgumentError("need matching, non-empty source and destination plane lists")
    n = len(ptrs_in)
    arr_in, arr_out = _ptr_array(ptrs_in), _ptr_array(ptrs_out)
    flags = (_lib.SC_EXTENDED if extended else 0) | (0 if ring else _lib.SC_NO_RING)
    L = _lib.load()
    if devices is not None and len(list(devices)) > 1:
        devs = [int(d) for d in devices]
        arr_dev = (ctypes.c_int * len(devs))(*devs)
        _lib.check(L.sc_two_pass_host_multi_f32(arr_in, arr_out, n, shape[0], shape[1], _fp(w),
                                                w.size, flags, ctypes.cast(arr_dev, ctypes.c_void_p), len(devs)))
        return
    if devices is not None and len(list(devices)) == 1:
        device = int(list(devices)[0])
    _lib.check(L.sc_two_pass_host_f32(arr_in, arr_out, n, shape[0], shape[1], _fp(w), w.size, flags, int(device)))


def two_pass_host_split(image_planes, scratch_planes, taps, *, extended: bool = False, device: int = 0,
                        register: bool = True, devices=None) -> None:
    """The reference's end state of convolve_image(TWO_PASS) with a workspace, on HOST
    planes (S/executors.py:303-326): scratch_planes := H0 (zero outside the row
    pass's rows and columns), image_planes[valid] := V(H0) in place, image ring
    untouched. Streamed through the GPU like two_pass_host; blocks until done.
    devices: row bands through several GPUs from this process, same bits."""
    w = _taps(taps)
    image_planes, scratch_planes = list(image_planes), list(scratch_planes)
    if register:
        host_registry.new_call()
        for a in image_planes + scratch_planes:
            host_registry.pin(a)
    ptrs_img, shape = _host_ptrs(image_planes)
    ptrs_scr, _ = _host_ptrs(scratch_planes, shape)
    if not ptrs_img or len(ptrs_img) != len(ptrs_scr):
        raise InvalidArgumentError("need matching, non-empty image and workspace plane lists")
    L = _lib.load()
    flags = _lib.SC_EXTENDED if extended else 0
    if devices is not None and len(list(devices)) > 1:
        devs = [int(d) for d in devices]
        arr_dev = (ctypes.c_int * len(devs))(*devs)
        _lib.check(L.sc_two_pass_host_multi_split_f32(_ptr_array(ptrs_img), _ptr_array(ptrs_scr), len(ptrs_img),
                                                      shape[0], shape[1], _fp(w), w.size, flags,
                                                      ctypes.cast(arr_dev, ctypes.c_void_p), len(devs)))
        return
    if devices is not None and len(list(devices)) == 1:
        device = int(list(devices)[0])
    _lib.check(L.sc_two_pass_host_split_f32(_ptr_array(ptrs_img), _ptr_array(ptrs_scr), len(ptrs_img), shape[0],
                                            shape[1], _fp(w), w.size, flags, int(device)))


def single_pass_host(image_planes, workspace_planes, dense, *, copy_back: bool = False, device: int = 0,
                     register: bool = True, devices=None) -> None:
    """convolve_image's single-pass variants on HOST planes (S/executors.py:327-356):
    workspace_planes[valid] := the dense fold of image_planes; with copy_back the
    same samples also go back into image_planes[valid] in place. Everything else
    in both buffers keeps its values. Streamed through the GPU like
    two_pass_host (chunked H2D / kernel / D2H); blocks until done."""
    m = _dense(dense)
    image_planes, workspace_planes = list(image_planes), list(workspace_planes)
    if register:
        host_registry.new_call()
        for a in image_planes + workspace_planes:
            host_registry.pin(a)
    ptrs_img, shape = _host_ptrs(image_planes)
    ptrs_ws, _ = _host_ptrs(workspace_planes, shape)
    if not ptrs_img or len(ptrs_img) != len(ptrs_ws):
        raise InvalidArgumentError("need matching, non-empty image and workspace plane lists")
    L = _lib.load()
    flags = _lib.SC_COPY_BACK if copy_back else 0
    if devices is not None and len(list(devices)) > 1:  # row bands through several GPUs from this process
        devs = [int(d) for d in devices]
        arr_dev = (ctypes.c_int * len(devs))(*devs)
        _lib.check(L.sc_single_pass_host_multi_f32(_ptr_array(ptrs_img), _ptr_array(ptrs_ws), len(ptrs_img), shape[0],
                                                   shape[1], _fp(m), m.shape[0], flags,
                                                   ctypes.cast(arr_dev, ctypes.c_void_p), len(devs)))
        return
    if devices is not None and len(list(devices)) == 1:
        device = int(list(devices)[0])
    _lib.check(L.sc_single_pass_host_f32(_ptr_array(ptrs_img), _ptr_array(ptrs_ws), len(ptrs_img), shape[0],
                                         shape[1], _fp(m), m.shape[0], _lib.SC_COPY_BACK if copy_back else 0,
                                         int(device)))


def pass_host(src_planes, dst_planes, taps, *, vertical: bool, device: int = 0, register: bool = True) -> None:
    """horizontal_pass / vertical_pass on HOST planes (S/conv.py:362-389): dst[valid] :=
    the row (or column) pass of src; dst elsewhere keeps its values. Streamed
    through the GPU like two_pass_host; blocks until done."""
    w = _taps(taps)
    src_planes, dst_planes = list(src_planes), list(dst_planes)
    if register:
        host_registry.new_call()
        for a in src_planes + dst_planes:
            host_registry.pin(a)
    ptrs_src, shape = _host_ptrs(src_planes)
    ptrs_dst, _ = _host_ptrs(dst_planes, shape)
    if not ptrs_src or len(ptrs_src) != len(ptrs_dst):
        raise InvalidArgumentError("need matching, non-empty source and destination plane lists")
    L = _lib.load()
    _lib.check(L.sc_pass_host_f32(_ptr_array(ptrs_src), _ptr_array(ptrs_dst), len(ptrs_src), shape[0], shape[1],
                                  _fp(w), w.size, 1 if vertical else 0, int(device)))


def two_pass_host_band(src_rows, dst_rows, taps, *, global_rows: int, row0: int, out_lo: int, out_hi: int,
                       extended: bool = False, ring: bool = True, device: int = 0) -> None:
    """One rank's row band of a host-resident image, end to end (streamed H2D ->
    fused kernel -> D2H, global-row rules): src_rows / dst_rows are host planes
    holding global rows [row0, row0 + their height); output rows [out_lo, out_hi)
    are written into dst_rows, reading src rows [out_lo - r, out_hi + r). No
    exchange with other ranks is needed: every rank reads its halo rows from its
    own host copy."""
    w = _taps(taps)
    r = w.size // 2
    ptrs_in, ptrs_out, shape = [], [], None
    for a, b in zip(src_rows, dst_rows):
        for arr in (a, b):
            if not isinstance(arr, torch.Tensor) or arr.is_cuda or arr.dtype != torch.float32 or \
                    not arr.is_contiguous() or arr.dim() != 2:
                raise InvalidArgumentError("band host planes must be contiguous 2-D CPU float32 tensors")
            if shape is not None and tuple(arr.shape) != shape:
                raise InvalidArgumentError("band host planes must share one shape")
            shape = tuple(arr.shape)
        C = shape[1]
        # address of the (virtual) global row 0: the library touches rows inside the band only
        ptrs_in.append(a.data_ptr() - row0 * C * 4)
        ptrs_out.append(b.data_ptr() - row0 * C * 4)
    if not ptrs_in:
        raise InvalidArgumentError("need non-empty plane lists")
    held_lo, held_hi = row0, row0 + shape[0]
    if max(out_lo - r, 0) < held_lo or min(out_hi + r, global_rows) > held_hi or out_lo < held_lo or out_hi > held_hi:
        raise InvalidArgumentError("the band's host rows do not cover the output rows plus halo")
    n = len(ptrs_in)
    arr_in = (ctypes.c_void_p * n)(*ptrs_in)
    arr_out = (ctypes.c_void_p * n)(*ptrs_out)
    flags = (_lib.SC_EXTENDED if extended else 0) | (0 if ring else _lib.SC_NO_RING)
    L = _lib.load()
    _lib.check(L.sc_two_pass_host_band_f32(ctypes.cast(arr_in, ctypes.c_void_p),
                                           ctypes.cast(arr_out, ctypes.c_void_p), n, global_rows, shape[1],
                                           out_lo, out_hi, _fp(w), w.size, flags, int(device)))


# ---------------------------------------------------------------------------
# PPM payload (interleaved u8 HWC, S/ppm.py) either side of the path

def _hwc(t: torch.Tensor, what: str):
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.uint8:
        raise InvalidArgumentError(f"{what} must be a CUDA uint8 tensor")
    if t.dim() != 3 or t.shape[2] != 3 or t.stride(2) != 1 or t.stride(1) != 3:
        raise InvalidArgumentError(f"{what} must be (rows, cols, 3) with interleaved pixels")
    return t.shape[0], t.shape[1], t.stride(0)


def hwc_to_planes(src: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(R, C, 3) uint8 -> (3, R, C) float32 (read_ppm_bytes, S/ppm.py:72-73)."""
    R, C, srs = _hwc(src, "src")
    if out is None:
        out = torch.empty((3, R, C), dtype=torch.float32, device=src.device)
    n, R2, C2, ps, rs = _planes(out, "out")
    if (n, R2, C2) != (3, R, C):
        raise InvalidArgumentError("out must be (3, rows, cols)")
    L = _lib.load()
    _lib.check(L.sc_hwc_u8_to_planes_f32(src.data_ptr(), out.data_ptr(), R, C, srs, ps, rs, _stream(src)))
    return out


def planes_to_hwc(src: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """(3, R, C) float32 -> (R, C, 3) uint8 with clip(rint(x), 0, 255) (S/ppm.py:87-89)."""
    n, R, C, ps, rs = _planes(src, "src")
    if n != 3:
        raise InvalidArgumentError(f"PPM output needs exactly 3 planes, image has {n}")
    if out is None:
        out = torch.empty((R, C, 3), dtype=torch.uint8, device=src.device)
    R2, C2, drs = _hwc(out, "out")
    if (R2, C2) != (R, C):
        raise InvalidArgumentError("out must be (rows, cols, 3)")
    L = _lib.load()
    _lib.check(L.sc_planes_f32_to_hwc_u8(src.data_ptr(), out.data_ptr(), R, C, ps, rs, drs, _stream(src)))
    return out


def two_pass_u8hwc(src: torch.Tensor, taps, out: torch.Tensor | None = None, *,
                   extended: bool = False) -> torch.Tensor:
    """read_ppm -> two-pass -> write_ppm on a (R, C, 3) uint8 payload: one fused
    kernel (3 B/pixel each way) for taps of width 1..9 and any row geometry (odd
    cols, padded or unaligned rows: the kernel's general build); wider taps run
    unpack, fused float two-pass and pack, all on the GPU. Same output bytes
    either way."""
    w = _taps(taps)
    R, C, srs = _hwc(src, "src")
    if out is None:
        out = torch.empty_like(src)
    R2, C2, drs = _hwc(out, "out")
    if (R2, C2) != (R, C):
        raise InvalidArgumentError("source and destination dimensions differ")
    flags = _lib.SC_EXTENDED if extended else 0
    L = _lib.load()
    if w.size <= 9:  # the fused u8 kernel covers widths 1..9; wider taps take the planes path
        _lib.check(L.sc_two_pass_u8hwc(src.data_ptr(), out.data_ptr(), R, C, srs, drs, _fp(w), w.size, flags,
                                       _stream(src)))
        return out
    planes = hwc_to_planes(src)
    conv = two_pass(planes, w, extended=extended)
    return planes_to_hwc(conv, out)
