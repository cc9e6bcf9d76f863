"""ctypes binding of libsepconv_b200.so (include/sepconv_b200.h).

The library is the product path: there is no CPU fallback. If the shared
object is missing or cannot be loaded, every entry point raises
``ExtensionMissingError`` instead of computing anything.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (
    ExecutionError,
    InvalidArgumentError,
    InvalidDimensionError,
    SepconvError,
    UnsupportedWidthError,
)

LIB_PATH = os.environ.get("SEPCONV_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libsepconv_b200.so")

SC_OK = 0
SC_INVALID_ARGUMENT = 1
SC_INVALID_DIMENSION = 2
SC_UNSUPPORTED_WIDTH = 3
SC_CUDA_ERROR = 4
SC_NCCL_ERROR = 5

SC_EXTENDED = 0x1
SC_NO_RING = 0x2
SC_ZERO_FILL = 0x4
SC_COPY_BACK = 0x8

# every symbol include/sepconv_b200.h declares
EXPORTS = (
    "sc_abi_version",
    "sc_last_error",
    "sc_launch_count",
    "sc_two_pass_fused_f32",
    "sc_two_pass_band_f32",
    "sc_two_pass_band2_f32",
    "sc_two_pass_band_peer_f32",
    "sc_two_pass_band_peer_sig_f32",
    "sc_band_signal_wait",
    "sc_nccl_unique_id",
    "sc_nccl_comm_init",
    "sc_nccl_comm_destroy",
    "sc_band_plan_create",
    "sc_band_plan_step",
    "sc_band_plan_graphed",
    "sc_band_plan_destroy",
    "sc_ipc_export",
    "sc_ipc_open",
    "sc_ipc_close",
    "sc_hpass_f32",
    "sc_vpass_f32",
    "sc_two_pass_split_f32",
    "sc_two_pass_inplace_f32",
    "sc_single_pass_f32",
    "sc_copy_region_f32",
    "sc_fill_synthetic_f32",
    "sc_two_pass_host_f32",
    "sc_two_pass_host_split_f32",
    "sc_single_pass_host_f32",
    "sc_single_pass_host_multi_f32",
    "sc_pass_host_f32",
    "sc_host_register",
    "sc_host_unregister",
    "sc_two_pass_host_band_f32",
    "sc_two_pass_host_multi_f32",
    "sc_two_pass_host_multi_split_f32",
    "sc_two_pass_u8hwc",
    "sc_hwc_u8_to_planes_f32",
    "sc_planes_f32_to_hwc_u8",
)


class ExtensionMissingError(SepconvError, RuntimeError):
    """libsepconv_b200.so is not built or failed to load (no CPU fallback exists)."""


_lock = threading.Lock()
_lib = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_fp = ctypes.c_void_p  # const float* (taps / dense matrix), passed as an address

_STRIDED = [_vp, _vp, _i32, _i32, _i32, _i64, _i64, _i64, _i64]

_SIGNATURES = {
    "sc_abi_version": ([], _i32),
    "sc_last_error": ([], ctypes.c_char_p),
    "sc_launch_count": ([], _u64),
    "sc_two_pass_fused_f32": (_STRIDED + [_fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_band_f32": (_STRIDED + [_i32, _i32, _i32, _i32, _i32, _fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_band2_f32": (_STRIDED + [_i32] * 7 + [_fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_band_peer_f32": (_STRIDED + [_i32, _i32, _vp, _i32, _i32, _i64, _i64, _vp, _i32, _i32, _i64, _i64,
                                              _i32, _i32, _i32, _fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_band_peer_sig_f32": (_STRIDED + [_i32, _i32, _vp, _i32, _i32, _i64, _i64, _vp, _i32, _i32, _i64,
                                                  _i64, _i32, _i32, _i32, _fp, _i32, _i32, _vp, _vp, _vp, _u64, _vp,
                                                  _vp], _i32),
    "sc_band_signal_wait": ([_vp, _vp, _i32, _u64, _vp, _vp], _i32),
    "sc_nccl_unique_id": ([_vp], _i32),
    "sc_nccl_comm_init": ([_vp, _i32, _i32, _i32, ctypes.POINTER(_vp)], _i32),
    "sc_nccl_comm_destroy": ([_vp], _i32),
    "sc_band_plan_create": ([_vp] + _STRIDED + [_i32, _i32, _i32, _i32, _fp, _i32, _i32, _i32, ctypes.POINTER(_vp)],
                            _i32),
    "sc_band_plan_step": ([_vp, _vp], _i32),
    "sc_band_plan_graphed": ([_vp], _i32),
    "sc_band_plan_destroy": ([_vp], _i32),
    "sc_ipc_export": ([_vp, _vp, ctypes.POINTER(_i64)], _i32),
    "sc_ipc_open": ([_vp, _i64, _i32, ctypes.POINTER(_vp)], _i32),
    "sc_ipc_close": ([_vp, _i64], _i32),
    "sc_hpass_f32": (_STRIDED + [_i32, _i32, _fp, _i32, _i32, _vp], _i32),
    "sc_vpass_f32": (_STRIDED + [_i32, _i32, _fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_split_f32": (_STRIDED + [_fp, _i32, _i32, _vp], _i32),
    "sc_two_pass_inplace_f32": ([_vp, _i32, _i32, _i32, _i64, _i64, _fp, _i32, _i32, _vp], _i32),
    "sc_single_pass_f32": (_STRIDED + [_fp, _i32, _i32, _vp], _i32),
    "sc_copy_region_f32": (_STRIDED + [_i32, _i32, _i32, _i32, _vp], _i32),
    "sc_fill_synthetic_f32": ([_vp, _i64, _u64, _u64, _i32, _vp], _i32),
    "sc_two_pass_host_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _i32], _i32),
    "sc_host_register": ([_vp, _i64], _i32),
    "sc_host_unregister": ([_vp], _i32),
    "sc_two_pass_host_split_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _i32], _i32),
    "sc_single_pass_host_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _i32], _i32),
    "sc_pass_host_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _i32], _i32),
    "sc_single_pass_host_multi_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _vp, _i32], _i32),
    "sc_two_pass_host_band_f32": ([_vp, _vp, _i32, _i32, _i32, _i32, _i32, _fp, _i32, _i32, _i32], _i32),
    "sc_two_pass_host_multi_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _vp, _i32], _i32),
    "sc_two_pass_host_multi_split_f32": ([_vp, _vp, _i32, _i32, _i32, _fp, _i32, _i32, _vp, _i32], _i32),
    "sc_two_pass_u8hwc": ([_vp, _vp, _i32, _i32, _i64, _i64, _fp, _i32, _i32, _vp], _i32),
    "sc_hwc_u8_to_planes_f32": ([_vp, _vp, _i32, _i32, _i64, _i64, _i64, _vp], _i32),
    "sc_planes_f32_to_hwc_u8": ([_vp, _vp, _i32, _i32, _i64, _i64, _i64, _vp], _i32),
}


def load():
    """Load (once) and return the ctypes library; raises ExtensionMissingError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissingError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1711_09791_b200.build` "
                "(there is no CPU fallback)"
            )
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:  # pragma: no cover - depends on the box
            raise ExtensionMissingError(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (args, res) in _SIGNATURES.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                # a substituted build of an older ABI (SEPCONV_B200_LIB, dev A/B
                # timings) may lack newer entry points; the shipped library may not
                if os.environ.get("SEPCONV_B200_LIB"):
                    continue
                raise ExtensionMissingError(f"{LIB_PATH} lacks {name}: rebuild it") from None
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def last_error() -> str:
    return load().sc_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().sc_launch_count())


def check(status: int) -> None:
    """Map an SC_* status onto the reference's exception hierarchy (S/errors.py)."""
    if status == SC_OK:
        return
    msg = last_error() or f"status {status}"
    if status == SC_INVALID_ARGUMENT:
        raise InvalidArgumentError(msg)
    if status == SC_INVALID_DIMENSION:
        raise InvalidDimensionError(msg)
    if status == SC_UNSUPPORTED_WIDTH:
        raise UnsupportedWidthError(msg)
    raise ExecutionError([(0, RuntimeError(msg))])  # SC_CUDA_ERROR, SC_NCCL_ERROR


def floats(values) -> ctypes.Array:
    vals = [float(v) for v in values]
    return (ctypes.c_float * len(vals))(*vals)
