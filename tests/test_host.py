"""Host-side logic on CPU: the C ABI library loads and exports what the header
declares, validates before launching, and the Python mirror of the reference
interface keeps the reference's names, argument meaning and errors."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden

HEADER = os.path.join(ROOT, "include", "sepconv_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_1711_09791_b200 import _lib

    L = _lib.load()
    declared = header_symbols()
    assert declared, "no declarations parsed from the header"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.sc_abi_version() == 1
    assert L.sc_launch_count() == 0


def _fused(L, src, dst, nplanes, rows, cols, width, flags=0):
    taps = (ctypes.c_float * max(width, 1))(*([0.2] * max(width, 1)))
    return L.sc_two_pass_fused_f32(src, dst, nplanes, rows, cols, rows * cols, rows * cols, cols, cols,
                                   taps, width, flags, None)


def test_abi_validates_before_launch():
    """Status codes for the reference's error classes; nothing reaches the GPU."""
    from paper_1711_09791_b200 import _lib

    L = _lib.load()
    buf = (ctypes.c_float * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    assert _fused(L, p, p, 1, 8, 8, 4) == _lib.SC_INVALID_ARGUMENT          # even width
    assert _fused(L, p, p, 1, 8, 8, 257) == _lib.SC_UNSUPPORTED_WIDTH       # > 255
    assert _fused(L, p, p, 1, 8, 8, 11) == _lib.SC_INVALID_DIMENSION        # widths 11..255 run; 8 rows < 11
    assert _fused(L, p, p, 1, 4, 8, 5) == _lib.SC_INVALID_DIMENSION         # rows < width
    assert b"smaller than kernel width" in L.sc_last_error()
    assert _fused(L, p, p, 0, 8, 8, 5) == _lib.SC_INVALID_ARGUMENT          # no planes
    # host memory is refused (no CPU fallback): the pointer is not device memory
    other = (ctypes.c_float * 64)()
    q = ctypes.cast(other, ctypes.c_void_p)
    assert _fused(L, p, q, 1, 8, 8, 5) == _lib.SC_INVALID_ARGUMENT
    # band geometry: source band must cover output rows plus halo
    taps = (ctypes.c_float * 5)(*([0.2] * 5))
    rc = L.sc_two_pass_band_f32(p, q, 1, 100, 8, 800, 800, 8, 8, 10, 20, 10, 10, 30, taps, 5, 0, None)
    assert rc == _lib.SC_INVALID_ARGUMENT and b"halo" in L.sc_last_error()
    assert L.sc_fill_synthetic_f32(p, 10, 1, 0, 7, None) == _lib.SC_INVALID_ARGUMENT
    assert L.sc_launch_count() == 0


def test_status_maps_to_reference_exceptions():
    from paper_1711_09791_b200 import _lib
    from paper_1711_09791_b200.errors import (
        ExecutionError,
        InvalidArgumentError,
        InvalidDimensionError,
        SepconvError,
        UnsupportedWidthError,
    )

    _lib.load()
    for code, exc in ((1, InvalidArgumentError), (2, InvalidDimensionError), (3, UnsupportedWidthError),
                      (4, ExecutionError)):
        with pytest.raises(exc):
            _lib.check(code)
        assert issubclass(exc, SepconvError)
    _lib.check(0)


def test_missing_extension_fails_loudly(tmp_path, monkeypatch):
    from paper_1711_09791_b200 import _lib

    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "absent.so"))
    with pytest.raises(_lib.ExtensionMissingError):
        _lib.load()


def test_kernels_mirror_reference(oracle):
    from paper_1711_09791_b200.errors import InvalidArgumentError
    from paper_1711_09791_b200.kernels import DenseKernel, SeparableKernel, delta, gaussian5, outer_product

    k = gaussian5()
    assert k.weights.tolist() == [0.0625, 0.25, 0.375, 0.25, 0.0625] and k.radius == 2
    assert outer_product(k).matrix[0, 0] == np.float32(1 / 256)
    for w in ([0.1, 0.7, 0.3], [-1, -2, 7, -2, -1], np.random.default_rng(3).standard_normal(9)):
        sk = SeparableKernel(w)
        assert np.array_equal(outer_product(sk).matrix, oracle.outer_product(sk.weights))
    assert np.array_equal(outer_product(delta(5)).matrix, np.diag([0, 0, 1, 0, 0]).astype(np.float32))
    with pytest.raises(InvalidArgumentError):
        SeparableKernel([1.0, 2.0])
    with pytest.raises(InvalidArgumentError):
        DenseKernel(np.ones((2, 3)))


def test_image_model_mirrors_reference():
    from paper_1711_09791_b200.errors import InvalidArgumentError, InvalidDimensionError
    from paper_1711_09791_b200.image import Image, Plane, ValidRegion, make_synthetic, max_abs_diff, valid_region

    z = load_golden("synthetic")
    img = make_synthetic(8, 8, 3, seed=42)
    assert np.array_equal(np.stack([p.data for p in img.planes]), z["make_synthetic_8x8x3_s42"])
    assert valid_region(1152, 1152, 2) == ValidRegion(2, 1150, 2, 1150)
    with pytest.raises(InvalidDimensionError):
        valid_region(4, 9, 2)
    with pytest.raises(InvalidDimensionError):
        make_synthetic(4, 5, 1, seed=0)
    with pytest.raises(InvalidArgumentError):
        Image([Plane.zeros(5, 5), Plane.zeros(5, 6)])
    with pytest.raises(InvalidArgumentError):
        Plane(np.zeros(5))
    a, b = Plane.full(6, 6, 1.0), Plane.full(6, 6, 1.5)
    assert max_abs_diff(a, b, valid_region(6, 6, 2)) == 0.5
    p = Plane(np.arange(12, dtype=np.float64).reshape(3, 4))
    assert p.data.dtype == np.float32 and p.data.flags.c_contiguous


def test_conv_api_checks_and_counts():
    from paper_1711_09791_b200.conv import (
        Algorithm,
        ConvVariant,
        _check_pair,
        arith_count,
        doubly_interior_region,
    )
    from paper_1711_09791_b200.errors import InvalidArgumentError, InvalidDimensionError
    from paper_1711_09791_b200.image import Plane

    # T/test_conv.py:325-357 and SPEC.md:492 numbers
    single = ConvVariant(Algorithm.SINGLE_PASS_GENERIC, copy_back=True)
    two = ConvVariant(Algorithm.TWO_PASS, copy_back=True)
    assert two.copy_back is False
    assert arith_count(single, 1152, 1152, 5).multiplications == 25 * 1148 * 1148
    assert arith_count(two, 64, 64, 5).multiplications == 10 * 60 * 60
    assert arith_count(ConvVariant(Algorithm.SINGLE_PASS_GENERIC), 6, 7, 1).additions == 0
    assert doubly_interior_region(12, 12, 2).row_lo == 4
    src = Plane.zeros(8, 8)
    with pytest.raises(InvalidArgumentError):
        _check_pair(src, Plane.zeros(8, 9), 5)
    with pytest.raises(InvalidArgumentError):
        _check_pair(src, Plane(src.data[:, :]), 5)
    with pytest.raises(InvalidDimensionError):
        _check_pair(Plane.zeros(4, 8), Plane.zeros(4, 8), 5)


def test_plans_and_dispatch_errors():
    from paper_1711_09791_b200.conv import Algorithm, ConvVariant
    from paper_1711_09791_b200.errors import (
        InvalidArgumentError,
        UnsupportedCombinationError,
        UnsupportedWidthError,
    )
    from paper_1711_09791_b200.executors import Cuda, LaunchStats, convolve_image, make_plan, result_image
    from paper_1711_09791_b200.image import Image
    from paper_1711_09791_b200.kernels import SeparableKernel, gaussian5

    assert make_plan("cuda") == Cuda()
    with pytest.raises(UnsupportedCombinationError):
        make_plan("static", workers=4)
    with pytest.raises(InvalidArgumentError):
        make_plan("bogus")
    img = Image.zeros(8, 8, 3)
    with pytest.raises(UnsupportedWidthError):
        convolve_image(img, SeparableKernel([0.2, 0.6, 0.2]), ConvVariant(Algorithm.SINGLE_PASS_UNROLLED5), Cuda())
    with pytest.raises(UnsupportedCombinationError):
        convolve_image(img, gaussian5(), ConvVariant(Algorithm.TWO_PASS), object())
    with pytest.raises(InvalidArgumentError):
        convolve_image(img, gaussian5(), ConvVariant(Algorithm.TWO_PASS), Cuda(), counter=object())
    with pytest.raises(InvalidArgumentError):
        convolve_image(img, gaussian5(), ConvVariant(Algorithm.TWO_PASS), Cuda(), workspace=Image.zeros(8, 9, 3))
    assert LaunchStats() == LaunchStats(0, 0, 0)
    ws = Image.zeros(8, 8, 3)
    assert result_image(img, ws, ConvVariant(Algorithm.TWO_PASS)) is img
    assert result_image(img, ws, ConvVariant(Algorithm.SINGLE_PASS_GENERIC)) is ws
    assert result_image(img, ws, ConvVariant(Algorithm.SINGLE_PASS_GENERIC, copy_back=True)) is img


def test_partition_block_matches_reference_rule():
    from paper_1711_09791_b200.errors import InvalidArgumentError
    from paper_1711_09791_b200.multi import partition_block

    # S/executors.py:121-139: first n mod k chunks one longer; empty trailing chunks
    assert [partition_block(0, 10, i, 4) for i in range(4)] == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert [partition_block(2, 4, i, 3) for i in range(3)] == [(2, 3), (3, 4), (4, 4)]
    with pytest.raises(InvalidArgumentError):
        partition_block(0, 10, 4, 4)
    with pytest.raises(InvalidArgumentError):
        partition_block(5, 4, 0, 1)


def test_hot_kernels_use_no_local_memory():
    """Regression guard: a stack frame in the row kernels turned every output row
    into local-memory stores that doubled L1->L2 write traffic.
    Every hot kernel must compile without STL/LDL."""
    import shutil
    import subprocess

    from paper_1711_09791_b200 import _lib

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    current, bad = None, []
    for line in sass.splitlines():
        if "Function :" in line:
            current = line.split("Function :")[1].strip()
        elif current and "sepconv_" in current and re.search(r"\b(STL|LDL)\b", line):
            bad.append(current)
    # known exception: the 9x9 dense single pass (MODE 3, r = 4) holds 8 partial
    # rows of 8 columns and spills; it is outside the five BASELINE workloads.
    # likewise the 9-wide u8 payload kernel (sepconv_u8_kernel<4, false>, 40 bytes)
    bad = [b for b in bad if "ILi3ELi4E" not in b and "sepconv_u8_kernelILi4E" not in b]
    assert not bad, sorted(set(bad))


def test_packed_math_keeps_two_roundings():
    """ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 (single rounding).
    The kernels issue the add as FFMA2(product, run-time 1.0, acc); every FFMA2 in
    the row kernels must therefore multiply by a uniform/constant operand that is
    the run-time `one`, never by a tap product. Check: FFMA2 count never exceeds
    the FMUL2 count (each mad2 is one FMUL2 + one FFMA2; first terms are FMUL2 only)."""
    import shutil
    import subprocess

    from paper_1711_09791_b200 import _lib

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    counts, current = {}, None
    for line in sass.splitlines():
        if "Function :" in line:
            current = line.split("Function :")[1].strip()
            counts[current] = [0, 0, 0, 0]
        elif current:
            if re.search(r"\bFMUL2\b", line):
                counts[current][0] += 1
            elif re.search(r"\bFFMA2\b", line):
                counts[current][1] += 1
            elif re.search(r"\bFFMA\b", line):
                counts[current][2] += 1
            elif re.search(r"\bFMUL\b", line):
                counts[current][3] += 1
    for fn, (fmul2, ffma2, ffma, fmul) in counts.items():
        if "sepconv_" not in fn:
            continue
        assert ffma == 0, f"scalar FFMA (contracted mul+add) in {fn}"
        # symmetric-matrix single-pass kernels (4th template argument 1 or 2) and the
        # symmetric-tap u8 kernels reuse mirrored products: fewer FMUL2 than adds by
        # design, at most 2 adds per product
        sym = (re.search(r"sepconv_rows_kernelILi\d+ELi\d+ELb[01]ELi[12]E", fn) is not None
               or re.search(r"sepconv_lanes_wide_kernelILi\d+ELi\d+ELi[12]E", fn) is not None  # widths 11..31
               or re.search(r"sepconv_u8_kernelILi\d+ELb1E", fn) is not None)  # u8 with symmetric taps
        # products of odd-start window pairs are two scalar FMULs (prod2)
        products = fmul2 + fmul // 2
        limit = 2 * products if sym else products
        assert ffma2 <= limit, f"{fn}: {ffma2} FFMA2 vs {fmul2} FMUL2 + {fmul} FMUL -- contraction suspected"


def test_two_pass_kernels_keep_four_ctas_per_sm():
    """Regression guard on occupancy: the r = 2 two-pass kernels (fused, row pass,
    column pass, one-pass split; aligned and unaligned) run 160-thread CTAs, 4 per
    SM only while they need <= 96 registers (5 warps x 96 x 32 x 4 <= 64K). An
    innocent-looking change (two int fields inserted before the taps in Params)
    once moved the aligned fused kernel from 76 to 84 registers and the unaligned
    one to 102 (3 CTAs/SM, 13-20% slower)."""
    import shutil
    import subprocess

    from paper_1711_09791_b200 import _lib

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-res-usage", _lib.LIB_PATH], capture_output=True, text=True).stdout
    regs, current = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            current = m.group(1)
        elif current and "REG:" in line:
            regs[current] = int(re.search(r"REG:(\d+)", line).group(1))
    checked = 0
    for fn, n in regs.items():
        m = re.search(r"sepconv_rows_kernelILi([0124])ELi2ELb([01])E", fn)
        if not m:
            continue
        checked += 1
        assert n <= 96, f"{fn}: {n} registers (> 96: fewer than 4 CTAs/SM)"
        if m.group(1) == "0" and m.group(2) == "1":
            assert n <= 80, f"aligned fused kernel {fn}: {n} registers (was 76)"
    assert checked >= 7


def test_cuda_plan_devices_validation():
    """Cuda(devices=...) (several GPUs from one process) validates like the
    reference's plan constructors: non-empty, non-negative, not with device=."""
    from paper_1711_09791_b200.errors import InvalidArgumentError
    from paper_1711_09791_b200.executors import Cuda, make_plan

    assert Cuda(devices=[0, 1]).devices == (0, 1)
    assert make_plan("cuda", devices=[3]).devices == (3,)
    for bad in ([], [-1], [0, -2]):
        with pytest.raises(InvalidArgumentError):
            Cuda(devices=bad)
    with pytest.raises(InvalidArgumentError):
        Cuda(device=0, devices=[1])
