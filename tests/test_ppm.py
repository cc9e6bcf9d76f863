"""PPM payload either side of the path (S/ppm.py): header parsing on CPU against
the reference's own errors/offsets; GPU unpack/pack and the fused
read -> two-pass -> write kernel against bytes the reference wrote."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden


def test_header_errors_match_reference():
    from paper_1711_09791_b200.errors import PpmParseError
    from paper_1711_09791_b200.ppm import parse_header

    z = load_golden("ppm")
    for i, (msg, off) in enumerate(zip(z["bad_messages"], z["bad_offsets"])):
        data = z[f"bad_{i}"].tobytes()
        if off < 0:
            parse_header(data)
            continue
        with pytest.raises(PpmParseError) as ei:
            parse_header(data)
        assert str(ei.value) == str(msg) and ei.value.byte_offset == int(off), i


def test_header_of_valid_files():
    from paper_1711_09791_b200.ppm import parse_header

    z = load_golden("ppm")
    for key in z:
        if key.startswith("in_"):
            R, C = (int(v) for v in key[3:].split("_")[0].split("x"))
            rows, cols, pos = parse_header(z[key].tobytes())
            assert (rows, cols) == (R, C) and len(z[key]) - pos == R * C * 3


def _cases():
    z = load_golden("ppm")
    return sorted(k[3:] for k in z if k.startswith("in_"))


@pytest.mark.gpu
@pytest.mark.parametrize("key", _cases())
def test_fused_ppm_convolution_matches_reference_bytes(key):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200.ppm import convolve_ppm_bytes, read_ppm_bytes, write_ppm_bytes

    z = load_golden("ppm")
    data = z[f"in_{key}"].tobytes()
    want = z[f"out_{key}"].tobytes()
    assert convolve_ppm_bytes(data, z[f"taps_{key}"]) == want
    img = read_ppm_bytes(data)
    assert np.array_equal(np.stack([p.data for p in img.planes]), z[f"planes_{key}"])
    dimg = read_ppm_bytes(data, device="cuda")
    assert write_ppm_bytes(dimg) == data  # integer planes round-trip byte for byte


@pytest.mark.gpu
def test_pack_rounding_half_even_and_clip():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device as dev

    vals = np.array([-3.0, -0.5, -0.0, 0.4999, 0.5, 1.5, 2.5, 2.5000002, 127.5, 128.5, 254.5, 255.49, 255.5,
                     300.0, np.inf, -np.inf, 1e30], dtype=np.float32)
    n = vals.size
    planes = np.stack([vals, vals[::-1], np.roll(vals, 3)]).reshape(3, 1, n).astype(np.float32)
    got = dev.planes_to_hwc(torch.from_numpy(planes).cuda()).cpu().numpy()
    want = np.clip(np.rint(np.moveaxis(planes, 0, -1)), 0, 255).astype(np.uint8)
    assert np.array_equal(got, want)


@pytest.mark.gpu
def test_fused_u8_large_against_float_path():
    """cfg-sized payload: the fused u8 kernel equals unpack -> fused f32 -> pack."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device as dev

    R, C = 1080, 1920
    g = torch.Generator(device="cuda").manual_seed(3)
    src = torch.randint(0, 256, (R, C, 3), dtype=torch.uint8, device="cuda", generator=g)
    # gauss5 and [0, .5, 0, .5, 0] put many outputs on exact .5 ties (round half
    # even), the sharpen taps drive outputs far outside [0, 255] (clip)
    for taps in ([1 / 16, 4 / 16, 6 / 16, 4 / 16, 1 / 16], [0, 0.5, 0, 0.5, 0], [-1, -2, 7, -2, -1]):
        fused = dev.two_pass_u8hwc(src, np.asarray(taps, np.float32))
        ref = dev.planes_to_hwc(dev.two_pass(dev.hwc_to_planes(src), np.asarray(taps, np.float32)))
        assert torch.equal(fused, ref)


@pytest.mark.gpu
def test_fused_u8_large_payload_lean_loops():
    """Payloads of >= 32 Mpixel take the u8 kernel's lean loops (interior strips,
    full stages without per-row tests): same bytes as unpack -> fused f32 -> pack."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device as dev

    R, C = 4100, 8192  # 33.6 Mpixel; 4100 rows: the last band is short
    g = torch.Generator(device="cuda").manual_seed(11)
    src = torch.randint(0, 256, (R, C, 3), dtype=torch.uint8, device="cuda", generator=g)
    for taps in ([1 / 16, 4 / 16, 6 / 16, 4 / 16, 1 / 16], [-1, -2, 7, -2, -1], [0.1, -0.3, 0.9, 0.2, 0.1]):
        w = np.asarray(taps, np.float32)
        fused = dev.two_pass_u8hwc(src, w)
        ref = dev.planes_to_hwc(dev.two_pass(dev.hwc_to_planes(src), w))
        assert torch.equal(fused, ref)
        fused_ext = dev.two_pass_u8hwc(src, w, extended=True)
        ref_ext = dev.planes_to_hwc(dev.two_pass(dev.hwc_to_planes(src), w, extended=True))
        assert torch.equal(fused_ext, ref_ext)


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["32x48", "40x64"])
def test_fused_u8_subnormal_taps(key):
    """Subnormal / near-FLT_MIN taps through the fused u8 kernel (cols % 16 == 0) and
    the float planes path: bytes and float planes the reference produced
    (tests/golden/make_golden.py subnormal_ppm)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.ppm import convolve_ppm_bytes, read_ppm_bytes

    z = load_golden("subnormal_ppm")
    data = z[f"in_{key}"].tobytes()
    assert convolve_ppm_bytes(data, z[f"taps_{key}"]) == z[f"out_{key}"].tobytes()
    planes = np.stack([p.data for p in read_ppm_bytes(data).planes])
    got = dev.two_pass(torch.from_numpy(planes).cuda(), z[f"taps_{key}"]).cpu().numpy()
    assert np.array_equal(got.view(np.uint32), z[f"planes_out_{key}"].view(np.uint32))


def _u8_view(torch, R, C, pad, off, seed):
    """(R, C, 3) uint8 view `off` bytes into a buffer, rows `3C + pad` bytes apart."""
    srs = 3 * C + pad
    g = torch.Generator(device="cuda").manual_seed(seed)
    buf = torch.randint(0, 256, (off + R * srs + 64,), dtype=torch.uint8, device="cuda", generator=g)
    return buf, buf.as_strided((R, C, 3), (srs, 3, 1), off)


# (rows, cols, source row padding, source offset, destination row padding, destination offset)
_GEOMETRIES = [(9, 9, 0, 0, 0, 0), (37, 17, 0, 1, 0, 0), (64, 33, 5, 3, 0, 1), (23, 127, 0, 7, 2, 2),
               (130, 1001, 1, 13, 3, 3), (75, 1921, 0, 0, 0, 0), (48, 640, 7, 0, 0, 0), (48, 640, 0, 0, 1, 0),
               (33, 2050, 0, 15, 0, 3), (520, 517, 2, 5, 1, 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("geom", _GEOMETRIES, ids=lambda g: "x".join(map(str, g)))
def test_fused_u8_any_geometry(geom):
    """The fused u8 kernel's general build (cols % 16 != 0, padded rows, rows and
    buffers at any byte offset): the same bytes as unpack -> fused f32 -> pack, for
    every tap width 1..9 (mirror-symmetric and not), in both ring modes, and no
    byte outside the destination view touched."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import device as dev

    R, C, spad, soff, dpad, doff = geom
    _, src = _u8_view(torch, R, C, spad, soff, R * 7 + C)
    rng = np.random.default_rng(R + C)
    taps = [np.array([1.0], np.float32), np.array([0.25, 0.5, 0.25], np.float32),
            np.float32([1, 4, 6, 4, 1]) / np.float32(16), np.float32([-1, -2, 7, -2, -1]),
            rng.standard_normal(7).astype(np.float32), np.float32([1, 2, 3, 4, 5, 4, 3, 2, 1]) / np.float32(25),
            rng.uniform(-0.5, 1, 9).astype(np.float32)]
    for w in taps:
        if w.size > min(R, C):
            continue
        for extended in (False, True):
            dbuf, dst = _u8_view(torch, R, C, dpad, doff, 99)
            before = dbuf.clone()
            dev.two_pass_u8hwc(src, w, dst, extended=extended)
            ref = dev.planes_to_hwc(dev.two_pass(dev.hwc_to_planes(src), w, extended=extended))
            assert torch.equal(dst, ref), (w.size, extended)
            mask = torch.ones_like(dbuf, dtype=torch.bool)
            mask.as_strided((R, C, 3), (3 * C + dpad, 3, 1), doff).fill_(False)
            assert torch.equal(dbuf[mask], before[mask]), "bytes outside the view were written"


@pytest.mark.gpu
def test_fused_u8_general_build_on_aligned_rows_and_large_payloads():
    """SC_U8_GEN=1 forces the general build on aligned rows (it must equal the
    aligned build), and a >= 32 Mpixel payload with odd cols runs the general
    build's lean loops."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import os

    from paper_1711_09791_b200 import device as dev

    w = np.float32([1, 4, 6, 4, 1]) / np.float32(16)
    g = torch.Generator(device="cuda").manual_seed(5)
    src = torch.randint(0, 256, (1080, 1920, 3), dtype=torch.uint8, device="cuda", generator=g)
    want = dev.two_pass_u8hwc(src, w)
    os.environ["SC_U8_GEN"] = "1"
    try:
        got = dev.two_pass_u8hwc(src, w)
    finally:
        del os.environ["SC_U8_GEN"]
    assert torch.equal(got, want)
    _, big = _u8_view(torch, 4097, 8195, 1, 3, 21)  # 33.6 Mpixel
    for taps in (w, np.float32([0.1, -0.3, 0.9, 0.2, 0.1])):
        fused = dev.two_pass_u8hwc(big, taps)
        ref = dev.planes_to_hwc(dev.two_pass(dev.hwc_to_planes(big), taps))
        assert torch.equal(fused, ref)
