"""The reference-facing API (paper_1711_09791_b200 mirrors sepconv_lab's names)
on the GPU: host numpy planes and HBM-resident planes, checked against the
fixtures the reference itself produced, plus ports of the reference's own
conv tests (T/test_conv.py) run through this package."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SENTINEL = np.float32(-777.0)


@pytest.fixture(scope="module")
def sc():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1711_09791_b200 as sc

    return sc


def host_image(sc, arr):
    return sc.Image([sc.Plane(a.copy()) for a in arr])


def stack(img):
    return np.stack([p.numpy() for p in img.planes])


CASES = ["syn_12x13_s3_sharpen", "syn_16x16_s5_gauss5", "syn_37x23_s8_normal", "syn_24x64_s21_gauss5",
         "syn_129x131_s20_sharpen", "special_20x28_sigma1"]


@pytest.mark.parametrize("name", CASES)
def test_conv_two_pass_plane_api(sc, name):
    g = load_golden(name)
    k = sc.SeparableKernel(g["taps"])
    for ext, tag in ((False, "faithful"), (True, "ext")):
        for p in range(g["input"].shape[0]):
            plane = sc.Plane(g["input"][p].copy())
            scratch = sc.Plane.full(*g["input"].shape[1:], SENTINEL)
            sc.conv_two_pass(plane, k, scratch, extended=ext)
            assert np.array_equal(plane.data, g[f"two_pass_{tag}_image"][p])
            assert np.array_equal(scratch.data, g[f"two_pass_{tag}_scratch"][p])


@pytest.mark.parametrize("name", CASES)
def test_passes_single_copyback_plane_api(sc, name):
    g = load_golden(name)
    k = sc.SeparableKernel(g["taps"])
    dense = sc.outer_product(k)
    R, C = g["input"].shape[1:]
    for p in range(g["input"].shape[0]):
        src = sc.Plane(g["input"][p].copy())
        for fn, key in ((sc.horizontal_pass, "horizontal_sentinel"), (sc.vertical_pass, "vertical_sentinel")):
            d = sc.Plane.full(R, C, SENTINEL)
            fn(src, k, d)
            assert np.array_equal(d.data, g[key][p])
        for fn in (sc.conv_single_pass_generic, sc.conv_single_pass_unrolled5):
            d = sc.Plane.full(R, C, SENTINEL)
            fn(src, dense, d)
            assert np.array_equal(d.data, g["single_sentinel"][p])
        a = sc.Plane(g["input"][p].copy())
        b = sc.Plane.zeros(R, C)
        sc.conv_single_pass_unrolled5(a, dense, b)
        sc.copy_back(b, a, sc.valid_region(R, C, 2))
        assert np.array_equal(a.data, g["convolve_single_copy_image"][p])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("where", ["host-fused", "host-split", "device"])
def test_convolve_image_two_pass(sc, name, where):
    g = load_golden(name)
    k = sc.SeparableKernel(g["taps"])
    variant = sc.ConvVariant(sc.Algorithm.TWO_PASS)
    if where == "device":
        img = sc.Image.from_tensor(torch.from_numpy(g["input"].copy()).cuda())
        ws = sc.Image.zeros_like(img)
        stats = sc.convolve_image(img, k, variant, sc.Cuda(), workspace=ws)
        assert np.array_equal(stack(ws), g["two_pass_faithful_scratch"])
    else:
        # with a workspace given, both host paths leave the reference's end state
        # in BOTH buffers: H0 in the workspace (S/executors.py:312-323)
        img = host_image(sc, g["input"])
        ws = sc.Image([sc.Plane(np.full(g["input"].shape[1:], SENTINEL, np.float32))
                       for _ in range(g["input"].shape[0])])
        stats = sc.convolve_image(img, k, variant, sc.Cuda(fused=(where == "host-fused")), workspace=ws)
        assert np.array_equal(stack(ws), g["two_pass_faithful_scratch"])
    out = sc.result_image(img, ws, variant)
    assert out is img
    assert np.array_equal(stack(out), g["two_pass_faithful_image"])
    assert stats.parallel_region_launches >= 1 and stats.wall_time_ns > 0


@pytest.mark.parametrize("name", CASES)
def test_convolve_image_two_pass_device_no_workspace(sc, name):
    """Device image, no workspace: the in-place pass without scratch writes."""
    g = load_golden(name)
    img = sc.Image.from_tensor(torch.from_numpy(g["input"].copy()).cuda())
    stats = sc.convolve_image(img, sc.SeparableKernel(g["taps"]), sc.ConvVariant(sc.Algorithm.TWO_PASS), sc.Cuda())
    assert np.array_equal(stack(img), g["two_pass_faithful_image"])
    assert stats.parallel_region_launches >= 1


@pytest.mark.parametrize("name", CASES)
def test_convolve_image_two_pass_host_no_workspace(sc, name):
    """No workspace: the reference allocates an internal zero one the caller never
    sees (S/executors.py:303-304), so the streamed fused path runs (image only)."""
    g = load_golden(name)
    img = host_image(sc, g["input"])
    sc.convolve_image(img, sc.SeparableKernel(g["taps"]), sc.ConvVariant(sc.Algorithm.TWO_PASS), sc.Cuda())
    assert np.array_equal(stack(img), g["two_pass_faithful_image"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("copy", [False, True])
@pytest.mark.parametrize("on_device", [False, True])
def test_convolve_image_single_pass(sc, name, copy, on_device):
    g = load_golden(name)
    k = sc.SeparableKernel(g["taps"])
    variant = sc.ConvVariant(sc.Algorithm.SINGLE_PASS_UNROLLED5, copy_back=copy)
    if on_device:
        img = sc.Image.from_tensor(torch.from_numpy(g["input"].copy()).cuda())
    else:
        img = host_image(sc, g["input"])
    ws = sc.Image.zeros_like(img)
    sc.convolve_image(img, k, variant, sc.Cuda(), workspace=ws)
    assert np.array_equal(stack(ws), g["single_zero"])
    want_img = g["convolve_single_copy_image"] if copy else g["input"]
    assert np.array_equal(stack(img), want_img)
    assert sc.result_image(img, ws, variant) is (img if copy else ws)


def test_device_planes_of_separate_allocations(sc):
    """Planes that are not views of one tensor still work (one launch per plane)."""
    g = load_golden("syn_24x64_s21_sharpen")
    img = sc.Image([sc.Plane(torch.from_numpy(p.copy()).cuda()) for p in g["input"]])
    ws = sc.Image([sc.Plane(torch.zeros(p.shape, device="cuda")) for p in g["input"]])
    sc.convolve_image(img, sc.SeparableKernel(g["taps"]), sc.ConvVariant(sc.Algorithm.TWO_PASS), sc.Cuda(),
                      workspace=ws)
    assert np.array_equal(stack(img), g["two_pass_faithful_image"])


# ---- ports of the reference's own conv tests (T/test_conv.py), through this package

def test_golden_center_value(sc):
    # T/test_conv.py:55-61
    src = sc.make_synthetic(7, 7, 1, seed=42).planes[0]
    dense = sc.outer_product(sc.gaussian5())
    for op in (sc.conv_single_pass_generic, sc.conv_single_pass_unrolled5):
        dst = sc.Plane.zeros(7, 7)
        op(src, dense, dst)
        assert dst.data[3, 3] == np.float32(113.06233978271484)


def test_horizontal_and_vertical_hand_dot_product(sc):
    # T/test_conv.py:113-139
    row = np.array([3, 1, 4, 1, 5, 9, 2], dtype=np.float32)
    src = sc.Plane(np.tile(row, (7, 1)))
    dst = sc.Plane.zeros(7, 7)
    sc.horizontal_pass(src, sc.gaussian5(), dst)
    assert dst.data[3, 2] == np.float32(2.5)
    src = sc.Plane(np.tile(row[:, None], (1, 7)))
    dst = sc.Plane.zeros(7, 7)
    sc.vertical_pass(src, sc.gaussian5(), dst)
    assert dst.data[2, 3] == np.float32(2.5)


def test_delta_identity_and_transpose_symmetry(sc):
    # T/test_conv.py:90-101, :152-161
    src = sc.make_synthetic(10, 10, 1, seed=4).planes[0]
    region = sc.valid_region(10, 10, 2)
    for op in (sc.horizontal_pass, sc.vertical_pass):
        dst = sc.Plane.zeros(10, 10)
        op(src, sc.delta(5), dst)
        assert sc.max_abs_diff(src, dst, region) == 0.0
    src = sc.make_synthetic(9, 12, 1, seed=8).planes[0]
    v = sc.Plane.zeros(9, 12)
    sc.vertical_pass(src, sc.gaussian5(), v)
    h = sc.Plane.zeros(12, 9)
    sc.horizontal_pass(sc.Plane(np.ascontiguousarray(src.data.T)), sc.gaussian5(), h)
    r = sc.valid_region(9, 12, 2)
    assert np.array_equal(v.data[r.row_lo:r.row_hi, r.col_lo:r.col_hi], h.data.T[r.row_lo:r.row_hi, r.col_lo:r.col_hi])


def test_two_pass_vs_single_pass_tolerance_and_counts(sc):
    # T/test_conv.py:182-191 (doubly interior, 1e-4 rel / 1e-5 abs) and :325-357 (op counts)
    plane = sc.make_synthetic(12, 12, 1, seed=7).planes[0]
    ref = sc.Plane.zeros(12, 12)
    sc.conv_single_pass_generic(plane, sc.outer_product(sc.gaussian5()), ref)
    counter = sc.OpCounter()
    sc.conv_two_pass(plane, sc.gaussian5(), sc.Plane.zeros(12, 12), counter=counter)
    d = sc.doubly_interior_region(12, 12, 2)
    got = plane.data[d.row_lo:d.row_hi, d.col_lo:d.col_hi]
    want = ref.data[d.row_lo:d.row_hi, d.col_lo:d.col_hi]
    assert np.allclose(got, want, rtol=1e-4, atol=1e-5)
    law = sc.arith_count(sc.ConvVariant(sc.Algorithm.TWO_PASS), 12, 12, 5)
    assert (counter.multiplications, counter.additions) == (law.multiplications, law.additions)


def test_reference_errors(sc):
    # T/test_conv.py:301-322
    src = sc.make_synthetic(8, 8, 1, seed=1).planes[0]
    dense = sc.outer_product(sc.gaussian5())
    with pytest.raises(sc.InvalidArgumentError):
        sc.conv_single_pass_generic(src, dense, src)
    with pytest.raises(sc.InvalidArgumentError):
        sc.horizontal_pass(src, sc.gaussian5(), sc.Plane(src.data[:, :]))
    with pytest.raises(sc.InvalidArgumentError):
        sc.conv_single_pass_generic(src, dense, sc.Plane.zeros(8, 9))
    with pytest.raises(sc.UnsupportedWidthError):
        sc.conv_single_pass_unrolled5(src, sc.outer_product(sc.delta(3)), sc.Plane.zeros(8, 8))
    dsrc = sc.Plane(torch.zeros((8, 8), device="cuda"))
    with pytest.raises(sc.InvalidArgumentError):
        sc.conv_two_pass(dsrc, sc.gaussian5(), sc.Plane(dsrc.data[:, :]))


def test_convolve_image_multi_device_plan(sc):
    """convolve_image with Cuda(devices=[...]) on a host image (the reference's
    single-process plan model, several GPUs): same bits as Cuda()."""
    rng = np.random.default_rng(12)
    data = rng.random((3, 300, 517), dtype=np.float32)
    k = sc.SeparableKernel(np.array([1, 4, 6, 4, 1], np.float32) / 16)
    variant = sc.ConvVariant(sc.Algorithm.TWO_PASS)
    a = sc.Image([sc.Plane(p.copy()) for p in data])
    b = sc.Image([sc.Plane(p.copy()) for p in data])
    sc.convolve_image(a, k, variant, sc.Cuda())
    sc.convolve_image(b, k, variant, sc.Cuda(devices=[0, 0, 0, 0]))
    for pa, pb in zip(a.planes, b.planes):
        assert np.array_equal(pa.data.view(np.uint32), pb.data.view(np.uint32))
