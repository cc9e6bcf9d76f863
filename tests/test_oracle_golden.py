"""Pin the CPU oracle to the reference: golden fixtures made by the reference
itself (tests/golden/make_golden.py) and the reference tests' own constants.
CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden_cases, load_golden

SENTINEL = np.float32(-777.0)

# T/test_conv.py:34 -- seed-42 7x7 plane, gaussian5 outer product, value at (3, 3)
GOLDEN_7X7_CENTER = np.float32(113.06233978271484)
# T/test_image.py:25-26
SEED42_FIRST_DRAW = 0xBDD732262FEB6E95
SEED42_FIRST_SAMPLE = 189.84060668945312


@pytest.mark.parametrize("name", golden_cases())
def test_two_pass_matches_reference(oracle, name):
    g = load_golden(name)
    for ext, tag in ((False, "faithful"), (True, "ext")):
        out = oracle.two_pass(g["input"], g["taps"], extended=ext)
        assert np.array_equal(out, g[f"two_pass_{tag}_image"], equal_nan=True), tag
        scr = oracle.two_pass_scratch(g["input"], g["taps"], extended=ext)
        assert np.array_equal(scr, g[f"two_pass_{tag}_scratch"]), tag


@pytest.mark.parametrize("name", golden_cases())
def test_single_pass_and_passes_match_reference(oracle, name):
    g = load_golden(name)
    dense = oracle.outer_product(g["taps"])
    assert np.array_equal(dense, g["dense"])
    assert np.array_equal(oracle.single_pass(g["input"], dense), g["single_zero"])
    sent = np.full_like(g["input"], SENTINEL)
    assert np.array_equal(oracle.single_pass(g["input"], dense, sent), g["single_sentinel"])
    P, R, C = g["input"].shape
    r = len(g["taps"]) // 2
    for pname, fn in (("horizontal", oracle.horizontal_rows), ("vertical", oracle.vertical_rows)):
        d = np.full_like(g["input"], SENTINEL)
        for p in range(P):
            fn(g["input"][p], d[p], g["taps"], r, R - r)
        assert np.array_equal(d, g[f"{pname}_sentinel"]), pname
    if "convolve_single_copy_image" in g:
        img = g["input"].copy()
        single = oracle.single_pass(g["input"], dense)
        for p in range(P):
            oracle.lib().orc_copy_region(
                oracle._p(single[p]), oracle._p(img[p]), R, C, r, R - r, r, C - r
            )
        assert np.array_equal(img, g["convolve_single_copy_image"])


@pytest.mark.parametrize("name", golden_cases())
def test_numpy_port_matches_reference(oracle, name):
    """The numpy port timed as the CPU baseline computes the reference's bits."""
    g = load_golden(name)
    planes = [p.copy() for p in g["input"]]
    scratch = [np.full_like(p, SENTINEL) for p in planes]
    run = oracle.NumpyTwoPass(3)
    try:
        run(planes, scratch, g["taps"])
    finally:
        run.close()
    assert np.array_equal(np.stack(planes), g["two_pass_faithful_image"])
    assert np.array_equal(np.stack(scratch), g["two_pass_faithful_scratch"])


def test_golden_center_constant(oracle):
    g = load_golden("syn_7x7_s42_gauss5")
    out = oracle.single_pass(g["input"], oracle.outer_product(g["taps"]))
    assert out[0, 3, 3] == GOLDEN_7X7_CENTER


def test_hand_dot_product(oracle):
    # T/test_conv.py:113-139: (3*1 + 1*4 + 4*6 + 1*4 + 5*1) / 16 == 2.5
    from paper_1711_09791_b200.configs import CONFIG_TAPS

    row = np.array([3, 1, 4, 1, 5, 9, 2], dtype=np.float32)
    src = np.tile(row, (7, 1))
    dst = np.zeros_like(src)
    oracle.horizontal_rows(src, dst, CONFIG_TAPS["gauss5"], 2, 5)
    assert dst[3, 2] == np.float32(2.5)
    col = np.ascontiguousarray(src.T)
    dst = np.zeros_like(col)
    oracle.vertical_rows(col, dst, CONFIG_TAPS["gauss5"], 2, 5)
    assert dst[2, 3] == np.float32(2.5)


def test_synthetic_generator_matches_reference(oracle):
    z = load_golden("synthetic")
    assert int(oracle.splitmix64(42, 1)[0]) == SEED42_FIRST_DRAW
    assert np.array_equal(oracle.splitmix64(42, 64), z["splitmix64_s42_64"])
    assert np.array_equal(oracle.splitmix64(2**64 - 1, 64), z["splitmix64_smax_64"])
    for key in z:
        if not key.startswith("make_synthetic_"):
            continue
        dims, seed = key[len("make_synthetic_"):].split("_s")
        R, C, P = (int(v) for v in dims.split("x"))
        got = oracle.synthetic(R * C * P, int(seed), kind=0).reshape(P, R, C)
        assert np.array_equal(got, z[key]), key
    first = oracle.synthetic(1, 42, kind=0)[0]
    assert first == np.float32(SEED42_FIRST_SAMPLE)
    # counter-based offsets: a shard starting mid-stream sees the same samples
    full = oracle.synthetic(1000, 7, kind=1)
    assert np.array_equal(oracle.synthetic(300, 7, kind=1, offset=500), full[500:800])


def test_faithful_rows_differ_from_extended(oracle):
    """faithful and extended differ only on rows {2,3,R-4,R-3}."""
    g = load_golden("syn_16x16_s5_gauss5")
    a = g["two_pass_faithful_image"]
    b = g["two_pass_ext_image"]
    rows = sorted(set(np.nonzero((a != b).any(axis=(0, 2)))[0].tolist()))
    assert rows == [2, 3, 12, 13]
