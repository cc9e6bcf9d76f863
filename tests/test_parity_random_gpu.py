"""Randomised parity on the GPU (hypothesis, like the reference's property tests,
T/conftest.py:13-19): random shapes from the 5x5 minimum up, every odd width
1..9, random taps and values, all entry points and both producer paths, bit for
bit against the oracle (which is pinned to the reference)."""

from __future__ import annotations

import os

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


shapes = st.tuples(st.integers(1, 3), st.integers(5, 90), st.integers(5, 300))
_N = int(os.environ.get("SC_HYPO_SCALE", "1"))  # stress runs: multiply the example counts
widths = st.sampled_from([1, 3, 5, 7, 9])
# plus the lane-strided kernels' widths (11..31) and the first plain-kernel width
widths_any = st.sampled_from([1, 3, 5, 7, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31, 33])


@settings(max_examples=200 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(shape=shapes, width=widths_any, seed=st.integers(0, 2**32 - 1), generic=st.booleans(),
       extended=st.booleans())
def test_random_two_pass_and_passes(oracle, monkeypatch, shape, width, seed, generic, extended):
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    P, R, C = shape
    if R < width or C < width:
        return
    monkeypatch.setenv("SC_FORCE_GENERIC", "1" if generic else "0")
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    x = rng.uniform(-300, 300, size=(P, R, C)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    got = dev.two_pass(xd, w, extended=extended).cpu().numpy()
    assert bits(got, oracle.two_pass(x, w, extended=extended))
    img, scr = xd.clone(), torch.zeros_like(xd)
    dev.two_pass_split(img, scr, w, extended=extended)
    assert bits(img.cpu().numpy(), oracle.two_pass(x, w, extended=extended))
    assert bits(scr.cpu().numpy(), oracle.two_pass_scratch(x, w, extended=extended))
    r = width // 2
    for fn, ofn in ((dev.hpass, oracle.horizontal_rows), (dev.vpass, oracle.vertical_rows)):
        d = torch.full_like(xd, -5.0)
        fn(xd, w, d)
        want = np.full_like(x, -5.0)
        for p in range(P):
            ofn(x[p], want[p], w, r, R - r)
        assert bits(d.cpu().numpy(), want)


@settings(max_examples=150 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(shape=shapes, width=widths_any, seed=st.integers(0, 2**32 - 1), generic=st.booleans(), copy=st.booleans(),
       sym=st.booleans())
def test_random_single_pass(oracle, monkeypatch, shape, width, seed, generic, copy, sym):
    """sym: mirror-symmetric taps, so the dense matrix takes the product-reuse kernel."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    P, R, C = shape
    if R < width or C < width:
        return
    monkeypatch.setenv("SC_FORCE_GENERIC", "1" if generic else "0")
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    if sym:
        w = ((w + w[::-1]) / np.float32(2)).astype(np.float32)  # bitwise w[m] == w[W-1-m]
        assert np.array_equal(w.view(np.uint32), w[::-1].view(np.uint32))
    dense = oracle.outer_product(w)
    x = rng.uniform(-300, 300, size=(P, R, C)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    out = torch.zeros_like(xd)
    dev.single_pass(xd, dense, out, copy_back=copy)
    want = oracle.single_pass(x, dense)
    assert bits(out.cpu().numpy(), want)
    if copy:
        r = width // 2
        exp = x.copy()
        exp[:, r:R - r, r:C - r] = want[:, r:R - r, r:C - r]
        assert bits(xd.cpu().numpy(), exp)


@settings(max_examples=60 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(R=st.integers(5, 200), C16=st.integers(1, 40), width=widths, seed=st.integers(0, 2**32 - 1))
def test_random_ppm_fused(oracle, R, C16, width, seed):
    """u8 HWC fused path (cols % 16 == 0) == oracle two-pass + rint/clip."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    C = 16 * C16
    if R < width or C < width:
        return
    rng = np.random.default_rng(seed)
    w = rng.uniform(-1, 1.5, size=width).astype(np.float32)
    pix = rng.integers(0, 256, size=(R, C, 3), dtype=np.uint8)
    got = dev.two_pass_u8hwc(torch.from_numpy(pix).cuda(), w).cpu().numpy()
    planes = np.moveaxis(pix, -1, 0).astype(np.float32)
    conv = oracle.two_pass(np.ascontiguousarray(planes), w)
    want = np.clip(np.rint(np.moveaxis(conv, 0, -1)), 0, 255).astype(np.uint8)
    assert np.array_equal(got, want)


def test_cuda_graph_capture_replays_bit_exact():
    """The C-ABI launches are capturable (launch-bound small images run as graphs)."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    w = np.array([1, 4, 6, 4, 1], np.float32) / 16
    x = dev.synthetic((3, 96, 1152), 3, 1)
    y = torch.empty_like(x)
    want = dev.two_pass(x, w)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        dev.two_pass(x, w, y)  # warm-up outside capture (caches, work counters)
        with torch.cuda.graph(g, stream=s):
            dev.two_pass(x, w, y)
    y.zero_()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(y, want)


def test_side_stream_ordering():
    """Launches follow torch's current stream: a producer/consumer chain on a side
    stream sees its own writes."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    w = np.array([-1, -2, 7, -2, -1], np.float32)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x = dev.synthetic((3, 257, 1024), 9, 2)
        y = dev.two_pass(x, w)
        z = dev.two_pass(y, w)
    s.synchronize()
    assert torch.equal(z, dev.two_pass(dev.two_pass(x, w), w))


@pytest.mark.parametrize("off", [0, 1, 2, 3])
def test_no_out_of_bounds_writes(oracle, off):
    """compute-sanitizer is closed on this pool, so out-of-bounds writes are
    checked with canaries: every destination is a view inside a larger buffer
    filled with a sentinel bit pattern; after each op nothing outside the view
    (and nothing the op must leave untouched) may change. Offsets 1-3 make the
    rows unaligned (shifted-TMA path)."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    canary = -123.25
    w = np.array([-1, -2, 7, -2, -1], np.float32)
    for (P, R, C) in ((3, 37, 131), (2, 64, 256), (1, 5, 5)):
        x = dev.synthetic((P, R, C), 11, 2)
        n = P * R * C
        big = torch.full((n + 64,), canary, device="cuda")
        dst = big[8 + off: 8 + off + n].view(P, R, C)
        dev.two_pass(x, w, dst)
        rest = torch.cat([big[: 8 + off], big[8 + off + n:]])
        assert bool((rest == canary).all()), "fused wrote outside its destination"
        assert bits(dst.cpu().numpy(), oracle.two_pass(x.cpu().numpy(), w))
        # valid-only and single pass must also leave the ring of the view untouched
        big.fill_(canary)
        dev.two_pass(x, w, dst, ring=False)
        dev_ring = dst.clone()
        dev_ring[:, 2:R - 2, 2:C - 2] = canary
        assert bool((dev_ring == canary).all()) and bool((torch.cat([big[: 8 + off], big[8 + off + n:]]) == canary).all())
        big.fill_(canary)
        dev.single_pass(x, oracle.outer_product(w), dst)
        assert bool((torch.cat([big[: 8 + off], big[8 + off + n:]]) == canary).all())
        d2 = dst.clone()
        d2[:, 2:R - 2, 2:C - 2] = canary
        assert bool((d2 == canary).all())


@settings(max_examples=80 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(R=st.integers(10, 120), C=st.integers(5, 300), world=st.integers(2, 5), width=widths,
       seed=st.integers(0, 2**32 - 1), extended=st.booleans())
def test_random_peer_bands(R, C, world, width, seed, extended):
    """Row bands reading their halo rows from the neighbouring bands' buffers
    (multi-GPU peer path, neighbours in-process) == the whole-image two-pass."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev
    from paper_1711_09791_b200.multi import band_plan

    r = width // 2
    if R < width or C < width or R // world < max(r, 1):
        return
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    x = torch.from_numpy(rng.uniform(-100, 100, size=(2, R, C)).astype(np.float32)).cuda()
    want = dev.two_pass(x, w, extended=extended).cpu().numpy()
    bands = [band_plan(R, k, world, r) for k in range(world)]
    owned = [x[:, b.lo:b.hi].clone() for b in bands]
    for k, b in enumerate(bands):
        out = torch.full((2, b.hi - b.lo, C), float("nan"), device="cuda")
        above = dev.PeerRows.of(owned[k - 1], bands[k - 1].lo) if k > 0 else None
        below = dev.PeerRows.of(owned[k + 1], bands[k + 1].lo) if k < world - 1 else None
        dev.two_pass_band_peer(owned[k], w, out, global_rows=R, src_row0=b.lo, dst_row0=b.lo, out_lo=b.lo,
                               out_hi=b.hi, above=above, below=below, extended=extended)
        assert bits(out.cpu().numpy(), want[:, b.lo:b.hi]), (k, b)


@settings(max_examples=20 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(P=st.integers(1, 3), R=st.integers(100, 1500), C=st.integers(100, 3000), width=widths,
       seed=st.integers(0, 2**32 - 1), generic=st.booleans())
def test_random_larger_shapes(oracle, monkeypatch, P, R, C, width, seed, generic):
    """Shapes large enough for multi-strip, guided (head/tail band) plans with
    partial last strips and any width: fused two-pass and single pass."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    monkeypatch.setenv("SC_FORCE_GENERIC", "1" if generic else "0")
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    x = rng.uniform(-300, 300, size=(P, R, C)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    assert bits(dev.two_pass(xd, w).cpu().numpy(), oracle.two_pass(x, w))
    dense = oracle.outer_product(w)
    out = torch.zeros_like(xd)
    dev.single_pass(xd, dense, out)
    assert bits(out.cpu().numpy(), oracle.single_pass(x, dense))


@settings(max_examples=25 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(P=st.integers(1, 3), R=st.integers(20, 1200), C4=st.integers(2, 700), width=widths,
       seed=st.integers(0, 2**32 - 1), extended=st.booleans(), sym=st.booleans())
def test_random_in_place_one_pass_modes(oracle, P, R, C4, width, seed, extended, sym):
    """The in-place one-pass kernels on 16-B aligned rows (C % 4 == 0) with
    planner-chosen strips and head/tail bands: the split two-pass (scratch H0 +
    image V) and the single pass with copy-back (workspace + image), whose other
    items' halos come from the pre-launch snapshot. Both buffers bit-exact."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    C = 4 * C4
    if R < width or C < width:
        return
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    if sym:
        w = ((w + w[::-1]) / np.float32(2)).astype(np.float32)
    x = rng.uniform(-300, 300, size=(P, R, C)).astype(np.float32)
    img, scr = torch.from_numpy(x).cuda(), torch.full((P, R, C), 5.0, device="cuda")
    dev.two_pass_split(img, scr, w, extended=extended)
    assert bits(img.cpu().numpy(), oracle.two_pass(x, w, extended=extended))
    assert bits(scr.cpu().numpy(), oracle.two_pass_scratch(x, w, extended=extended))
    dense = oracle.outer_product(w)
    img, ws = torch.from_numpy(x).cuda(), torch.full((P, R, C), -5.0, device="cuda")
    dev.single_pass(img, dense, ws, copy_back=True)
    want = oracle.single_pass(x, dense, np.full((P, R, C), -5.0, np.float32))
    r = width // 2
    exp = x.copy()
    exp[:, r:R - r, r:C - r] = want[:, r:R - r, r:C - r]
    assert bits(ws.cpu().numpy(), want)
    assert bits(img.cpu().numpy(), exp)


@settings(max_examples=120 * _N, deadline=None, suppress_health_check=[HealthCheck.too_slow, HealthCheck.function_scoped_fixture])
@given(shape=shapes, width=st.sampled_from([1, 3, 5, 7, 9, 11, 15]), seed=st.integers(0, 2**32 - 1),
       generic=st.booleans(), extended=st.booleans(), tiny=st.booleans())
def test_random_inplace_and_host_split(oracle, monkeypatch, shape, width, seed, generic, extended, tiny):
    """Round-2 paths: the in-place two-pass (no scratch) on device planes, and the
    host split path (image + workspace end state, 16-row chunks) on pageable
    planes; tiny: values around FLT_MIN (subnormal products and sums)."""
    _need_gpu()
    from paper_1711_09791_b200 import device as dev

    P, R, C = shape
    if R < width or C < width:
        return
    monkeypatch.setenv("SC_FORCE_GENERIC", "1" if generic else "0")
    monkeypatch.setenv("SC_HOST_CHUNK_MB", "0")
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    scale = np.float32(np.finfo(np.float32).tiny) if tiny else np.float32(300)
    x = (rng.uniform(-1, 1, size=(P, R, C)) * scale).astype(np.float32)
    want = oracle.two_pass(x, w, extended=extended)
    xd = torch.from_numpy(x).cuda()
    dev.two_pass_inplace(xd, w, extended=extended)
    assert bits(xd.cpu().numpy(), want)
    planes = [p.copy() for p in x]
    scr = [np.full_like(p, 9.0) for p in x]
    dev.two_pass_host_split(planes, scr, w, extended=extended, register=False)
    assert bits(np.stack(planes), want)
    assert bits(np.stack(scr), oracle.two_pass_scratch(x, w, extended=extended))
