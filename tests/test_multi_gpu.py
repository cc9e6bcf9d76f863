"""Multi-GPU transports on ONE GPU, without ranks that wait on one another.

* NCCL plan (csrc/nccl_band.cu): a one-rank communicator whose band names ITSELF
  as the neighbour above and below, so the packed boundary rows travel through
  ncclSend/ncclRecv and come back as the band's halo; the expected output is the
  oracle on an image whose halo rows are those boundary rows. Graph-captured and
  eager steps, repeated steps, edge bands.
* Peer signalling (kernels.cuh wait_signal): the neighbour's ready word lives in
  pinned HOST memory and a host thread publishes it late -- the kernel must wait,
  then produce the right bits; the timeout path flags the error word instead of
  hanging; the stream-ordered wait kernel (sc_band_signal_wait) likewise.
The cross-rank orchestration itself is covered over gloo on CPU
(tests/test_multi_gloo.py).
"""

from __future__ import annotations

import ctypes
import threading
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1711_09791_b200 import _lib, device, multi

    return _lib, device, multi


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def self_halo_expected(oracle, x, lo, hi, w, top, bot, extended=False):
    """Rows [lo, hi) of the two-pass of an image whose halo rows above / below the
    band are the band's own first / last r rows (what a self-exchange delivers)."""
    r = len(w) // 2
    g = x.copy()
    if top:
        g[:, lo - r:lo] = x[:, lo:lo + r]
    if bot:
        g[:, hi:hi + r] = x[:, hi - r:hi]
    return oracle.two_pass(g, w, extended=extended)[:, lo:hi]


@pytest.mark.parametrize("use_graph", [True, False])
@pytest.mark.parametrize("geom", [(3, 96, 256, 30, 70, True, True), (3, 64, 250, 0, 40, False, True),
                                  (2, 80, 128, 50, 80, True, False), (1, 40, 96, 10, 15, True, True)])
def test_nccl_plan_self_exchange(env, oracle, use_graph, geom):
    _lib, dev, multi = env
    P, R, C, lo, hi, top, bot = geom
    w = np.array([-1, -2, 7, -2, -1], np.float32)
    x = oracle.synthetic(P * R * C, lo + 3, kind=2).reshape(P, R, C)
    band = multi.Band(0, 1, R, 2, lo, hi)
    src = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])).cuda()
    dst = torch.full((P, hi - lo, C), -1.0, device="cuda")
    comm = multi.nccl_comm(None, 0)
    st = multi.NcclBandStepper(src, dst, band, w, use_graph=use_graph, comm=comm,
                               rank_above=0 if top else -1, rank_below=0 if bot else -1)
    try:
        assert st.graphed == use_graph
        want = self_halo_expected(oracle, x, lo, hi, w, top, bot)
        for it in range(3):
            dst.fill_(-1.0)
            st.step()
            torch.cuda.synchronize()
            assert bits_equal(dst.cpu().numpy(), want), it
        # fresh inputs between steps are picked up (the pack reads the current rows)
        x2 = x.copy()
        x2[:, lo:hi] = oracle.synthetic(P * (hi - lo) * C, 99, kind=2).reshape(P, hi - lo, C)
        src.copy_(torch.from_numpy(np.ascontiguousarray(x2[:, lo:hi])))
        st.step()
        torch.cuda.synchronize()
        assert bits_equal(dst.cpu().numpy(), self_halo_expected(oracle, x2, lo, hi, w, top, bot))
        # the interior-only launch used for the roofline
        ilo, ihi = st.kernel_rows
        d2 = torch.full_like(dst, -3.0)
        st.dst = d2
        args = list(st._kernel_args)
        args[1] = d2.data_ptr()
        _lib.check(_lib.load().sc_two_pass_band2_f32(*args))
        torch.cuda.synchronize()
        got = d2.cpu().numpy()
        full = oracle.two_pass(x2, w)
        assert bits_equal(got[:, ilo - lo:ihi - lo], full[:, ilo:ihi])
    finally:
        st.close()


def test_nccl_plan_rejects_bad_geometry(env):
    _lib, dev, multi = env
    from paper_1711_09791_b200.errors import InvalidArgumentError, UnsupportedWidthError

    src = torch.zeros((3, 40, 64), device="cuda")
    dst = torch.zeros_like(src)
    comm = multi.nccl_comm(None, 0)
    with pytest.raises(InvalidArgumentError):  # a middle band without a neighbour above
        multi.NcclBandStepper(src, dst, multi.Band(0, 1, 100, 2, 30, 70), np.ones(5, np.float32), comm=comm,
                              rank_above=-1, rank_below=0)
    with pytest.raises(UnsupportedWidthError):  # widths up to 31 (the lane-strided kernels)
        multi.NcclBandStepper(src, dst, multi.Band(0, 1, 100, 16, 30, 70), np.ones(33, np.float32), comm=comm)


def _host_words(n):
    t = torch.zeros(n, dtype=torch.int64).pin_memory()
    return t, t.data_ptr()  # pinned host memory is device-addressable at the same address (UVA)


def _peer_call(L, src, dst, above, lo, hi, R, C, P, w, sig_self, sig_above, epoch, err):
    r = len(w) // 2
    return L.sc_two_pass_band_peer_sig_f32(
        src.data_ptr(), dst.data_ptr(), P, R, C, (hi - lo) * C, (hi - lo) * C, C, C, lo, hi - lo,
        above.data_ptr(), lo - r, r, r * C, C, None, 0, 0, 0, 0,
        lo, lo, hi, w.ctypes.data, w.size, 0, sig_self, sig_above, None, epoch, err,
        torch.cuda.current_stream().cuda_stream)


def test_peer_signal_waits_for_late_neighbour(env, oracle):
    """The band's neighbour above publishes ready = epoch 300 ms after launch (a
    host thread writes the pinned word): the kernel waits for it, then reads the
    halo rows and produces the right bits; its own ready/done words end at epoch."""
    _lib, dev, multi = env
    L = _lib.load()
    P, R, C, lo, hi = 3, 120, 256, 40, 120
    w = np.array([1, 4, 6, 4, 1], np.float32) / np.float32(16)
    x = oracle.synthetic(P * R * C, 17, kind=1).reshape(P, R, C)
    src = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])).cuda()
    above = torch.from_numpy(np.ascontiguousarray(x[:, lo - 2:lo])).cuda()
    dst = torch.full((P, hi - lo, C), -1.0, device="cuda")
    sig_self = torch.zeros(multi.SIG_WORDS, dtype=torch.int64, device="cuda")
    nb, nb_ptr = _host_words(multi.SIG_WORDS)
    errw = torch.zeros(1, dtype=torch.int32).pin_memory()
    want = oracle.two_pass(x, w)[:, lo:hi]
    for epoch in (1, 2):
        def publish(e=epoch):
            time.sleep(0.3)
            nb[0] = e
        th = threading.Thread(target=publish)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th.start()
        _lib.check(_peer_call(L, src, dst, above, lo, hi, R, C, P, w, sig_self.data_ptr(), nb_ptr, epoch,
                              errw.data_ptr()))
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        th.join()
        assert el >= 0.25, el
        assert int(errw.item()) == 0
        assert bits_equal(dst.cpu().numpy(), want)
        s = sig_self.cpu().numpy()
        # ready, and the done count of the items that read the band above: every
        # launch adds its per-launch target (no band below here)
        assert s[0] == epoch and s[4] > 0 and s[2] == epoch * s[4] and s[3] == 0 and s[5] == 0, s


def test_peer_signal_timeout_flags_error(env, oracle, monkeypatch):
    _lib, dev, multi = env
    L = _lib.load()
    monkeypatch.setenv("SC_PEER_TIMEOUT_MS", "150")
    P, R, C, lo, hi = 1, 60, 128, 20, 60
    w = np.array([1, 4, 6, 4, 1], np.float32) / np.float32(16)
    src = torch.rand((P, hi - lo, C), device="cuda")
    above = torch.rand((P, 2, C), device="cuda")
    dst = torch.zeros_like(src)
    sig_self = torch.zeros(multi.SIG_WORDS, dtype=torch.int64, device="cuda")
    nb, nb_ptr = _host_words(multi.SIG_WORDS)  # never published
    errw = torch.zeros(1, dtype=torch.int32).pin_memory()
    t0 = time.perf_counter()
    _lib.check(_peer_call(L, src, dst, above, lo, hi, R, C, P, w, sig_self.data_ptr(), nb_ptr, 5, errw.data_ptr()))
    torch.cuda.synchronize()
    assert time.perf_counter() - t0 < 10.0
    assert int(errw.item()) == 1


def test_signal_wait_kernel(env):
    """sc_band_signal_wait: the stream waits (device side) until the neighbour's
    launch of the epoch has started (ready) and, for done, until every CTA of it
    has published done; work queued behind it runs after."""
    _lib, dev, multi = env
    L = _lib.load()
    nb, nb_ptr = _host_words(multi.SIG_WORDS)
    errw = torch.zeros(1, dtype=torch.int32).pin_memory()
    marker = torch.zeros(1, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    for word in (0, 1):
        nb.zero_()

        def publish():
            time.sleep(0.2)
            nb[5] = 3       # the neighbour above has 3 items per launch that read this band (its "below")
            nb[0] = 7       # ... and started epoch 7
            time.sleep(0.2)
            nb[3] = 20      # epochs 1..6 counted, 2 of 3 items of epoch 7
            time.sleep(0.1)
            nb[3] = 21      # its last such item finished: 7 * 3

        th = threading.Thread(target=publish)
        marker.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        th.start()
        _lib.check(L.sc_band_signal_wait(nb_ptr, None, word, 7, errw.data_ptr(), stream))
        marker.fill_(1.0)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        th.join()
        assert el >= (0.45 if word == 1 else 0.15), (word, el)
        assert marker.item() == 1.0 and int(errw.item()) == 0
    with pytest.raises(Exception):
        _lib.check(L.sc_band_signal_wait(nb_ptr, None, 2, 7, None, None))


def test_peer_stepper_world_one_unsignalled(env, oracle):
    """A world of one has no neighbours: PeerBandStepper runs the plain band kernel."""
    _lib, dev, multi = env
    P, R, C = 3, 50, 130
    w = np.array([-1, -2, 7, -2, -1], np.float32)
    x = oracle.synthetic(P * R * C, 4, kind=2).reshape(P, R, C)
    band = multi.band_plan(R, 0, 1, 2)
    src = torch.from_numpy(x).cuda()
    dst = torch.empty_like(src)
    st = multi.PeerBandStepper(src, dst, band, w)
    assert not st.signal
    st.step()
    st.check()
    torch.cuda.synchronize()
    assert bits_equal(dst.cpu().numpy(), oracle.two_pass(x, w))
    st.close()


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=40, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(P=st.integers(1, 3), R=st.integers(20, 90), C=st.integers(9, 200), width=st.sampled_from([3, 5, 7, 9, 11, 15]),
       cut=st.floats(0.1, 0.9), frac=st.floats(0.2, 0.8), top=st.booleans(), bot=st.booleans(),
       seed=st.integers(0, 2**20), extended=st.booleans())
def test_random_nccl_plan_self_exchange(env, oracle, P, R, C, width, cut, frac, top, bot, seed, extended):
    """Random bands, widths, shapes (aligned or not) and edges through the NCCL plan
    with a self-exchanging one-rank communicator: bit-exact vs the oracle on the
    image whose halo rows are the band's own boundary rows."""
    _lib, dev, multi = env
    r = width // 2
    lo = int(cut * R) if top else 0
    hi = min(R, lo + max(r, int(frac * R))) if bot else R
    if top and lo < r or bot and hi + r > R or hi - lo < r or (not top and lo != 0) or (not bot and hi != R):
        return
    if R < width or C < width:
        return
    rng = np.random.default_rng(seed)
    w = rng.uniform(-2, 2, size=width).astype(np.float32)
    x = rng.uniform(-100, 300, size=(P, R, C)).astype(np.float32)
    band = multi.Band(0, 1, R, r, lo, hi)
    src = torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])).cuda()
    dst = torch.full((P, hi - lo, C), -1.0, device="cuda")
    st_ = multi.NcclBandStepper(src, dst, band, w, extended=extended, comm=multi.nccl_comm(None, 0),
                                rank_above=0 if top else -1, rank_below=0 if bot else -1)
    try:
        st_.step()
        torch.cuda.synchronize()
        assert bits_equal(dst.cpu().numpy(), self_halo_expected(oracle, x, lo, hi, w, top, bot, extended=extended))
    finally:
        st_.close()
