"""The B200 path behind the REAL reference: sepconv_lab (baseline/_ref) with the
plugin installed, its own objects (numpy Planes / Images, SeparableKernel,
ConvVariant) and entry points, checked against its own CPU plans bit for bit --
both buffers included. Restates the reference's own test cases
(T/test_conv.py, T/test_executors.py:188-231) with the Cuda plan / GPU plane ops
added, and drives its CLI, HTTP service and ladder harness with plan "cuda".
"""

from __future__ import annotations

import base64
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REF_INSTALL, ROOT

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture
def sl(plugged):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return plugged


def stack(img):
    return np.stack([p.data for p in img.planes])


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


VARIANTS = [("generic-copy", "single-generic", True), ("generic-nocopy", "single-generic", False),
            ("unrolled-copy", "single-unrolled", True), ("unrolled-nocopy", "single-unrolled", False),
            ("two-pass", "two-pass", False)]


@pytest.mark.parametrize("vid,algo,copy", VARIANTS, ids=[v[0] for v in VARIANTS])
@pytest.mark.parametrize("rows,cols", [(64, 64), (37, 101)])
def test_scheduling_transparency_with_cuda_plan(sl, vid, algo, copy, rows, cols):
    """T/test_executors.py:188-221 with the Cuda plans added: every plan leaves the
    same bits in BOTH buffers (result image and workspace)."""
    variant = sl.ConvVariant(sl.Algorithm(algo), copy_back=copy)
    image = sl.make_synthetic(rows, cols, 3, seed=42)
    plans = [sl.Sequential(), sl.StaticChunked(workers=4), sl.TaskPool(workers=4, cutoff=3, agglomerate=True),
             sl.make_plan("cuda"), sl.Cuda(fused=False)]
    ends = []
    for plan in plans:
        work = image.copy()
        ws = sl.Image.zeros_like(work)
        stats = sl.convolve_image(work, sl.gaussian5(), variant, plan, workspace=ws)
        assert isinstance(stats, sl.LaunchStats)
        res = sl.result_image(work, ws, variant)
        ends.append((stack(work), stack(ws), stack(res)))
    for e in ends[1:]:
        for a, b in zip(e, ends[0]):
            assert bits_equal(a, b)


@pytest.mark.parametrize("taps", [[1, 4, 6, 4, 1], [-1, -2, 7, -2, -1], [0.2, -0.7, 1.3, 0.05, 0.15],
                                  [1, 2, 3, 4, 5, 4, 3, 2, 1], [0.5, 0.25, 0.25]])
def test_two_pass_workspace_end_state_matches_sequential(sl, taps):
    """A workspace given to convolve_image(TWO_PASS) ends holding H0 under the Cuda
    plan exactly as under Sequential (S/executors.py:312-323), on a pageable image
    big enough to stream through several chunks."""
    k = sl.SeparableKernel(taps)
    image = sl.make_synthetic(311, 517, 3, seed=9)
    a, b = image.copy(), image.copy()
    wa = sl.Image([sl.Plane(np.full((311, 517), -5.0, np.float32)) for _ in range(3)])
    wb = sl.Image([sl.Plane(np.full((311, 517), 7.0, np.float32)) for _ in range(3)])
    v = sl.ConvVariant(sl.Algorithm.TWO_PASS)
    sl.convolve_image(a, k, v, sl.Sequential(), workspace=wa)
    sl.convolve_image(b, k, v, sl.make_plan("cuda"), workspace=wb)
    assert bits_equal(stack(b), stack(a))
    assert bits_equal(stack(wb), stack(wa))
    c = image.copy()
    sl.convolve_image(c, k, v, sl.make_plan("cuda"))  # no workspace: the fused path
    assert bits_equal(stack(c), stack(a))


def test_plane_ops_golden_and_hand_values(sl):
    """T/test_conv.py:34, 55-61, 113-139 through the GPU plane ops on the
    reference's own Plane objects."""
    from paper_1711_09791_b200 import plugin

    ops = plugin.gpu_ops(sl)
    dense = sl.outer_product(sl.gaussian5())
    src = sl.make_synthetic(7, 7, 1, seed=42).planes[0]
    for name in ("conv_single_pass_generic", "conv_single_pass_unrolled5"):
        dst = sl.Plane.zeros(7, 7)
        ops[name](src, dense, dst)
        assert dst.data[3, 3] == np.float32(113.06233978271484)
    row = np.array([3, 1, 4, 1, 5, 9, 2], dtype=np.float32)
    dst = sl.Plane.zeros(7, 7)
    ops["horizontal_pass"](sl.Plane(np.tile(row, (7, 1))), sl.gaussian5(), dst)
    assert dst.data[3, 2] == np.float32(2.5)
    dst = sl.Plane.zeros(7, 7)
    ops["vertical_pass"](sl.Plane(np.tile(row[:, None], (1, 7))), sl.gaussian5(), dst)
    assert dst.data[2, 3] == np.float32(2.5)


@pytest.mark.parametrize("extended", [False, True])
@pytest.mark.parametrize("taps", [[1, 4, 6, 4, 1], [-1, -2, 7, -2, -1], [1, 1, 1], list(range(1, 12))])
def test_plane_ops_match_reference_ops(sl, taps, extended):
    """Every whole-plane op (S/conv.py:324-440) on GPU vs the reference's own CPU op,
    both buffers (scratch end state of conv_two_pass; dst ring untouched)."""
    from paper_1711_09791_b200 import plugin

    ops = plugin.gpu_ops(sl)
    k = sl.SeparableKernel([float(t) for t in taps])
    dense = sl.outer_product(k)
    src = sl.make_synthetic(41, 53, 1, seed=len(taps)).planes[0]
    p1, p2 = src.copy(), src.copy()
    s1, s2 = sl.Plane.full(41, 53, -1.0), sl.Plane.full(41, 53, -1.0)
    sl.conv_two_pass(p1, k, s1, extended=extended)
    ops["conv_two_pass"](p2, k, s2, extended=extended)
    assert bits_equal(p2.data, p1.data) and bits_equal(s2.data, s1.data)
    for name in ("horizontal_pass", "vertical_pass"):
        d1, d2 = sl.Plane.full(41, 53, 3.0), sl.Plane.full(41, 53, 3.0)
        getattr(sl, name)(src, k, d1)
        ops[name](src, k, d2)
        assert bits_equal(d2.data, d1.data), name
    d1, d2 = sl.Plane.full(41, 53, 3.0), sl.Plane.full(41, 53, 3.0)
    sl.conv_single_pass_generic(src, dense, d1)
    ops["conv_single_pass_generic"](src, dense, d2)
    assert bits_equal(d2.data, d1.data)
    r = k.radius
    region = sl.valid_region(41, 53, r)
    a, b = src.copy(), src.copy()
    sl.copy_back(d1, a, region)
    ops["copy_back"](d1, b, region)
    assert bits_equal(b.data, a.data)


def test_reference_exceptions_from_gpu_path(sl):
    """T/test_conv.py:301-322: the GPU path raises the reference's own classes."""
    from paper_1711_09791_b200 import plugin

    ops = plugin.gpu_ops(sl)
    src = sl.make_synthetic(8, 8, 1, seed=1).planes[0]
    dense = sl.outer_product(sl.gaussian5())
    with pytest.raises(sl.InvalidArgumentError):
        ops["conv_single_pass_generic"](src, dense, src)
    with pytest.raises(sl.InvalidArgumentError):
        ops["conv_single_pass_generic"](src, dense, sl.Plane.zeros(8, 9))
    with pytest.raises(sl.InvalidDimensionError):
        ops["horizontal_pass"](sl.Plane.zeros(4, 9), sl.gaussian5(), sl.Plane.zeros(4, 9))
    with pytest.raises(sl.UnsupportedWidthError):
        ops["conv_single_pass_unrolled5"](src, sl.outer_product(sl.delta(3)), sl.Plane.zeros(8, 8))
    image = sl.make_synthetic(16, 16, 3, seed=2)
    with pytest.raises(sl.InvalidArgumentError):
        sl.convolve_image(image, sl.gaussian5(), sl.ConvVariant(sl.Algorithm.TWO_PASS), sl.make_plan("cuda"),
                          workspace=sl.Image.zeros(16, 17, 3))
    with pytest.raises(sl.InvalidDimensionError):
        sl.convolve_image(sl.make_synthetic(5, 5, 3, seed=2), sl.SeparableKernel([1.0] * 7),
                          sl.ConvVariant(sl.Algorithm.TWO_PASS), sl.make_plan("cuda"))


def _run(args, cwd):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF_INSTALL]), PYTHONDONTWRITEBYTECODE="1")
    return subprocess.run([sys.executable, *args], capture_output=True, text=True, env=env, cwd=cwd, timeout=600)


@pytest.mark.parametrize("algo", ["two-pass", "single-unrolled"])
def test_cli_convolve_plan_cuda_bytes_identical(sl, tmp_path, algo):
    """`sepconv convolve --plan cuda` (S/cli.py:206-224) writes the same PPM bytes as
    `--plan sequential`."""
    r = _run(["-m", "sepconv_lab.cli", "gen", "--sizes", "96x130", "--seed", "5", "--out", "in.ppm"], tmp_path)
    assert r.returncode == 0, r.stderr
    outs = {}
    for plan in ("sequential", "cuda"):
        mod = "paper_1711_09791_b200.plugin" if plan == "cuda" else "sepconv_lab.cli"
        r = _run(["-m", mod, "convolve", "--plan", plan, "--algorithm", algo, "--in", "in.ppm",
                  "--out", f"{plan}.ppm"], tmp_path)
        assert r.returncode == 0, r.stdout + r.stderr
        assert f"[{algo}, {plan}]" in r.stdout
        outs[plan] = (tmp_path / f"{plan}.ppm").read_bytes()
    assert outs["cuda"] == outs["sequential"]
    r = _run(["-m", "sepconv_lab.cli", "convolve", "--plan", "cuda", "--in", "in.ppm"], tmp_path)
    assert r.returncode == 1  # without the plugin the reference rejects the mode (usage error, exit 1)


def test_service_convolve_plan_cuda(sl):
    """POST /convolve with {"plan": {"mode": "cuda"}} (S/service.py:98-122) returns the
    image the sequential plan returns."""
    from fastapi.testclient import TestClient

    client = TestClient(sl.service.app)
    got = {}
    for mode in ("sequential", "cuda"):
        for algo in ("two-pass", "single-generic"):
            body = {"image": {"synthetic": {"rows": 48, "cols": 70, "planes": 3, "seed": 4}},
                    "kernel": {"weights": [-1, -2, 7, -2, -1]}, "algorithm": algo,
                    "plan": {"mode": mode}, "return_image": True}
            r = client.post("/convolve", json=body)
            assert r.status_code == 200, r.text
            got[(mode, algo)] = base64.b64decode(r.json()["result_ppm_base64"])
    for algo in ("two-pass", "single-generic"):
        assert got[("cuda", algo)] == got[("sequential", algo)]
    bad = {"image": {"synthetic": {"rows": 48, "cols": 70}}, "kernel": {"weights": [1, 1, 1, 1]},
           "plan": {"mode": "cuda"}}
    assert client.post("/convolve", json=bad).status_code in (400, 422)


def test_ladder_gpu_stages_through_reference_harness(sl, tmp_path):
    """GPU stages in the reference's ladder (S/bench.py:226-259): checked by its own
    check_stage_output (CPU dense oracle) before timing, timed by time_variant,
    written by emit_csv with plan "cuda"."""
    cfg = sl.LadderConfig(sizes=((64, 64), (96, 80)), planes=3, seed=42, reps=3, workers=2, cutoff=4,
                          stages=("Opt-0", "Opt-2", "Gpu-0", "Gpu-1", "Gpu-1-nocopy", "Gpu-2"))
    res = sl.run_ladder(cfg)
    assert not res.failures, res.failures
    labels = sorted({r.label for r in res.records})
    assert labels == ["Gpu-0", "Gpu-1", "Gpu-1-nocopy", "Gpu-2", "Opt-0", "Opt-2"]
    assert all(r.speedup is not None for r in res.records)
    path = tmp_path / "ladder.csv"
    sl.emit_csv(res.records, str(path))
    rows = [ln.split(",") for ln in path.read_text().splitlines()[1:]]
    assert {r[3] for r in rows if r[0].startswith("Gpu")} == {"cuda"}
    assert [r[0] for r in rows][:4] == ["Opt-0", "Opt-0", "Opt-2", "Opt-2"]


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow,
                                                                 HealthCheck.function_scoped_fixture])
@given(rows=st.integers(5, 70), cols=st.integers(5, 90), planes=st.integers(1, 3), seed=st.integers(0, 2**20),
       algo=st.sampled_from(["two-pass", "single-generic", "single-unrolled"]), copy=st.booleans(),
       with_ws=st.booleans(), width=st.sampled_from([1, 3, 5, 7, 9, 11]), fused=st.booleans())
def test_random_cuda_plan_equals_sequential(sl, rows, cols, planes, seed, algo, copy, with_ws, width, fused):
    """Random images, taps and variants through the reference's own convolve_image:
    the Cuda plan leaves the same bits as Sequential in the image AND the workspace
    (T/test_executors.py:188-221, randomised like T/conftest.py:13-19)."""
    if rows < width or cols < width or (algo == "single-unrolled" and width != 5):
        return
    rng = np.random.default_rng(seed)
    k = sl.SeparableKernel(rng.uniform(-2, 2, size=width).astype(np.float32))
    variant = sl.ConvVariant(sl.Algorithm(algo), copy_back=copy)
    data = rng.uniform(-50, 300, size=(planes, rows, cols)).astype(np.float32)
    ends = []
    for plan in (sl.Sequential(), sl.Cuda(fused=fused)):
        img = sl.Image([sl.Plane(data[p].copy()) for p in range(planes)])
        ws = sl.Image([sl.Plane(np.full((rows, cols), -7.0, np.float32)) for _ in range(planes)]) if with_ws else None
        sl.convolve_image(img, k, variant, plan, workspace=ws)
        ends.append((stack(img), stack(ws) if ws is not None else None))
    assert bits_equal(ends[1][0], ends[0][0])
    if with_ws:
        assert bits_equal(ends[1][1], ends[0][1])


def test_cli_ladder_with_gpu_stages(sl, tmp_path):
    """`sepconv ladder --stages Opt-2,Gpu-2,...` (S/cli.py:229-256) through the plugin's
    entry point: the reference's harness checks and times the GPU stages and writes
    them in its CSV with plan "cuda"."""
    r = _run(["-m", "paper_1711_09791_b200.plugin", "ladder", "--sizes", "48x64,64x64", "--reps", "2",
              "--workers", "2", "--cutoff", "3", "--stages", "Opt-0,Opt-2,Gpu-0,Gpu-1-nocopy,Gpu-2",
              "--csv", "out.csv"], tmp_path)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [ln.split(",") for ln in (tmp_path / "out.csv").read_text().splitlines()[1:]]
    gpu = [row for row in rows if row[0].startswith("Gpu")]
    assert len(gpu) == 6 and {row[3] for row in gpu} == {"cuda"}
    assert all(row[13] for row in rows)  # speedups against Opt-0 filled in
