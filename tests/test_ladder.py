"""GPU ladder stages: CSV schema and record logic on CPU,
check-then-time runs on the B200."""

import io

import pytest

from paper_1711_09791_b200 import ladder
from paper_1711_09791_b200.conv import Algorithm, ConvVariant
from paper_1711_09791_b200.errors import ConfigError, InvalidArgumentError
from paper_1711_09791_b200.executors import Cuda


def _rec(label, rows, cols, ns, alg=Algorithm.TWO_PASS, copy=False):
    return ladder.BenchRecord(label=label, variant=ConvVariant(alg, copy), plan=Cuda(), rows=rows, cols=cols,
                              planes=3, reps=10, total_ns=ns * 10, per_image_ns=ns)


def test_header_is_reference_schema():
    assert ladder.CSV_HEADER.split(",") == [
        "label", "algorithm", "copy_back", "plan", "workers", "cutoff", "agglomerate", "rows", "cols", "planes",
        "reps", "total_ns", "per_image_ns", "speedup", "build_vectorized"]


def test_csv_order_and_cells():
    recs = [_rec("GPU-single", 64, 64, 50, Algorithm.SINGLE_PASS_UNROLLED5, False),
            _rec("GPU-fused", 128, 128, 40), _rec("GPU-fused", 64, 64, 20),
            _rec("GPU-single-copy", 64, 64, 60, Algorithm.SINGLE_PASS_UNROLLED5, True)]
    recs = ladder.speedup_table(recs, "GPU-fused")
    buf = io.StringIO()
    ladder.emit_csv(recs, buf, sms=148)
    lines = buf.getvalue().splitlines()
    assert lines[0] == ladder.CSV_HEADER
    assert [ln.split(",")[0] for ln in lines[1:]] == ["GPU-fused", "GPU-fused", "GPU-single", "GPU-single-copy"]
    first = lines[1].split(",")
    assert first == ["GPU-fused", "two-pass", "false", "cuda", "148", "", "", "64", "64", "3", "10", "200", "20",
                     "1.0000", "true"]
    assert lines[3].split(",")[13] == "0.4000"
    assert lines[4].split(",")[2] == "true"
    # byte-identical output for identical records
    buf2 = io.StringIO()
    ladder.emit_csv(list(reversed(recs)), buf2, sms=148)
    assert buf2.getvalue() == buf.getvalue()


def test_speedup_external_baseline_and_missing():
    recs = [_rec("GPU-fused", 64, 64, 20)]
    out = ladder.speedup_table(recs, "Opt-0", baseline_ns={(64, 64, 3): 2000})
    assert out[0].speedup == pytest.approx(100.0)
    with pytest.raises(ConfigError):
        ladder.speedup_table(recs, "Opt-0")
    bad = ladder.BenchRecord(**{**recs[0].__dict__, "speedup": -1.0})
    with pytest.raises(InvalidArgumentError):
        ladder.record_row(bad)


def test_config_validation():
    with pytest.raises(ConfigError):
        ladder.GpuLadderConfig(sizes=())
    with pytest.raises(ConfigError):
        ladder.GpuLadderConfig(sizes=((8, 8),), reps=0)
    with pytest.raises(ConfigError):
        ladder.GpuLadderConfig(sizes=((8, 8),), stages=("Opt-9",))


def test_csv_to_path(tmp_path):
    p = tmp_path / "ladder.csv"
    ladder.emit_csv([_rec("GPU-e2e", 8, 8, 5)], p)
    assert p.read_text().startswith(ladder.CSV_HEADER + "\nGPU-e2e,two-pass,false,cuda,,")


@pytest.mark.gpu
def test_gpu_ladder_runs_every_stage():
    from paper_1711_09791_b200.kernels import SeparableKernel

    cfg = ladder.GpuLadderConfig(sizes=((96, 130), (33, 17)), reps=3)
    res = ladder.run_gpu_ladder(cfg)
    assert not res.failures, res.failures
    assert {r.label for r in res.records} == {s[0] for s in ladder.GPU_STAGES}
    assert len(res.records) == 2 * len(ladder.GPU_STAGES)
    assert all(r.per_image_ns > 0 and r.planes == 3 for r in res.records)
    recs = ladder.speedup_table(res.records, "GPU-e2e")
    buf = io.StringIO()
    ladder.emit_csv(recs, buf)
    assert len(buf.getvalue().splitlines()) == 1 + len(recs)
    # width 3: single-pass stages report the generic algorithm
    res3 = ladder.run_gpu_ladder(ladder.GpuLadderConfig(sizes=((40, 40),), reps=2, stages=("GPU-single",)),
                                 SeparableKernel([0.25, 0.5, 0.25]))
    assert not res3.failures and res3.records[0].variant.algorithm is Algorithm.SINGLE_PASS_GENERIC


@pytest.mark.gpu
def test_gpu_ladder_check_catches_a_wrong_stage(monkeypatch):
    import torch

    real = ladder._run_once

    def broken(how, x, w, dense, copy_back, out, scratch, host):
        real(how, x, w, dense, copy_back, out, scratch, host)
        if how == "fused":
            out.add_(1e-2)

    monkeypatch.setattr(ladder, "_run_once", broken)
    res = ladder.run_gpu_ladder(ladder.GpuLadderConfig(sizes=((32, 32),), reps=1, stages=("GPU-fused",)))
    assert res.records == [] and len(res.failures) == 1
    assert "tolerance" in res.failures[0].detail
    torch.cuda.synchronize()


def test_parse_sizes():
    assert ladder._parse_sizes("8x9,1152X1152") == ((8, 9), (1152, 1152))
    with pytest.raises(ConfigError):
        ladder._parse_sizes("8by9")


@pytest.mark.gpu
def test_gpu_ladder_cli(tmp_path):
    p = tmp_path / "l.csv"
    assert ladder.main(["--sizes", "64x64", "--reps", "2", "--csv", str(p)]) == 0
    lines = p.read_text().splitlines()
    assert lines[0] == ladder.CSV_HEADER and len(lines) == 1 + len(ladder.GPU_STAGES)


@pytest.mark.parametrize("name", ["syn_37x23_s8_normal", "syn_24x64_s21_sharpen", "special_20x28_sigma1"])
def test_check_reference_is_cpu_dense_pinned_to_fixtures(name):
    """The ladder's check-before-timing reference is computed on the CPU (not by
    the GPU it checks) and equals the reference's own dense single pass bit for bit
    (fixtures made by sepconv_lab, tests/golden/make_golden.py)."""
    import numpy as np

    from conftest import load_golden
    from paper_1711_09791_b200.kernels import SeparableKernel

    g = load_golden(name)
    got = ladder._dense_reference(g["input"], SeparableKernel(g["taps"]))
    assert isinstance(got, np.ndarray)
    assert np.array_equal(got.view(np.uint32), g["single_zero"].view(np.uint32))
