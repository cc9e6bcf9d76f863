"""GPU stages for the reference's optimisation-ladder harness.

The reference walks one image through every variant, checks each stage's
output against the naive dense convolution BEFORE timing it, times a reps loop
around the whole multi-plane convolution after one untimed warm-up, and emits
one CSV row per (stage, size) (S/bench.py:134-259, :288-354). This module adds
B200 stages to that ladder with the same record type, check and CSV schema, so
GPU rows sit next to the reference's CPU rows:

  GPU-fused        TWO_PASS, fused single-read/single-write kernel, device-resident
  GPU-split        TWO_PASS, row pass + column pass (the reference's scratch state)
  GPU-single       SINGLE_PASS_UNROLLED5, no copy-back
  GPU-single-copy  SINGLE_PASS_UNROLLED5 with copy-back
  GPU-e2e          TWO_PASS from HOST planes: H2D + fused + D2H inside the timed loop

Timing uses CUDA events around the reps loop (wall time for GPU-e2e, which
blocks). The correctness check mirrors check_stage_output (S/bench.py:182-224):
single-pass variants bitwise against the naive dense convolution computed on
the CPU (the reference's conv_single_pass_generic, restated with the same
numpy float32 fold; independent of the GPU), two-pass within REL_TOL/ABS_TOL on
the doubly-interior region. The same stages also run inside the reference's
own harness through the plugin (plugin.py, labels Gpu-*), checked by its own
check_stage_output.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace
from pathlib import Path
from typing import IO, Sequence

import numpy as np

from .conv import Algorithm, ConvVariant, doubly_interior_region
from .errors import ConfigError, InvalidArgumentError
from .executors import Cuda
from .image import make_synthetic, valid_region
from .kernels import SeparableKernel, gaussian5, outer_product

REL_TOL = 1e-4  # S/bench.py:41
ABS_TOL = 1e-5  # S/bench.py:42

# label -> (algorithm, copy_back, how)
GPU_STAGES: tuple[tuple[str, Algorithm, bool, str], ...] = (
    ("GPU-fused", Algorithm.TWO_PASS, False, "fused"),
    ("GPU-split", Algorithm.TWO_PASS, False, "split"),
    ("GPU-single", Algorithm.SINGLE_PASS_UNROLLED5, False, "single"),
    ("GPU-single-copy", Algorithm.SINGLE_PASS_UNROLLED5, True, "single"),
    ("GPU-e2e", Algorithm.TWO_PASS, False, "host"),
)
_STAGE_ORDER = {s[0]: i for i, s in enumerate(GPU_STAGES)}

CSV_HEADER = (  # S/bench.py:288-291, unchanged
    "label,algorithm,copy_back,plan,workers,cutoff,agglomerate,"
    "rows,cols,planes,reps,total_ns,per_image_ns,speedup,build_vectorized"
)


@dataclass
class BenchRecord:
    """One ladder measurement (the reference's BenchRecord, S/bench.py:47-61)."""

    label: str
    variant: ConvVariant
    plan: Cuda
    rows: int
    cols: int
    planes: int
    reps: int
    total_ns: int
    per_image_ns: int
    speedup: float | None = None
    build_vectorized: bool = True


@dataclass(frozen=True)
class StageFailure:
    label: str
    rows: int
    cols: int
    detail: str


@dataclass
class LadderResult:
    records: list[BenchRecord] = field(default_factory=list)
    failures: list[StageFailure] = field(default_factory=list)


@dataclass(frozen=True)
class GpuLadderConfig:
    sizes: tuple[tuple[int, int], ...]
    planes: int = 3
    seed: int = 42
    reps: int = 100
    stages: tuple[str, ...] | None = None
    device: int = 0

    def __post_init__(self):
        if not self.sizes:
            raise ConfigError("ladder needs at least one image size")
        if self.reps < 1 or self.planes < 1:
            raise ConfigError("reps and planes must be >= 1")
        unknown = [s for s in (self.stages or ()) if s not in _STAGE_ORDER]
        if unknown:
            raise ConfigError(f"unknown GPU ladder stage(s): {', '.join(unknown)}")


def _run_once(how: str, x, w, dense, copy_back: bool, out, scratch, host):
    from . import device as dev

    if how == "fused":
        dev.two_pass(x, w, out)
    elif how == "split":
        out.copy_(x)
        dev.two_pass_split(out, scratch, w)
    elif how == "single":
        dev.single_pass(out if copy_back else x, dense, scratch, copy_back=copy_back)
    elif how == "host":
        dev.two_pass_host(host, host, w)
    else:  # pragma: no cover
        raise ConfigError(f"unknown stage kind {how!r}")


def _dense_reference(x, kernel: SeparableKernel) -> np.ndarray:
    """The check's reference: the naive dense convolution of every plane ON THE CPU,
    restated from the reference's vectorised single pass (single_pass_rows_vec,
    S/conv.py:86-114: products of the shifted valid-region slices with K[i][j],
    folded row-major from the first product, each a float32 numpy op), exactly as
    check_stage_output computes it with conv_single_pass_generic
    (S/bench.py:196-198). Independent of the GPU; zero outside the valid region."""
    src = x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x, np.float32)
    dense = outer_product(kernel).matrix
    W = dense.shape[0]
    r = W // 2
    P, R, C = src.shape
    out = np.zeros_like(src)
    acc = None
    for i in range(W):
        for j in range(W):
            term = src[:, i:R - 2 * r + i, j:C - 2 * r + j] * dense[i, j]
            acc = term if acc is None else acc + term
    out[:, r:R - r, r:C - r] = acc
    return out


def check_stage_output(x, kernel: SeparableKernel, variant: ConvVariant, how: str) -> str | None:
    """Compare one GPU stage with the dense reference (S/bench.py:182-224): bitwise for
    single-pass variants, REL_TOL/ABS_TOL on the doubly-interior region for two-pass."""
    import torch

    w = kernel.weights
    dense = outer_product(kernel).matrix
    P, R, C = x.shape
    ref = _dense_reference(x, kernel)
    out = torch.empty_like(x)
    scratch = torch.zeros_like(x)
    host = None
    if how == "host":
        host = [np.ascontiguousarray(p) for p in x.cpu().numpy()]
    if how == "single" and variant.copy_back:
        out.copy_(x)
    _run_once(how, x, w, dense, variant.copy_back, out, scratch, host)
    torch.cuda.synchronize()
    if how == "host":
        got = np.stack(host)
    elif how == "single":
        got = (out if variant.copy_back else scratch).cpu().numpy()
    else:
        got = out.cpu().numpy()
    r = kernel.radius
    if variant.algorithm is Algorithm.TWO_PASS:
        reg = doubly_interior_region(R, C, r)
        g = got[:, reg.row_lo:reg.row_hi, reg.col_lo:reg.col_hi].astype(np.float64)
        want = ref[:, reg.row_lo:reg.row_hi, reg.col_lo:reg.col_hi].astype(np.float64)
        err = np.abs(g - want)
        if not np.all(err <= ABS_TOL + REL_TOL * np.abs(want)):
            return f"max deviation {float(err.max()):.3e} beyond tolerance"
        return None
    reg = valid_region(R, C, r)
    s = (slice(None), slice(reg.row_lo, reg.row_hi), slice(reg.col_lo, reg.col_hi))
    if not np.array_equal(got[s], ref[s]):
        return "output not bitwise equal to the dense reference"
    return None


def time_stage(x, kernel: SeparableKernel, variant: ConvVariant, how: str, reps: int, label: str,
               plan: Cuda) -> BenchRecord:
    """One untimed warm-up, then `reps` convolutions timed as a block (S/bench.py:134-179)."""
    import torch

    if reps < 1:
        raise ConfigError(f"reps must be >= 1, got {reps}")
    w = kernel.weights
    dense = outer_product(kernel).matrix
    out = torch.empty_like(x)
    scratch = torch.zeros_like(x)
    host = None
    if how == "host":
        host = [torch.empty(x.shape[1:], dtype=torch.float32, pin_memory=True) for _ in range(x.shape[0])]
        for p in range(x.shape[0]):
            host[p].copy_(x[p])
    _run_once(how, x, w, dense, variant.copy_back, out, scratch, host)
    torch.cuda.synchronize()
    if how == "host":
        t0 = time.perf_counter_ns()
        for _ in range(reps):
            _run_once(how, x, w, dense, variant.copy_back, out, scratch, host)
        total = time.perf_counter_ns() - t0
    else:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            _run_once(how, x, w, dense, variant.copy_back, out, scratch, host)
        b.record()
        b.synchronize()
        total = int(a.elapsed_time(b) * 1e6)
    P, R, C = x.shape
    return BenchRecord(label=label, variant=variant, plan=plan, rows=R, cols=C, planes=P, reps=reps,
                       total_ns=total, per_image_ns=max(1, round(total / reps)))


def run_gpu_ladder(config: GpuLadderConfig, kernel: SeparableKernel | None = None) -> LadderResult:
    """Every configured GPU stage on every size: check first, then time (S/bench.py:227-259)."""
    import torch

    kernel = kernel or gaussian5()
    names = config.stages or tuple(s[0] for s in GPU_STAGES)
    by_name = {s[0]: s for s in GPU_STAGES}
    sizes = sorted(config.sizes, key=lambda rc: (rc[0] * rc[1], rc))
    plan = Cuda(device=config.device)
    result = LadderResult()
    for name in names:
        label, algorithm, copy, how = by_name[name]
        if algorithm is Algorithm.SINGLE_PASS_UNROLLED5 and kernel.width != 5:
            algorithm = Algorithm.SINGLE_PASS_GENERIC  # the unrolled body is width-5 only (S/conv.py:354)
        variant = ConvVariant(algorithm, copy_back=copy)
        for rows, cols in sizes:
            img = make_synthetic(rows, cols, config.planes, config.seed, device=f"cuda:{config.device}")
            x = torch.stack([p.data for p in img.planes])
            problem = check_stage_output(x, kernel, variant, how)
            if problem is not None:
                result.failures.append(StageFailure(label, rows, cols, problem))
                continue
            result.records.append(time_stage(x, kernel, variant, how, config.reps, label, plan))
    return result


def speedup_table(records: Sequence[BenchRecord], baseline_label: str,
                  baseline_ns: dict[tuple[int, int, int], int] | None = None) -> list[BenchRecord]:
    """Speedups against a baseline stage at the same size (S/bench.py:262-274); the
    baseline may come from another run (e.g. the reference's own CPU Opt-0 rows)."""
    base = dict(baseline_ns or {})
    for rec in records:
        if rec.label == baseline_label:
            base[(rec.rows, rec.cols, rec.planes)] = rec.per_image_ns
    if not base:
        raise ConfigError(f"baseline stage {baseline_label!r} missing from records")
    return [replace(r, speedup=(None if base.get((r.rows, r.cols, r.planes)) is None
                                else base[(r.rows, r.cols, r.planes)] / r.per_image_ns)) for r in records]


def _bool_cell(value: bool | None) -> str:
    if value is None:
        return ""
    return "true" if value else "false"


def record_row(rec: BenchRecord, sms: int | None = None) -> str:
    """CSV row in the reference's schema; plan "cuda", workers = SMs (S/bench.py:304-330)."""
    if rec.speedup is not None and rec.speedup <= 0:
        raise InvalidArgumentError("speedup must be positive")
    speedup = "" if rec.speedup is None else f"{rec.speedup:.4f}"
    return ",".join([
        rec.label, rec.variant.algorithm.value, _bool_cell(rec.variant.copy_back), "cuda",
        "" if sms is None else str(sms), "", "", str(rec.rows), str(rec.cols), str(rec.planes), str(rec.reps),
        str(rec.total_ns), str(rec.per_image_ns), speedup, _bool_cell(rec.build_vectorized),
    ])


def emit_csv(records: Sequence[BenchRecord], sink: str | Path | IO[str], sms: int | None = None) -> None:
    """Records as CSV, stage order then size ascending (S/bench.py:333-354)."""
    ordered = sorted(records, key=lambda r: (_STAGE_ORDER.get(r.label, len(_STAGE_ORDER)), r.label,
                                             r.rows * r.cols, r.rows, r.cols, r.planes))
    text = "\n".join([CSV_HEADER] + [record_row(r, sms) for r in ordered]) + "\n"
    if isinstance(sink, (str, Path)):
        Path(sink).write_text(text, encoding="ascii")
    else:
        sink.write(text)


REFERENCE_SIZES = ((1152, 1152), (1728, 1728), (2592, 2592), (3888, 3888), (5832, 5832), (8748, 8748))


def _parse_sizes(text: str) -> tuple[tuple[int, int], ...]:
    out = []
    for item in text.split(","):
        try:
            r, c = item.lower().split("x")
            out.append((int(r), int(c)))
        except ValueError as exc:
            raise ConfigError(f"bad size {item!r}, expected ROWSxCOLS") from exc
    return tuple(out)


def main(argv: Sequence[str] | None = None) -> int:
    """`python -m paper_1711_09791_b200.ladder`: the reference's `sepconv ladder` flags
    (--sizes/--planes/--seed/--reps/--kernel/--stages/--csv, S/cli.py:104-141) for the
    GPU stages; exit 2 on a correctness failure like _cmd_ladder (S/cli.py:227-250)."""
    import argparse
    import sys

    import torch

    from .kernels import SeparableKernel

    ap = argparse.ArgumentParser(prog="sepconv-b200-ladder", description="GPU stages of the optimisation ladder")
    ap.add_argument("--sizes", type=_parse_sizes, default=REFERENCE_SIZES)
    ap.add_argument("--planes", type=int, default=3)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--reps", type=int, default=1000)
    ap.add_argument("--kernel", default="gaussian5", help='"gaussian5" or comma-separated weights')
    ap.add_argument("--stages", default=None, help="comma-separated GPU stage labels")
    ap.add_argument("--csv", dest="csv_out", default=None)
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)
    kernel = gaussian5() if a.kernel == "gaussian5" else SeparableKernel([float(v) for v in a.kernel.split(",")])
    cfg = GpuLadderConfig(sizes=a.sizes, planes=a.planes, seed=a.seed, reps=a.reps, device=a.device,
                          stages=None if a.stages is None else tuple(a.stages.split(",")))
    res = run_gpu_ladder(cfg, kernel)
    sms = torch.cuda.get_device_properties(a.device).multi_processor_count
    if a.csv_out is not None:
        emit_csv(res.records, a.csv_out, sms=sms)
        print(f"wrote {len(res.records)} records to {a.csv_out}")
    else:
        emit_csv(res.records, sys.stdout, sms=sms)
    for f in res.failures:
        print(f"correctness failure: {f.label} on {f.rows}x{f.cols}: {f.detail}", file=sys.stderr)
    return 2 if res.failures else 0


if __name__ == "__main__":
    raise SystemExit(main())
