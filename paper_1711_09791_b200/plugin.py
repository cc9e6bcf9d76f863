"""Reference-side plugin: the B200 path registered inside the real sepconv_lab.

A sepconv_lab user switches by installing the plugin once and passing the new
plan; nothing else in their code changes::

    import sepconv_lab as sl
    from paper_1711_09791_b200 import plugin

    plugin.install()                       # patches the imported sepconv_lab
    stats = sl.convolve_image(image, sl.gaussian5(), sl.ConvVariant(sl.Algorithm.TWO_PASS),
                              sl.make_plan("cuda"), workspace=workspace)

`install()` patches the imported reference modules at run time (the reference's
files are not modified, so its own plans and tests keep their behaviour):

* ``convolve_image`` (S/executors.py:269-405) -- a ``Cuda`` plan runs on the GPU
  through libsepconv_b200.so (executors.py here); every other plan goes to the
  reference's own implementation. The reference's Image / Plane /
  SeparableKernel / ConvVariant objects are used as they are (numpy planes are
  read and written in place, pageable memory included), and the end state of
  BOTH buffers is the reference's: with a workspace, two-pass leaves H0 in it.
* ``make_plan("cuda", ...)`` (S/executors.py:88-109) returns ``Cuda()``.
* ``bench.plan_summary`` (S/bench.py:288-295) reports mode "cuda"; GPU ladder
  stages ``Gpu-*`` (``bench.GPU_LADDER_STAGES``, beside ``LADDER_STAGES``,
  S/bench.py:104-119) run when named in ``LadderConfig.stages``, with the
  reference's check-before-timing rule (its own CPU dense oracle,
  ``check_stage_output``, S/bench.py:182-224), its timing loop
  (``time_variant``) and CSV schema; the default ladder is unchanged.
* CLI ``sepconv convolve --plan cuda`` (S/cli.py:133, 187-188): the --plan
  choices gain "cuda"; ``python -m paper_1711_09791_b200.plugin ...`` is the
  ``sepconv`` entry point with the plugin installed.
* service ``PlanSpec.mode = "cuda"`` (S/schemas.py:58-65, S/service.py:98-122):
  the request model accepts it and ``POST /convolve`` is re-registered with it.

Errors raised by the GPU path come out as the reference's own exception classes
(S/errors.py), so callers' ``except sepconv_lab.InvalidArgumentError`` keeps working.
"""

from __future__ import annotations

import contextlib
import dataclasses
import functools
import sys
from typing import Literal

from . import conv as _conv
from . import errors as _errors
from . import executors as _executors
from .executors import Cuda

GPU_STAGES = (
    # label, algorithm value, copy_back, plan kind, vectorized
    ("Gpu-0", "single-generic", True, "cuda", True),
    ("Gpu-1", "single-unrolled", True, "cuda", True),
    ("Gpu-1-nocopy", "single-unrolled", False, "cuda", True),
    ("Gpu-2", "two-pass", False, "cuda", True),
)

_state: dict = {}


def _ref_module(module=None):
    if module is not None:
        return module
    import sepconv_lab

    return sepconv_lab


def translate(ref, exc: BaseException) -> BaseException:
    """The reference's exception for one of this package's (same class name)."""
    if not isinstance(exc, _errors.SepconvError):
        return exc
    name = type(exc).__name__
    cls = getattr(ref.errors, name, None)
    if cls is None:
        return ref.errors.SepconvError(str(exc))
    if name == "ExecutionError":
        return cls(getattr(exc, "failures", [(0, RuntimeError(str(exc)))]))
    if name == "PpmParseError":
        return cls(str(exc), getattr(exc, "byte_offset", 0))
    return cls(*exc.args)


@contextlib.contextmanager
def reference_errors(ref):
    try:
        yield
    except _errors.SepconvError as exc:
        raise translate(ref, exc) from exc


def _gpu_convolve(ref, image, kernel, variant, plan, *, vectorized=True, workspace=None, pool=None, counter=None):
    with reference_errors(ref):
        st = _executors.convolve_image(image, kernel, variant, plan, vectorized=vectorized, workspace=workspace,
                                       pool=pool, counter=counter)
    return ref.executors.LaunchStats(parallel_region_launches=st.parallel_region_launches,
                                     tasks_spawned=st.tasks_spawned, wall_time_ns=st.wall_time_ns)


def gpu_ops(ref=None) -> dict:
    """The reference's whole-plane operations (S/conv.py:324-440) on the GPU, taking
    the reference's Plane / SeparableKernel / DenseKernel objects and raising its
    exceptions: conv_two_pass, conv_single_pass_generic,
    conv_single_pass_unrolled5, horizontal_pass, vertical_pass, copy_back."""
    ref = _ref_module(ref)

    def wrap(fn):
        @functools.wraps(fn)
        def inner(*args, **kwargs):
            with reference_errors(ref):
                return fn(*args, **kwargs)

        return inner

    names = ("conv_two_pass", "conv_single_pass_generic", "conv_single_pass_unrolled5", "horizontal_pass",
             "vertical_pass", "copy_back")
    return {n: wrap(getattr(_conv, n)) for n in names}


def _patch(mod, name, value):
    if not hasattr(mod, name):
        return
    _state["saved"].append((mod, name, getattr(mod, name)))
    setattr(mod, name, value)


def install(module=None):
    """Register the Cuda plan in the imported sepconv_lab (idempotent); returns it."""
    ref = _ref_module(module)
    if _state.get("module") is ref:
        return ref
    if _state.get("module") is not None:
        uninstall()
    import importlib

    ex = ref.executors
    bench = importlib.import_module(ref.__name__ + ".bench")
    _state["saved"] = []
    _state["module"] = ref
    orig_convolve = ex.convolve_image
    orig_make_plan = ex.make_plan

    @functools.wraps(orig_convolve)
    def convolve_image(image, kernel, variant, plan, *, vectorized=True, workspace=None, pool=None, counter=None):
        if isinstance(plan, Cuda):
            return _gpu_convolve(ref, image, kernel, variant, plan, vectorized=vectorized, workspace=workspace,
                                 pool=pool, counter=counter)
        return orig_convolve(image, kernel, variant, plan, vectorized=vectorized, workspace=workspace, pool=pool,
                             counter=counter)

    @functools.wraps(orig_make_plan)
    def make_plan(mode, workers=None, cutoff=100, agglomerate=False):
        if mode == "cuda":
            return Cuda()
        return orig_make_plan(mode, workers, cutoff, agglomerate)

    orig_summary = bench.plan_summary

    @functools.wraps(orig_summary)
    def plan_summary(plan):
        if isinstance(plan, Cuda):
            return "cuda", len(plan.devices) if plan.devices else 1, None, None
        return orig_summary(plan)

    # GPU ladder stages beside the reference's own (LADDER_STAGES itself is left
    # alone: the reference's callers and tests size things by it), same CSV
    # schema, the same check-before-timing rule and timing loop
    algos = {a.value: a for a in ref.conv.Algorithm}
    gpu_stages = tuple((lab, algos[a], cb, kind, vec) for lab, a, cb, kind, vec in GPU_STAGES)
    orig_run_ladder = bench.run_ladder

    @functools.wraps(orig_run_ladder)
    def run_ladder(config):
        names = config.stages
        gpu = {s[0]: s for s in gpu_stages}
        if names is None or not any(n in gpu for n in names):
            return orig_run_ladder(config)  # the default ladder stays the reference's
        ref_names = tuple(n for n in names if n not in gpu)
        result = bench.LadderResult()
        if ref_names:
            part = orig_run_ladder(dataclasses.replace(config, stages=ref_names))
            result.records.extend(part.records)
            result.failures.extend(part.failures)
        kernel = ref.kernels.gaussian5()
        sizes = sorted(config.sizes, key=lambda rc: (rc[0] * rc[1], rc))
        for name in names:
            if name not in gpu:
                continue
            label, algorithm, copy, _kind, vectorized = gpu[name]
            variant = ref.conv.ConvVariant(algorithm, copy_back=copy)
            for rows, cols in sizes:
                image = ref.image.make_synthetic(rows, cols, config.planes, config.seed)
                problem = bench.check_stage_output(image, kernel, variant, Cuda(), vectorized)
                if problem is not None:
                    result.failures.append(bench.StageFailure(label, rows, cols, problem))
                    continue
                result.records.append(bench.time_variant(image, kernel, variant, Cuda(), config.reps,
                                                         vectorized=vectorized, label=label))
        if any(r.label == bench.BASELINE_LABEL for r in result.records):
            result.records = bench.speedup_table(result.records, bench.BASELINE_LABEL)
        return result

    for mod in (ref, ex, bench):
        _patch(mod, "convolve_image", convolve_image)
    for mod in (ref, ex):
        _patch(mod, "make_plan", make_plan)
    _patch(bench, "plan_summary", plan_summary)
    _patch(bench, "run_ladder", run_ladder)
    _patch(ref, "run_ladder", run_ladder)
    _patch(ref, "Cuda", Cuda)
    _patch(ex, "Cuda", Cuda)
    _state["added"] = []
    for mod, name, value in ((ref, "Cuda", Cuda), (ex, "Cuda", Cuda), (bench, "GPU_LADDER_STAGES", gpu_stages)):
        if not hasattr(mod, name):
            setattr(mod, name, value)
            _state["added"].append((mod, name))
    _install_surfaces(ref, convolve_image, make_plan, plan_summary, run_ladder)
    return ref


def _install_surfaces(ref, convolve_image, make_plan, plan_summary, run_ladder):
    """CLI and HTTP service, when their dependencies import (S/cli.py, S/service.py)."""
    import importlib

    try:
        cli = importlib.import_module(ref.__name__ + ".cli")
    except ImportError:  # pragma: no cover - httpx missing
        cli = None
    if cli is not None:
        _patch(cli, "convolve_image", convolve_image)
        _patch(cli, "make_plan", make_plan)
        _patch(cli, "run_ladder", run_ladder)
        orig_build = cli.build_parser

        @functools.wraps(orig_build)
        def build_parser():
            parser = orig_build()
            for action in parser._subparsers._group_actions:
                for name, sub in action.choices.items():
                    for a in sub._actions:
                        if "--plan" in a.option_strings and a.choices is not None and "cuda" not in a.choices:
                            a.choices = list(a.choices) + ["cuda"]
            return parser

        _patch(cli, "build_parser", build_parser)
    try:
        schemas = importlib.import_module(ref.__name__ + ".schemas")
        service = importlib.import_module(ref.__name__ + ".service")
    except ImportError:  # pragma: no cover - fastapi missing
        return
    _patch(schemas, "make_plan", make_plan)
    _patch(service, "convolve_image", convolve_image)
    _patch(service, "plan_summary", plan_summary)
    _patch(service, "run_ladder", run_ladder)
    spec = schemas.PlanSpec
    field = spec.model_fields["mode"]
    modes = tuple(getattr(field.annotation, "__args__", ()))
    if "cuda" not in modes:
        _state["schema"] = (spec, field.annotation, spec.__annotations__.get("mode"))
        new = Literal[modes + ("cuda",)] if modes else Literal["sequential", "static", "taskpool", "cuda"]
        field.annotation = new
        spec.__annotations__["mode"] = new
        spec.model_rebuild(force=True)
        schemas.ConvolveRequest.model_rebuild(force=True)
        _reroute(service, "/convolve", service.convolve)


def _reroute(service, path, endpoint):
    """Re-register a POST route so FastAPI rebuilds its body validator from the
    (rebuilt) request model."""
    from fastapi.routing import APIRoute

    app = service.app
    old = [r for r in app.router.routes if isinstance(r, APIRoute) and r.path == path and "POST" in r.methods]
    if not old:
        return
    route = old[0]
    _state.setdefault("routes", []).append((app, list(app.router.routes)))
    app.router.routes = [r for r in app.router.routes if r is not route]
    app.post(path, response_model=route.response_model)(endpoint)


def uninstall():
    """Undo install() (tests)."""
    for mod, name, value in reversed(_state.get("saved", [])):
        setattr(mod, name, value)
    for mod, name in _state.get("added", []):
        if hasattr(mod, name):
            delattr(mod, name)
    sch = _state.get("schema")
    if sch is not None:
        spec, ann, raw = sch
        spec.model_fields["mode"].annotation = ann
        if raw is not None:
            spec.__annotations__["mode"] = raw
        spec.model_rebuild(force=True)
        mod = sys.modules.get(spec.__module__)
        if mod is not None:
            mod.ConvolveRequest.model_rebuild(force=True)
    for app, routes in reversed(_state.get("routes", [])):
        app.router.routes = routes
    _state.clear()


def main(argv=None) -> int:
    """The reference's `sepconv` command line with the plugin installed
    (`python -m paper_1711_09791_b200.plugin convolve --plan cuda ...`)."""
    ref = install()
    import importlib

    cli = importlib.import_module(ref.__name__ + ".cli")
    return cli.entrypoint(argv)


if __name__ == "__main__":
    sys.exit(main())
