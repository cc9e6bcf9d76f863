"""`convolve_image` with a CUDA execution plan (S/executors.py:269-412).

The reference's plans schedule row blocks on CPU threads (Sequential,
StaticChunked, TaskPool); here one plan type, `Cuda`, replaces all three: every
plane of the image is covered by ONE grid launch per pass (the reference's
plane agglomeration, S/executors.py:334-356, taken to its limit), and the
results are bit-identical to every reference plan (T/test_executors.py:188-231).

Two-pass end states are the reference's in every case (S/executors.py:303-326):
workspace = H0 scratch (zeroed, then the row pass), image = V(H0) with its ring
untouched.
  * device image with a workspace given: one pass that writes both buffers (K5,
    or K2+K3); without one: the same pass without the scratch writes
    (sc_two_pass_inplace_f32, 2 traversals).
  * host image with a workspace given: the streamed split path (H2D -> K1 + the
    row pass -> D2H of both buffers, sc_two_pass_host_split_f32).
  * host image without a workspace (the reference then allocates a zero one the
    caller never sees): the streamed fused path, image only (H2D -> K1 -> D2H).
    Cuda(fused=False) takes the split path here too.

The arguments are duck-typed: the reference's own Image / Plane /
SeparableKernel / ConvVariant objects work as well as this package's mirrors
(the reference-side plugin, plugin.py, relies on that).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .conv import Algorithm, ConvVariant, OpCounter
from .errors import InvalidArgumentError, UnsupportedCombinationError, UnsupportedWidthError
from .image import Image, valid_region
from .kernels import SeparableKernel, outer_product
from .multi import partition_block  # noqa: F401  (re-exported like the reference)


@dataclass(frozen=True)
class Cuda:
    """Run on CUDA devices. device=None: the image's device (or the current one
    for host images). fused: stream host images through the fused kernel.
    devices: several GPUs from this one process (host images, fused two-pass):
    the image is split into row bands (the reference's partition_block), each
    streamed through its own GPU and PCIe link concurrently; same bits.
    register_host: host images' buffers of 64 MB and more are page-locked on
    first use and stay registered while they live, so repeated calls DMA
    straight from them (False: always stage through the pinned ring)."""

    device: int | None = None
    fused: bool = True
    devices: tuple[int, ...] | None = None
    register_host: bool = True  # page-lock large host buffers once, for their lifetime (device.HostRegistry)

    def __post_init__(self):
        if self.device is not None and self.device < 0:
            raise InvalidArgumentError(f"device must be >= 0, got {self.device}")
        if self.devices is not None:
            devs = tuple(int(d) for d in self.devices)
            if not devs or any(d < 0 for d in devs):
                raise InvalidArgumentError(f"devices must be a non-empty list of indices >= 0, got {self.devices}")
            if self.device is not None:
                raise InvalidArgumentError("give either device or devices, not both")
            object.__setattr__(self, "devices", devs)


ExecPlan = Cuda


def make_plan(mode: str, workers: int | None = None, cutoff: int = 100, agglomerate: bool = False,
              *, device: int | None = None, fused: bool = True, devices=None) -> ExecPlan:
    """Plan from loose configuration (CLI flags, request bodies), S/executors.py:88-109.

    mode "cuda" is the B200 plan. The reference's CPU thread modes are not part of
    this build and raise UnsupportedCombinationError naming the replacement.
    """
    if mode == "cuda":
        if agglomerate:
            # every launch already covers all planes; accepted for compatibility
            pass
        return Cuda(device=device, fused=fused, devices=tuple(devices) if devices is not None else None)
    if mode in ("sequential", "static", "taskpool"):
        raise UnsupportedCombinationError(
            f"plan mode {mode!r} schedules CPU threads; the B200 build runs mode 'cuda'"
        )
    raise InvalidArgumentError(f"unknown plan mode {mode!r}")


@dataclass
class LaunchStats:
    """Kernel launches issued and wall time (S/executors.py:112-118)."""

    parallel_region_launches: int = 0
    tasks_spawned: int = 0
    wall_time_ns: int = 0


def _stacked(image: Image):
    """A (P, R, C) strided view when the planes are evenly spaced in one CUDA
    allocation (one grid for all planes), else None."""
    import torch

    ts = [p.data for p in image.planes]
    t0 = ts[0]
    if len(ts) == 1:
        return t0.unsqueeze(0)
    step = ts[1].data_ptr() - t0.data_ptr()
    if step <= 0 or step % 4:
        return None
    for i, t in enumerate(ts):
        if (t.data_ptr() - t0.data_ptr() != i * step or t.stride() != t0.stride()
                or t.device != t0.device or t.untyped_storage().data_ptr() != t0.untyped_storage().data_ptr()):
            return None
    ps = step // 4
    rs = t0.stride(0)
    if ps < image.rows * rs:
        return None
    return torch.as_strided(t0, (len(ts), image.rows, image.cols), (ps, rs, 1))


def _device_groups(image: Image):
    st = _stacked(image)
    if st is not None:
        return [st]
    return [p.data.unsqueeze(0) for p in image.planes]


def convolve_image(image: Image, kernel: SeparableKernel, variant: ConvVariant, plan: ExecPlan, *,
                   vectorized: bool = True, workspace: Image | None = None, pool=None,
                   counter: OpCounter | None = None) -> LaunchStats:
    """Convolve every plane of `image` (S/executors.py:269-405), on the GPU.

    Single-pass variants write `workspace` (allocated if not given) and optionally
    copy the valid region back into `image`; two-pass finishes with the result in
    `image`. Returns launch statistics; samples are bit-identical to the reference.
    """
    import torch

    from . import device as dev

    algo = Algorithm(getattr(variant.algorithm, "value", variant.algorithm))
    if algo is Algorithm.SINGLE_PASS_UNROLLED5 and kernel.width != 5:
        raise UnsupportedWidthError(f"unrolled variant needs width 5, got {kernel.width}")
    if not isinstance(plan, Cuda):
        raise UnsupportedCombinationError(
            f"plan {plan!r} is a CPU thread plan; pass Cuda() (make_plan('cuda'))"
        )
    if counter is not None:
        raise InvalidArgumentError("operation counters are supported for sequential runs only")
    if pool is not None:
        raise UnsupportedCombinationError("worker pools belong to the CPU plans; Cuda() takes none")

    rows, cols = image.rows, image.cols
    r = kernel.radius
    region = valid_region(rows, cols, r)
    nplanes = image.plane_count
    taps = np.ascontiguousarray(kernel.weights, dtype=np.float32)
    on_dev = _on_device(image)
    if not on_dev and any(_on_device_plane(p) for p in image.planes):
        raise InvalidArgumentError("image planes must all be host arrays or all CUDA tensors")
    two_pass = algo is Algorithm.TWO_PASS
    copy_back = bool(variant.copy_back) and not two_pass
    given_ws = workspace is not None
    if workspace is None and not (two_pass and plan.fused):
        workspace = Image.zeros_like(image)  # the reference's fresh zero workspace (S/executors.py:303-304)
    if workspace is not None:
        if workspace.rows != rows or workspace.cols != cols or workspace.plane_count != nplanes:
            raise InvalidArgumentError("workspace must match the image's dimensions")
        if _on_device(workspace) != on_dev:
            raise InvalidArgumentError("workspace must live where the image lives")
    # (two-pass without a workspace: the fused paths need none, nothing is allocated)

    stats = LaunchStats()
    before = _lib.launch_count()
    t0 = time.perf_counter_ns()

    if on_dev:
        device_index = image.planes[0].data.device
        with torch.cuda.device(device_index):
            img_groups = _device_groups(image)
            ws_groups = _device_groups(workspace) if workspace is not None else [None] * len(img_groups)
            if len(img_groups) != len(ws_groups):
                img_groups = [p.data.unsqueeze(0) for p in image.planes]
                ws_groups = [p.data.unsqueeze(0) for p in workspace.planes]
            for ig, wg in zip(img_groups, ws_groups):
                if two_pass and not given_ws and plan.fused:
                    dev.two_pass_inplace(ig, taps)  # the workspace is unobservable: image only
                elif two_pass:
                    dev.two_pass_split(ig, wg, taps)
                else:
                    dev.single_pass(ig, outer_product(kernel).matrix, wg, copy_back=copy_back)
            torch.cuda.current_stream().synchronize()
    else:
        device_index = plan.device if plan.device is not None else (
            plan.devices[0] if plan.devices else torch.cuda.current_device())
        img_planes = [_host_array(p) for p in image.planes]
        ws_planes = [_host_array(p) for p in workspace.planes] if workspace is not None else None
        if two_pass and plan.fused and not given_ws:
            # the workspace is the reference's internal zero buffer: unobservable
            dev.two_pass_host(img_planes, img_planes, taps, device=device_index, devices=plan.devices,
                              register=plan.register_host)
        elif two_pass:
            dev.two_pass_host_split(img_planes, ws_planes, taps, device=device_index, register=plan.register_host,
                                    devices=plan.devices)
        else:
            # streamed like the two-pass: workspace[valid] (and image[valid] with
            # copy-back) written in place, nothing else touched
            dev.single_pass_host(img_planes, ws_planes, outer_product(kernel).matrix, copy_back=copy_back,
                                 device=device_index, register=plan.register_host, devices=plan.devices)

    stats.wall_time_ns = time.perf_counter_ns() - t0
    stats.parallel_region_launches = _lib.launch_count() - before
    return stats


def _on_device_plane(plane) -> bool:
    d = plane.data
    return bool(getattr(d, "is_cuda", False))


def _on_device(image) -> bool:
    return all(_on_device_plane(p) for p in image.planes)


def _host_array(plane) -> np.ndarray:
    """The plane's host buffer, written in place (a reference Plane keeps a
    C-contiguous float32 numpy array, S/image.py:37-39)."""
    a = plane.data
    if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous or a.ndim != 2:
        raise InvalidArgumentError("host planes must be C-contiguous 2-D float32 numpy arrays")
    return a


def result_image(image: Image, workspace: Image, variant: ConvVariant) -> Image:
    """Where the convolved samples live after convolve_image (S/executors.py:408-412)."""
    if variant.algorithm is Algorithm.TWO_PASS or variant.copy_back:
        return image
    return workspace
