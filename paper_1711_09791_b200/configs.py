"""The five BASELINE.json workloads and their float32 tap vectors.

Taps are computed once in float64 and cast to float32; the same float32 taps go
to the CUDA path and to the oracle. Inputs are seeded
splitmix64 streams (the reference's own generator, S/image.py:131-162) so any
row band of any plane can be regenerated on either side without a transfer.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _gauss5() -> np.ndarray:
    # gaussian5, S/kernels.py:54-56: [1,4,6,4,1] / 16 in float32
    return np.array([1, 4, 6, 4, 1], dtype=np.float32) / np.float32(16)


def _normal_taps(seed: int = 2) -> np.ndarray:
    """Config 2: five N(0,1) draws from `seed`, normalised to unit sum in float64.
    Redraws (seed+1, ...) if the raw sum is too small to normalise safely."""
    s = seed
    while True:
        w = np.random.default_rng(s).standard_normal(5)
        if abs(w.sum()) > 0.25:
            return (w / w.sum()).astype(np.float32)
        s += 1


def _sigma1() -> np.ndarray:
    m = np.arange(5, dtype=np.float64)
    w = np.exp(-((m - 2.0) ** 2) / 2.0)
    return (w / w.sum()).astype(np.float32)


CONFIG_TAPS: dict[str, np.ndarray] = {
    "gauss5": _gauss5(),
    "normal": _normal_taps(),
    "sharpen": np.array([-1, -2, 7, -2, -1], dtype=np.float32),
    "sigma1": _sigma1(),
}

# value kinds of the synthetic generator (csrc fill kernel == oracle/orc_fill_synthetic)
KIND_REF256 = 0  # make_synthetic's [0, 256) mapping, S/image.py:158-160
KIND_U01 = 1     # uniform [0, 1)
KIND_U255 = 2    # uniform [0, 255)


@dataclass(frozen=True)
class Workload:
    name: str
    frames: int
    planes: int
    rows: int
    cols: int
    kind: int
    taps: str
    seed: int
    note: str

    @property
    def pixels(self) -> int:
        """(row, col) locations across all frames; one pixel = `planes` float32 samples."""
        return self.frames * self.rows * self.cols

    @property
    def samples(self) -> int:
        return self.frames * self.planes * self.rows * self.cols

    @property
    def alg_bytes(self) -> int:
        """One read + one write of every sample: 24 B/pixel at 3 planes."""
        return 2 * 4 * self.samples

    def tap_vector(self) -> np.ndarray:
        return CONFIG_TAPS[self.taps].copy()


CONFIGS: dict[str, Workload] = {
    "cfg1": Workload("cfg1", 1, 3, 1152, 1152, KIND_U01, "gauss5", 1,
                     "3x1152x1152, U[0,1), [1,4,6,4,1]/16, two-pass faithful (PR1 oracle)"),
    "cfg2": Workload("cfg2", 1, 3, 4096, 4096, KIND_U01, "normal", 2,
                     "3x4096x4096, U[0,1), N(0,1) taps normalised to sum 1; two-pass and single-pass"),
    "cfg3": Workload("cfg3", 1, 3, 8192, 8192, KIND_U255, "sharpen", 3,
                     "3x8192x8192, U[0,255), [-1,-2,7,-2,-1]; row bands over 1/2/4/8 GPUs"),
    "cfg4": Workload("cfg4", 512, 3, 1080, 1920, KIND_U01, "sigma1", 4,
                     "512 frames x 3x1080x1920, U[0,1), Gaussian sigma=1; frames sharded"),
    "cfg5": Workload("cfg5", 1, 3, 16384, 16384, KIND_U01, "gauss5", 5,
                     "3x16384x16384, U[0,1), [1,4,6,4,1]/16; fused, row bands over 1/2/4/8 GPUs"),
}
