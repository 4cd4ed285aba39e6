"""Gaussian stage (filtering.py): kernel construction on the host, blur on the GPU.

gaussian_blur runs the exact float64 separable pass on the device in the
reference's tap order (ef_stages_f64), so the blurred image is bit-identical to
filtering.py:66-91.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .engine import WorkerConfig
from .image import GrayImage


@dataclass(frozen=True)
class GaussianKernel:
    sigma: float
    radius: int
    weights: np.ndarray = field(repr=False)

    def __post_init__(self):
        w = np.asarray(self.weights, dtype=np.float64)
        if w.shape != (2 * self.radius + 1,):
            raise ValueError(f"expected {2 * self.radius + 1} weights, got {w.shape}")
        if not np.array_equal(w, w[::-1]):
            raise ValueError("kernel weights must be symmetric")
        if abs(w.sum() - 1.0) > 1e-12:
            raise ValueError(f"kernel weights must sum to 1, got {w.sum()!r}")
        w.flags.writeable = False
        object.__setattr__(self, "weights", w)


def build_gaussian_kernel(sigma: float, radius: int | None = None) -> GaussianKernel:
    """Sampled Gaussian normalised to unit sum (filtering.py:32-40).  radius
    defaults to the reference's ceil(3*sigma); radius=2 gives the configs'
    5x5 kernel."""
    if not (math.isfinite(sigma) and sigma > 0):
        raise ValueError(f"sigma must be positive and finite, got {sigma}")
    r = math.ceil(3.0 * sigma) if radius is None else int(radius)
    if r < 0:
        raise ValueError(f"radius must be >= 0, got {r}")
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    w /= w.sum()
    return GaussianKernel(sigma=sigma, radius=r, weights=w)


def gaussian_blur(img: GrayImage, kernel: GaussianKernel, cfg: WorkerConfig | None = None,
                  band_times: list[list[int]] | None = None) -> GrayImage:
    """Exact float64 separable blur on the GPU, replicate borders."""
    from . import canny

    torch = canny.require_cuda()
    src = torch.from_numpy(np.ascontiguousarray(img.pixels)).cuda()
    out = canny.blur_f64(src, kernel.weights)
    return GrayImage.from_array(out.cpu().numpy())
