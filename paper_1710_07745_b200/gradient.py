"""Sobel gradient field and the Laplacian operator (gradient.py), on the GPU.

sobel(img) is the exact float64 stage kernel run with the identity smoothing
kernel (radius 0, weight 1.0 -- multiplying by 1.0 is exact), so gx, gy and
magnitude are bit-identical to gradient.py:73-90 and the orientation uses the
same certified sector test as the fused path.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import WorkerConfig
from .image import GrayImage

SOBEL_X = np.array([[-1, 0, 1], [-2, 0, 2], [-1, 0, 1]], dtype=np.float64)
SOBEL_Y = np.array([[-1, -2, -1], [0, 0, 0], [1, 2, 1]], dtype=np.float64)
LAPLACIAN_MASK = np.array([[0, 1, 0], [1, -4, 1], [0, 1, 0]], dtype=np.float64)
ORIENTATIONS = (0, 45, 90, 135)
_IDENTITY = np.array([1.0])


@dataclass(frozen=True)
class GradientField:
    width: int
    height: int
    gx: np.ndarray = field(repr=False)
    gy: np.ndarray = field(repr=False)
    magnitude: np.ndarray = field(repr=False)
    orientation: np.ndarray = field(repr=False)  # int degrees in {0, 45, 90, 135}

    def __post_init__(self):
        shape = (self.height, self.width)
        for name in ("gx", "gy", "magnitude", "orientation"):
            arr = getattr(self, name)
            if arr.shape != shape:
                raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
            arr.flags.writeable = False


def quantize_orientation_array(gx: np.ndarray, gy: np.ndarray) -> np.ndarray:
    """Nearest of 0/45/90/135 of atan2(gy, gx) folded into [0, 180); ties to
    the larger bin; (0, 0) -> 0 (gradient.py:37-44).  GPU kernel."""
    from . import canny

    torch = canny.require_cuda()
    a = np.ascontiguousarray(np.broadcast_arrays(np.asarray(gx, np.float64), np.asarray(gy, np.float64))[0])
    b = np.ascontiguousarray(np.broadcast_arrays(np.asarray(gx, np.float64), np.asarray(gy, np.float64))[1])
    out = canny.quantize_f64(torch.from_numpy(a.reshape(-1)).cuda(), torch.from_numpy(b.reshape(-1)).cuda())
    return out.cpu().numpy().reshape(a.shape)


def quantize_orientation(gx: float, gy: float) -> int:
    return int(quantize_orientation_array(np.float64(gx), np.float64(gy)))


def sobel(img: GrayImage, cfg: WorkerConfig | None = None,
          band_times: list[list[int]] | None = None) -> GradientField:
    from . import canny

    torch = canny.require_cuda()
    src = torch.from_numpy(np.ascontiguousarray(img.pixels)).cuda()
    st = canny.stages_f64(src, _IDENTITY, 0.0, 0.0)
    return GradientField(width=img.width, height=img.height, gx=st["gx"].cpu().numpy(),
                         gy=st["gy"].cpu().numpy(), magnitude=st["magnitude"].cpu().numpy(),
                         orientation=st["orientation"].cpu().numpy())


def laplacian(img: GrayImage, cfg: WorkerConfig | None = None,
              band_times: list[list[int]] | None = None) -> GrayImage:
    """5-point Laplacian with replicate borders (gradient.py:96-107)."""
    from . import canny

    torch = canny.require_cuda()
    src = torch.from_numpy(np.ascontiguousarray(img.pixels)).cuda()
    return GrayImage.from_array(canny.laplacian_f64(src).cpu().numpy())
