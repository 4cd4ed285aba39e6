"""Non-maximum suppression (nms.py) on the GPU."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import WorkerConfig
from .gradient import GradientField

# offsets (dy, dx) of the two neighbours along each quantised direction
# (nms.py:28-33; 45 compares up-right/down-left, 135 up-left/down-right)
NEIGHBORS = {
    0: ((0, -1), (0, 1)),
    45: ((-1, 1), (1, -1)),
    90: ((-1, 0), (1, 0)),
    135: ((-1, -1), (1, 1)),
}


@dataclass(frozen=True)
class ThinnedField:
    width: int
    height: int
    magnitude: np.ndarray = field(repr=False)

    def __post_init__(self):
        if self.magnitude.shape != (self.height, self.width):
            raise ValueError(
                f"magnitude has shape {self.magnitude.shape}, expected {(self.height, self.width)}")
        self.magnitude.flags.writeable = False


def non_max_suppress(grad: GradientField, cfg: WorkerConfig | None = None,
                     band_times: list[list[int]] | None = None) -> ThinnedField:
    """Keep pixels >= both neighbours along their direction (ties survive),
    replicate borders; suppressed pixels become 0.0."""
    from . import canny

    torch = canny.require_cuda()
    mag = torch.from_numpy(np.ascontiguousarray(grad.magnitude, dtype=np.float64)).cuda()
    ori = torch.from_numpy(np.ascontiguousarray(grad.orientation, dtype=np.int64)).cuda()
    thin = canny.nms_f64(mag, ori)
    return ThinnedField(width=grad.width, height=grad.height, magnitude=thin.cpu().numpy())
