"""Double threshold and hysteresis tracing (hysteresis.py) on the GPU.

trace_edges runs the tile union-find kernels (ef_trace_edges); the result is
the same edge set as the reference's scipy.ndimage.label + isin
(hysteresis.py:63-69).  trace_edges_parallel runs the band-partitioned
variant -- per-band GPU labelling, then the band-seam union-find
(ef_band_merge, the analogue of hysteresis.py:112-130) -- and returns the
identical set, as the reference's does.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .engine import WorkerConfig, plan_bands
from .nms import ThinnedField

LABEL_NONE = 0
LABEL_WEAK = 1
LABEL_STRONG = 2


@dataclass(frozen=True)
class Thresholds:
    low: float
    high: float

    def __post_init__(self):
        if not (0 <= self.low <= self.high):
            raise ValueError(f"need 0 <= low <= high, got low={self.low}, high={self.high}")


@dataclass(frozen=True)
class EdgeMap:
    width: int
    height: int
    labels: np.ndarray = field(repr=False)  # uint8 in {NONE, WEAK, STRONG}
    final: np.ndarray | None = field(default=None, repr=False)  # bool once traced

    def __post_init__(self):
        shape = (self.height, self.width)
        if self.labels.shape != shape:
            raise ValueError(f"labels have shape {self.labels.shape}, expected {shape}")
        self.labels.flags.writeable = False
        if self.final is not None:
            if self.final.shape != shape:
                raise ValueError(f"final has shape {self.final.shape}, expected {shape}")
            self.final.flags.writeable = False


def double_threshold(thin: ThinnedField, t: Thresholds) -> EdgeMap:
    """Strong where magnitude >= high, weak where >= low, else none."""
    from . import canny

    torch = canny.require_cuda()
    mag = torch.from_numpy(np.ascontiguousarray(thin.magnitude, dtype=np.float64)).cuda()
    labels = canny.threshold_f64(mag, t.low, t.high)
    return EdgeMap(width=thin.width, height=thin.height, labels=labels.cpu().numpy())


def _labels_on_device(edge_map: EdgeMap):
    from . import canny

    torch = canny.require_cuda()
    lab = np.ascontiguousarray(edge_map.labels, dtype=np.uint8)
    if lab.size and lab.max() > LABEL_STRONG:
        raise ValueError("labels must be in {0, 1, 2}")
    return torch.from_numpy(lab).cuda()


def trace_edges(edge_map: EdgeMap) -> EdgeMap:
    """Flood from all strong seeds through 8-connected weak/strong pixels."""
    from . import canny

    lab = _labels_on_device(edge_map)
    final = canny.trace_edges_u8(lab)[0]
    return EdgeMap(width=edge_map.width, height=edge_map.height, labels=edge_map.labels,
                   final=final.cpu().numpy().view(np.bool_))


def trace_edges_parallel(edge_map: EdgeMap, cfg: WorkerConfig) -> EdgeMap:
    """Same final set as trace_edges via per-band labelling plus the band-seam
    merge; bands follow plan_bands(height, cfg) like the reference."""
    from . import bands

    lab = _labels_on_device(edge_map)
    final = bands.trace_bands_local(lab, plan_bands(edge_map.height, cfg))
    return EdgeMap(width=edge_map.width, height=edge_map.height, labels=edge_map.labels,
                   final=final.cpu().numpy().view(np.bool_))
