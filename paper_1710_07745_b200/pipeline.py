"""run_pipeline -- the drop-in for the reference's Canny entry point
(bench.py:20-140): same PipelineConfig / PipelineResult surface, computed by
the sm_100a kernels of libedgeforge_b200.so.

Paths:
  * integer pixels in [0, 255] (every config and PGM input): the fused fp32
    classify kernel with certified decisions + exact float64 fix-ups +
    tile union-find hysteresis (ef_canny_u8_host: H2D, kernels, D2H);
  * any other finite float64 pixels: the exact float64 stencil kernel in the
    reference's operation order + the same hysteresis (ef_canny_f64).
Both give labels/final bit-identical to the reference.  There is no CPU path.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .engine import StageTiming, WorkerConfig
from .filtering import GaussianKernel, build_gaussian_kernel
from .gradient import GradientField
from .hysteresis import EdgeMap, Thresholds, trace_edges_parallel
from .image import GrayImage
from .nms import ThinnedField

AUTO_HIGH_RATIO = 0.2  # high = ratio * max thinned magnitude (bench.py:20)
AUTO_LOW_RATIO = 0.4  # low = ratio * high (bench.py:21)
WORKER_HARD_CAP = 64


@dataclass
class PipelineConfig:
    sigma: float = 1.4
    thresholds: Thresholds | None = None  # None = auto ratios from the thinned field
    workers: WorkerConfig = field(default_factory=WorkerConfig)
    hysteresis_mode: str = "serial"  # serial | parallel
    operator: str = "canny"  # canny | laplacian
    radius: int | None = None  # Gaussian radius; None = ceil(3*sigma) as the reference

    def __post_init__(self):
        if self.hysteresis_mode not in ("serial", "parallel"):
            raise ValueError(f"unknown hysteresis mode {self.hysteresis_mode!r}")
        if self.operator not in ("canny", "laplacian"):
            raise ValueError(f"unknown operator {self.operator!r}")
        if self.radius is not None and self.radius < 0:
            raise ValueError(f"radius must be >= 0, got {self.radius}")

    def kernel(self) -> GaussianKernel:
        return build_gaussian_kernel(self.sigma, self.radius)


@dataclass
class PipelineResult:
    edges: EdgeMap | None = None
    response: GrayImage | None = None  # laplacian operator output
    blurred: GrayImage | None = None
    grad: GradientField | None = None
    thinned: ThinnedField | None = None
    thresholds: Thresholds | None = None


def auto_thresholds(thin: ThinnedField) -> Thresholds:
    """bench.py:51-58: high = 0.2 * max thinned magnitude, low = 0.4 * high."""
    return _auto_from_peak(float(thin.magnitude.max()))


def _auto_from_peak(peak: float) -> Thresholds:
    if peak == 0.0:
        return Thresholds(low=1.0, high=1.0)
    high = AUTO_HIGH_RATIO * peak
    return Thresholds(low=AUTO_LOW_RATIO * high, high=high)


def run_pipeline(img: GrayImage, cfg: PipelineConfig, timings: list[StageTiming] | None = None,
                 band_times: dict[str, list[list[int]]] | None = None,
                 keep_intermediates: bool = False) -> PipelineResult:
    """blur -> sobel -> nms -> threshold -> trace (or blur -> laplacian), on the GPU.

    Output is bit-identical to the reference for the same inputs and config.
    ``timings`` receives the reference's five StageTiming records (bench.py:
    76-120) with device times from CUDA events: "gaussian" carries the fused
    classifier (blur, Sobel, NMS and thresholds run in one kernel, plus its
    exact fix-ups), "sobel" / "nms" / "threshold" record 0 ns (fused into it),
    "hysteresis" the tracing kernels; operator="laplacian" records "gaussian"
    and "laplacian".  ``band_times`` is accepted for signature compatibility
    (there are no CPU bands)."""
    from . import canny

    torch = canny.require_cuda()
    clock = time.perf_counter_ns
    kernel = cfg.kernel()
    w = kernel.weights
    result = PipelineResult()
    px = img.pixels
    u8 = img.as_u8()

    def record(stage: str, t0: int, ns: int | None = None):
        if timings is not None:
            timings.append(StageTiming(stage_name=stage, workers=cfg.workers.workers,
                                       wall_ns=int(clock() - t0 if ns is None else ns), rows_processed=img.height))

    if cfg.operator == "laplacian":
        src = torch.from_numpy(np.ascontiguousarray(px)).cuda()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        blurred = canny.blur_f64(src, w)
        ev[1].record()
        resp = canny.laplacian_f64(blurred)
        ev[2].record()
        result.response = GrayImage.from_array(resp.cpu().numpy())
        record("gaussian", 0, ev[0].elapsed_time(ev[1]) * 1e6)
        record("laplacian", 0, ev[1].elapsed_time(ev[2]) * 1e6)
        if keep_intermediates:
            result.blurred = GrayImage.from_array(blurred.cpu().numpy())
        return result

    t0 = clock()
    dev_src = None
    thresholds = cfg.thresholds
    if thresholds is None or keep_intermediates:
        dev_src = torch.from_numpy(u8 if u8 is not None else np.ascontiguousarray(px)).cuda()
    if thresholds is None:
        thresholds = _auto_from_peak(canny.thinned_max(dev_src, w))
    stage_ms = None
    if u8 is not None and cfg.hysteresis_mode == "serial" and timings is not None:
        # device-resident call with per-phase events (the host-buffer path
        # pipelines several chunks on internal streams)
        if dev_src is None:
            dev_src = torch.from_numpy(u8).cuda()
        lab_d, fin_d, c_ms, h_ms = canny.canny_u8_timed(dev_src, w, thresholds.low, thresholds.high)
        labels, final = lab_d[0].cpu().numpy(), fin_d[0].cpu().numpy()
        stage_ms = (c_ms, h_ms)
    elif u8 is not None and cfg.hysteresis_mode == "serial":
        labels, final = canny.canny_u8_host(u8, w, thresholds.low, thresholds.high)
    else:
        if dev_src is None:
            dev_src = torch.from_numpy(u8 if u8 is not None else np.ascontiguousarray(px)).cuda()
        if u8 is not None:
            lab_d = canny.classify_u8(dev_src, w, thresholds.low, thresholds.high)[0]
        else:
            lab_d = canny.canny_f64(dev_src, w, thresholds.low, thresholds.high)[0][0]
        if cfg.hysteresis_mode == "parallel":
            from . import bands
            from .engine import plan_bands

            fin_d = bands.trace_bands_local(lab_d, plan_bands(img.height, cfg.workers))
        else:
            fin_d = canny.trace_edges_u8(lab_d)[0]
        labels, final = lab_d.cpu().numpy(), fin_d.cpu().numpy()
    if timings is not None:
        if stage_ms is None:  # exact / parallel paths: the whole call as the fused stage
            stage_ms = ((clock() - t0) / 1e6, 0.0)
        record("gaussian", t0, stage_ms[0] * 1e6)
        for fused in ("sobel", "nms", "threshold"):
            record(fused, t0, 0)
        record("hysteresis", t0, stage_ms[1] * 1e6)
    edges = EdgeMap(width=img.width, height=img.height, labels=np.ascontiguousarray(labels),
                    final=np.ascontiguousarray(final).view(np.bool_))
    result.edges = edges
    result.thresholds = thresholds
    if keep_intermediates:
        st = canny.stages_f64(dev_src, w, thresholds.low, thresholds.high)
        h = {k: v.cpu().numpy() for k, v in st.items()}
        result.blurred = GrayImage.from_array(h["blurred"])
        result.grad = GradientField(width=img.width, height=img.height, gx=h["gx"], gy=h["gy"],
                                    magnitude=h["magnitude"], orientation=h["orientation"])
        result.thinned = ThinnedField(width=img.width, height=img.height, magnitude=h["thinned"])
    return result


def detect_pgm(data: bytes, cfg: PipelineConfig) -> bytes:
    """The CLI's detect path (cli.py:82-90) as one call: PGM bytes in, P5
    bytes of the edge map out -- equal to
    save_pgm(edges_to_image(run_pipeline(load_pgm(data), cfg).edges)), or for
    operator="laplacian" to save_pgm(rescale_for_view(response)).

    Canny: the pixels are decoded straight into pinned host memory as bytes
    (no float64 image), cross PCIe at 1 B/px, the edge map is encoded as the
    0/255 payload on the device, and only that payload comes back."""
    import ctypes

    from . import _lib, canny
    from .image import decode_pgm_u8, pgm_header

    torch = canny.require_cuda()
    if cfg.operator != "canny":
        from .image import load_pgm, save_pgm

        res = run_pipeline(load_pgm(data), cfg)
        return save_pgm(rescale_for_view(res.response.pixels))
    # header first (errors before any device work), then the pixels into pinned memory
    info = _lib.EfPgmInfo()
    off = ctypes.c_int64(0)
    buf = bytes(data)
    rc = _lib.load().ef_pgm_parse(buf, len(buf), ctypes.byref(info), ctypes.byref(off))
    if rc != _lib.EF_OK:
        decode_pgm_u8(buf)  # raises the PgmFormatError
    h, w = info.height, info.width
    pinned = torch.empty((h, w), dtype=torch.uint8).pin_memory()
    decode_pgm_u8(buf, out=pinned.numpy())
    src = pinned.to("cuda", non_blocking=True)
    weights = cfg.kernel().weights
    thresholds = cfg.thresholds
    if thresholds is None:
        thresholds = _auto_from_peak(canny.thinned_max(src, weights))
    _, final = canny.canny_u8(src, weights, thresholds.low, thresholds.high)
    payload = torch.empty(h * w, dtype=torch.uint8, device=src.device)
    st = int(torch.cuda.current_stream().cuda_stream)
    _lib.check(_lib.load().ef_pgm_encode_edges(final.data_ptr(), h * w, payload.data_ptr(), st), "ef_pgm_encode_edges")
    out = torch.empty(h * w, dtype=torch.uint8).pin_memory()
    out.copy_(payload, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return pgm_header(w, h) + out.numpy().tobytes()


def edges_to_image(edges: EdgeMap) -> GrayImage:
    """Binary edge map as a 0/255 image (bench.py:129-133)."""
    if edges.final is None:
        raise ValueError("edge map has not been traced")
    return GrayImage.from_array(np.where(edges.final, 255.0, 0.0))


def rescale_for_view(arr: np.ndarray) -> GrayImage:
    """Linear rescale of |values| to [0, 255] (bench.py:136-140)."""
    mag = np.abs(np.asarray(arr, dtype=np.float64))
    peak = mag.max()
    return GrayImage.from_array(mag * (255.0 / peak) if peak > 0 else mag)
