"""CPU ORACLE -- test infrastructure only.

ctypes front-end for ``oracle/ef_oracle.c``, the plain-C float64 restatement of
the reference Canny path (see that file's header for the file:line map).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module, and only as the checker or
the timed CPU baseline.  The product package never imports it.

Parity pin: ``tests/test_oracle_golden.py`` checks this oracle bit-for-bit
against golden vectors produced by running the reference package itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libef_oracle.so")
_lib = None


def build() -> str:
    """Compile the oracle shared library (plain gcc via oracle/Makefile)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "ef_oracle.c")
    ):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    lib.ef_oracle_stages.argtypes = [P, I64, I64, P, I, D, D, P, P, P, P, P, P, P]
    lib.ef_oracle_stages.restype = I
    lib.ef_oracle_canny.argtypes = [P, P, I64, I64, I64, P, I, D, D, P, P, I, I64]
    lib.ef_oracle_canny.restype = I
    lib.ef_oracle_trace.argtypes = [P, I64, I64, P]
    lib.ef_oracle_trace.restype = I
    lib.ef_oracle_quantize.argtypes = [D, D]
    lib.ef_oracle_quantize.restype = I64
    _lib = lib
    return lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def gaussian_weights(sigma: float, radius: int | None = None) -> np.ndarray:
    """Restates build_gaussian_kernel (filtering.py:32-40): radius ceil(3*sigma),
    w = exp(-x^2 / (2 sigma^2)) normalised by its numpy sum.  An explicit
    radius gives the configs' "5x5" kernel (radius 2) with the same formula."""
    if not (math.isfinite(sigma) and sigma > 0):
        raise ValueError(f"sigma must be positive and finite, got {sigma}")
    r = math.ceil(3.0 * sigma) if radius is None else int(radius)
    x = np.arange(-r, r + 1, dtype=np.float64)
    w = np.exp(-(x * x) / (2.0 * sigma * sigma))
    w /= w.sum()
    return w


def stages(pixels: np.ndarray, weights: np.ndarray, low: float, high: float) -> dict:
    """Every intermediate of the reference pipeline for one float64 frame."""
    px = np.ascontiguousarray(pixels, dtype=np.float64)
    h, w = px.shape
    wt = np.ascontiguousarray(weights, dtype=np.float64)
    r = (len(wt) - 1) // 2
    out = {k: np.empty((h, w), np.float64) for k in ("blurred", "gx", "gy", "magnitude", "thinned")}
    out["orientation"] = np.empty((h, w), np.int64)
    out["labels"] = np.empty((h, w), np.uint8)
    rc = _load().ef_oracle_stages(
        _ptr(px), h, w, _ptr(wt), r, float(low), float(high), _ptr(out["blurred"]),
        _ptr(out["gx"]), _ptr(out["gy"]), _ptr(out["magnitude"]), _ptr(out["orientation"]),
        _ptr(out["thinned"]), _ptr(out["labels"]),
    )
    if rc != 0:
        raise RuntimeError(f"ef_oracle_stages failed ({rc})")
    out["final"] = trace(out["labels"])
    return out


def canny(frames: np.ndarray, weights: np.ndarray, low: float, high: float,
          threads: int = 0, band_rows: int = 64) -> tuple[np.ndarray, np.ndarray]:
    """labels (u8) and final (bool) for a (B, H, W) or (H, W) u8/float64 input."""
    arr = np.asarray(frames)
    squeeze = arr.ndim == 2
    if squeeze:
        arr = arr[None]
    b, h, w = arr.shape
    if arr.dtype == np.uint8:
        px8, px = np.ascontiguousarray(arr), None
    else:
        px8, px = None, np.ascontiguousarray(arr, dtype=np.float64)
    wt = np.ascontiguousarray(weights, dtype=np.float64)
    labels = np.empty((b, h, w), np.uint8)
    final = np.empty((b, h, w), np.uint8)
    rc = _load().ef_oracle_canny(_ptr(px), _ptr(px8), b, h, w, _ptr(wt), (len(wt) - 1) // 2,
                                 float(low), float(high), _ptr(labels), _ptr(final),
                                 int(threads), int(band_rows))
    if rc != 0:
        raise RuntimeError(f"ef_oracle_canny failed ({rc})")
    final = final.view(np.bool_)
    return (labels[0], final[0]) if squeeze else (labels, final)


def trace(labels: np.ndarray) -> np.ndarray:
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    h, w = lab.shape
    final = np.empty((h, w), np.uint8)
    if _load().ef_oracle_trace(_ptr(lab), h, w, _ptr(final)) != 0:
        raise RuntimeError("ef_oracle_trace failed")
    return final.view(np.bool_)


def quantize(gx: float, gy: float) -> int:
    return int(_load().ef_oracle_quantize(float(gx), float(gy)))


def blur(pixels: np.ndarray, weights: np.ndarray) -> np.ndarray:
    """gaussian_blur (filtering.py:43-91) for one float64 frame: the oracle's C
    restatement's `blurred` stage."""
    return stages(pixels, weights, 0.0, 0.0)["blurred"]


def laplacian(blurred: np.ndarray) -> np.ndarray:
    """Restates laplacian (gradient.py:93-107) over _stencil_band
    (gradient.py:51-70): replicate 1-pixel margin, LAPLACIAN_MASK taps in
    row-major order, zero taps skipped, accumulated from +0.0 with separately
    rounded multiply and add (numpy elementwise float64 ops, no FMA)."""
    p = np.pad(np.asarray(blurred, dtype=np.float64), 1, mode="edge")
    h, w = p.shape[0] - 2, p.shape[1] - 2
    out = np.zeros((h, w), np.float64)
    for dy, dx, c in ((0, 1, 1.0), (1, 0, 1.0), (1, 1, -4.0), (1, 2, 1.0), (2, 1, 1.0)):
        out = out + c * p[dy:dy + h, dx:dx + w]
    return out
