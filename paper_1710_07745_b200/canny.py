"""Device-level API over the C ABI: torch CUDA tensors in, torch tensors out.

This is the layer bench.py and the multi-GPU band runner use; the drop-in
mirror of the reference (pipeline.py, hysteresis.py, ...) sits on top of it.
PyTorch provides device memory and streams only -- every pixel is computed by
libedgeforge_b200.so kernels.  There is no CPU fallback: without a CUDA device
these functions raise.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib

_ws_local = threading.local()


def _torch():
    import torch

    return torch


def require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1710_07745_b200 computes on a CUDA device (B200, sm_100a); no CUDA device is visible "
            "and there is deliberately no CPU fallback"
        )
    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def host_weights(weights) -> tuple[np.ndarray, ctypes.c_void_p, int]:
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
    if w.ndim != 1 or len(w) % 2 != 1:
        raise ValueError(f"expected an odd-length 1-D weight vector, got shape {w.shape}")
    r = (len(w) - 1) // 2
    if r > _lib.MAX_RADIUS:
        raise ValueError(f"radius {r} exceeds the supported maximum {_lib.MAX_RADIUS}")
    return w, w.ctypes.data_as(ctypes.c_void_p), r


def workspace(batch: int, height: int, width: int, device=None, stream=None):
    """A cached device workspace large enough for (batch, height, width).

    One cache per (host thread, device, stream): the header's thread-safety rule
    is one workspace per concurrent launch sequence, and two threads (or two
    streams) sharing one would reset each other's counters and bit planes
    mid-call.  The tensor is marked in use on the launch stream, so a workspace
    that is replaced (grown) is not recycled while queued kernels still use it."""
    torch = require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    need = int(_lib.load().ef_workspace_bytes(batch, height, width))
    cache = getattr(_ws_local, "cache", None)
    if cache is None:
        cache = _ws_local.cache = {}
    key = (dev.index, int(st.cuda_stream))
    ws = cache.get(key)
    if ws is None or ws.numel() < need:
        if ws is not None:
            ws.record_stream(st)  # freed only after the work already queued on `st`
        with torch.cuda.stream(st):  # allocated on the launch stream's pool
            ws = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
        cache[key] = ws
    return ws


def new_workspace(batch: int, height: int, width: int, device=None):
    torch = require_cuda()
    need = int(_lib.load().ef_workspace_bytes(batch, height, width))
    return torch.empty(max(need, 1), dtype=torch.uint8, device=device or "cuda")


def _frames(t, dtype_name: str):
    if t.dim() == 2:
        t = t.unsqueeze(0)
    if t.dim() != 3:
        raise ValueError(f"expected (batch, H, W) or (H, W), got shape {tuple(t.shape)}")
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if str(t.dtype) != dtype_name:
        raise ValueError(f"expected {dtype_name}, got {t.dtype}")
    return t.contiguous()


def canny_u8(frames, weights, low: float, high: float, labels=None, final=None, ws=None, stream=None):
    """Fused Canny on u8 frames already in HBM -> (labels u8, final u8)."""
    torch = require_cuda()
    x = _frames(frames, "torch.uint8")
    b, h, w = x.shape
    labels = torch.empty_like(x) if labels is None else labels
    final = torch.empty_like(x) if final is None else final
    ws = workspace(b, h, w, x.device, stream) if ws is None else ws
    _, wp, r = host_weights(weights)
    rc = _lib.load().ef_canny_u8(_ptr(x), b, h, w, wp, r, float(low), float(high), _ptr(labels), _ptr(final),
                                 _ptr(ws), ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "ef_canny_u8")
    return labels, final


def canny_u8_timed(frames, weights, low: float, high: float):
    """canny_u8 on the current stream with device time per phase (CUDA events
    the library records around the classifier and its fix-ups): returns
    (labels, final, classify_ms, hysteresis_ms).  Synchronises."""
    torch = require_cuda()
    lib = _lib.load()
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(st)  # torch creates its events on first record
    ev[1].record(st)
    _lib.check(lib.ef_set_classify_events(ev[0].cuda_event, ev[1].cuda_event), "ef_set_classify_events")
    try:
        labels, final = canny_u8(frames, weights, low, high, stream=st)
    finally:
        _lib.check(lib.ef_set_classify_events(None, None), "ef_set_classify_events")
    ev[2].record(st)
    ev[2].synchronize()
    return labels, final, ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])


def classify_u8(frames, weights, low: float, high: float, labels=None, ws=None, stream=None):
    torch = require_cuda()
    x = _frames(frames, "torch.uint8")
    b, h, w = x.shape
    labels = torch.empty_like(x) if labels is None else labels
    ws = workspace(b, h, w, x.device, stream) if ws is None else ws
    _, wp, r = host_weights(weights)
    rc = _lib.load().ef_classify_u8(_ptr(x), b, h, w, wp, r, float(low), float(high), _ptr(labels), _ptr(ws),
                                    ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "ef_classify_u8")
    return labels


def canny_f64(frames, weights, low: float, high: float, ws=None, stream=None):
    torch = require_cuda()
    x = _frames(frames, "torch.float64")
    b, h, w = x.shape
    labels = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    final = torch.empty_like(labels)
    ws = workspace(b, h, w, x.device, stream) if ws is None else ws
    _, wp, r = host_weights(weights)
    rc = _lib.load().ef_canny_f64(_ptr(x), b, h, w, wp, r, float(low), float(high), _ptr(labels), _ptr(final),
                                  _ptr(ws), ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "ef_canny_f64")
    return labels, final


def trace_edges_u8(labels, final=None, ws=None, stream=None):
    torch = require_cuda()
    x = _frames(labels, "torch.uint8")
    b, h, w = x.shape
    final = torch.empty_like(x) if final is None else final
    ws = workspace(b, h, w, x.device, stream) if ws is None else ws
    rc = _lib.load().ef_trace_edges(_ptr(x), b, h, w, _ptr(final), _ptr(ws), ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "ef_trace_edges")
    return final


def stages_f64(frame, weights, low: float, high: float, stream=None) -> dict:
    """Every float64 intermediate of one frame (u8 or float64 CUDA tensor)."""
    torch = require_cuda()
    if frame.dim() != 2 or not frame.is_cuda:
        raise ValueError("expected one (H, W) CUDA frame")
    x = frame.contiguous()
    h, w = x.shape
    dev = x.device
    out = {k: torch.empty((h, w), dtype=torch.float64, device=dev)
           for k in ("blurred", "gx", "gy", "magnitude", "thinned")}
    out["orientation"] = torch.empty((h, w), dtype=torch.int64, device=dev)
    out["labels"] = torch.empty((h, w), dtype=torch.uint8, device=dev)
    src8 = _ptr(x) if x.dtype == torch.uint8 else None
    src64 = _ptr(x) if x.dtype == torch.float64 else None
    if src8 is None and src64 is None:
        raise ValueError(f"unsupported dtype {x.dtype}")
    _, wp, r = host_weights(weights)
    rc = _lib.load().ef_stages_f64(src8, src64, h, w, wp, r, float(low), float(high), _ptr(out["blurred"]),
                                   _ptr(out["gx"]), _ptr(out["gy"]), _ptr(out["magnitude"]),
                                   _ptr(out["orientation"]), _ptr(out["thinned"]), _ptr(out["labels"]),
                                   _stream_ptr(stream))
    _lib.check(rc, "ef_stages_f64")
    return out


def blur_f64(frame, weights, stream=None):
    torch = require_cuda()
    x = frame.contiguous()
    h, w = x.shape
    blurred = torch.empty((h, w), dtype=torch.float64, device=x.device)
    _, wp, r = host_weights(weights)
    src8 = _ptr(x) if x.dtype == torch.uint8 else None
    src64 = _ptr(x) if x.dtype == torch.float64 else None
    rc = _lib.load().ef_stages_f64(src8, src64, h, w, wp, r, 0.0, 0.0, _ptr(blurred), None, None, None, None,
                                   None, None, _stream_ptr(stream))
    _lib.check(rc, "ef_stages_f64")
    return blurred


def thinned_max(frame, weights, stream=None) -> float:
    torch = require_cuda()
    x = frame.contiguous()
    h, w = x.shape
    out = torch.zeros(1, dtype=torch.float64, device=x.device)
    _, wp, r = host_weights(weights)
    src8 = _ptr(x) if x.dtype == torch.uint8 else None
    src64 = _ptr(x) if x.dtype == torch.float64 else None
    rc = _lib.load().ef_thinned_max(src8, src64, h, w, wp, r, _ptr(out), _stream_ptr(stream))
    _lib.check(rc, "ef_thinned_max")
    return float(out.item())


def nms_f64(magnitude, orientation, stream=None):
    torch = require_cuda()
    h, w = magnitude.shape
    thin = torch.empty_like(magnitude)
    rc = _lib.load().ef_nms_f64(_ptr(magnitude), _ptr(orientation), h, w, _ptr(thin), _stream_ptr(stream))
    _lib.check(rc, "ef_nms_f64")
    return thin


def threshold_f64(thinned, low: float, high: float, stream=None):
    torch = require_cuda()
    labels = torch.empty(thinned.shape, dtype=torch.uint8, device=thinned.device)
    rc = _lib.load().ef_double_threshold_f64(_ptr(thinned), thinned.numel(), float(low), float(high),
                                             _ptr(labels), _stream_ptr(stream))
    _lib.check(rc, "ef_double_threshold_f64")
    return labels


def quantize_f64(gx, gy, stream=None):
    torch = require_cuda()
    ori = torch.empty(gx.shape, dtype=torch.int64, device=gx.device)
    rc = _lib.load().ef_quantize_f64(_ptr(gx), _ptr(gy), gx.numel(), _ptr(ori), _stream_ptr(stream))
    _lib.check(rc, "ef_quantize_f64")
    return ori


def laplacian_f64(frame, stream=None):
    torch = require_cuda()
    h, w = frame.shape
    out = torch.empty_like(frame)
    rc = _lib.load().ef_laplacian_f64(_ptr(frame), h, w, _ptr(out), _stream_ptr(stream))
    _lib.check(rc, "ef_laplacian_f64")
    return out


def canny_u8_host(frames: np.ndarray, weights, low: float, high: float, labels: np.ndarray | None = None,
                  final: np.ndarray | None = None, device: int | None = None, edges_only: bool = False):
    """Host buffers in, host buffers out: the e2e entry point (H2D + kernels + D2H
    pipelined inside the library).  Pinned (page-locked) buffers give full
    PCIe bandwidth; pageable ones work but are staged.  edges_only=True returns
    (None, final): the labels stay on the device and the edge map comes back at
    1 bit per pixel."""
    torch = require_cuda()
    arr = np.asarray(frames)
    if arr.dtype != np.uint8:
        raise ValueError(f"expected uint8 frames, got {arr.dtype}")
    squeeze = arr.ndim == 2
    x = np.ascontiguousarray(arr[None] if squeeze else arr)
    b, h, w = x.shape
    if edges_only and labels is not None:
        raise ValueError("edges_only=True takes no labels array")
    labels = None if edges_only else (np.empty(x.shape, np.uint8) if labels is None else labels)
    final = np.empty(x.shape, np.uint8) if final is None else final
    for name, a in (("labels", labels), ("final", final)):
        if a is None:
            continue
        if (a.shape != x.shape or a.dtype != np.uint8 or not a.flags.c_contiguous or not a.flags.writeable):
            raise ValueError(f"{name} must be a writeable C-contiguous uint8 array of shape {x.shape}")
    _, wp, r = host_weights(weights)
    dev = torch.cuda.current_device() if device is None else int(device)
    rc = _lib.load().ef_canny_u8_host(x.ctypes.data, b, h, w, wp, r, float(low), float(high),
                                      None if labels is None else labels.ctypes.data, final.ctypes.data, dev)
    _lib.check(rc, "ef_canny_u8_host")
    if squeeze:
        return (None if labels is None else labels[0]), final[0]
    return labels, final


def canny_u8_host_ptr(src_ptr: int, batch: int, height: int, width: int, weights, low: float, high: float,
                      labels_ptr: int, final_ptr: int, device: int = 0) -> None:
    """Raw-pointer form of canny_u8_host (pinned torch CPU tensors in bench.py);
    labels_ptr 0 / None = edges only."""
    _, wp, r = host_weights(weights)
    rc = _lib.load().ef_canny_u8_host(src_ptr, batch, height, width, wp, r, float(low), float(high),
                                      labels_ptr or None, final_ptr, device)
    _lib.check(rc, "ef_canny_u8_host")


def read_stats(ws, stream=None) -> dict:
    st = _lib.EfStats()
    rc = _lib.load().ef_read_stats(_ptr(ws), ws.numel(), _stream_ptr(stream), ctypes.byref(st))
    _lib.check(rc, "ef_read_stats")
    return st.as_dict()


def set_block_tile_threshold(tiles_per_sm: int) -> None:
    """Hysteresis tuning: block-per-tile at or below this many tiles per SM (0: never)."""
    _lib.check(_lib.load().ef_set_block_tile_threshold(int(tiles_per_sm)), "ef_set_block_tile_threshold")


def set_tile_reach(on: bool) -> None:
    """Hysteresis tuning: tile-local reach before the tile union-find (default on)."""
    _lib.check(_lib.load().ef_set_tile_reach(1 if on else 0), "ef_set_tile_reach")


def read_paths(ws, stream=None) -> dict:
    """Capacity fallbacks the last call on `ws` took (ef_read_paths)."""
    out = (ctypes.c_uint32 * 4)()
    _lib.check(_lib.load().ef_read_paths(_ptr(ws), ws.numel(), _stream_ptr(stream), out), "ef_read_paths")
    return {"fix_overflow": bool(out[0]), "pending_overflow": bool(out[1]), "dense_tiles": int(out[2]),
            "node_overflow": bool(out[3])}


def reset_stats(ws, stream=None) -> None:
    rc = _lib.load().ef_reset_stats(_ptr(ws), ws.numel(), _stream_ptr(stream))
    _lib.check(rc, "ef_reset_stats")
