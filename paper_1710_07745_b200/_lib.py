"""ctypes binding of libedgeforge_b200.so (include/edgeforge_b200.h).

The library is built in-tree by ``paper_1710_07745_b200.build``.  There is no
CPU fallback: if the library or a CUDA device is missing, every compute entry
point raises.  Status codes map to the reference's exceptions: EF_EINVAL ->
ValueError (the reference raises ValueError for invalid parameters),
anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libedgeforge_b200.so")

EF_OK, EF_EINVAL, EF_ECUDA, EF_ENOMEM = 0, -1, -2, -3
MAX_RADIUS = 15


class EfPgmInfo(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int32), ("height", ctypes.c_int32), ("maxval", ctypes.c_int32),
                ("binary", ctypes.c_int32), ("payload_offset", ctypes.c_int64)]


class EfStats(ctypes.Structure):
    _fields_ = [
        ("fixups", ctypes.c_int64),
        ("ambiguous", ctypes.c_int64),
        ("border_nodes", ctypes.c_int64),
        ("pending_tiles", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


P, I32, I64, D, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_size_t
_SIGNATURES = {
    "ef_abi_version": ([], ctypes.c_int),
    "ef_last_error": ([], ctypes.c_char_p),
    "ef_workspace_bytes": ([I64, I32, I32], SZ),
    "ef_reset_stats": ([P, SZ, P], ctypes.c_int),
    "ef_read_stats": ([P, SZ, P, ctypes.POINTER(EfStats)], ctypes.c_int),
    "ef_set_classify_events": ([P, P], ctypes.c_int),
    "ef_host_f64_to_u8": ([P, I64, P], ctypes.c_int),
    "ef_canny_u8": ([P, I64, I32, I32, P, I32, D, D, P, P, P, SZ, P], ctypes.c_int),
    "ef_canny_f64": ([P, I64, I32, I32, P, I32, D, D, P, P, P, SZ, P], ctypes.c_int),
    "ef_classify_u8": ([P, I64, I32, I32, P, I32, D, D, P, P, SZ, P], ctypes.c_int),
    "ef_trace_edges": ([P, I64, I32, I32, P, P, SZ, P], ctypes.c_int),
    "ef_stages_f64": ([P, P, I32, I32, P, I32, D, D, P, P, P, P, P, P, P, P], ctypes.c_int),
    "ef_thinned_max": ([P, P, I32, I32, P, I32, P, P], ctypes.c_int),
    "ef_nms_f64": ([P, P, I32, I32, P, P], ctypes.c_int),
    "ef_double_threshold_f64": ([P, I64, D, D, P, P], ctypes.c_int),
    "ef_quantize_f64": ([P, P, I64, P, P], ctypes.c_int),
    "ef_laplacian_f64": ([P, I32, I32, P, P], ctypes.c_int),
    "ef_canny_u8_host": ([P, I64, I32, I32, P, I32, D, D, P, P, I32], ctypes.c_int),
    "ef_band_halo_rows": ([I32], ctypes.c_int),
    "ef_band_canny_u8": ([P, I32, I32, I32, I32, P, I32, D, D, P, P, P, SZ, P], ctypes.c_int),
    "ef_band_trace": ([P, I32, I32, P, P, SZ, P], ctypes.c_int),
    "ef_band_canny_u8_peer": ([P, P, I32, P, I32, I32, I32, I32, I32, P, I32, D, D, P, P, P, SZ, P], ctypes.c_int),
    "ef_ipc_export": ([P, P, ctypes.POINTER(ctypes.c_uint64)], ctypes.c_int),
    "ef_ipc_open": ([P, ctypes.c_uint64, ctypes.POINTER(P), ctypes.POINTER(P)], ctypes.c_int),
    "ef_ipc_close": ([P], ctypes.c_int),
    "ef_pgm_last_error": ([], ctypes.c_char_p),
    "ef_pgm_parse": ([P, SZ, P, ctypes.POINTER(I64)], ctypes.c_int),
    "ef_pgm_decode_u8": ([P, SZ, P, P, ctypes.POINTER(I64)], ctypes.c_int),
    "ef_pgm_header": ([I32, I32, ctypes.c_char_p, SZ], ctypes.c_int),
    "ef_pgm_encode_edges": ([P, I64, P, P], ctypes.c_int),
    "ef_band_edges": ([P, SZ, I32, I32, P, P, P], ctypes.c_int),
    "ef_band_merge": ([I32, I32, P, P, P], ctypes.c_int),
    "ef_band_merge_scratch_bytes": ([I32, I32], SZ),
    "ef_read_paths": ([P, SZ, P, P], ctypes.c_int),
    "ef_set_block_tile_threshold": ([I32], ctypes.c_int),
    "ef_set_tile_reach": ([I32], ctypes.c_int),
    "ef_band_merge_device": ([I32, I32, P, P, P, P, SZ, P], ctypes.c_int),
    "ef_band_finalize": ([P, I32, I32, P, P, P, SZ, P], ctypes.c_int),
}

_lib = None


def load():
    """Load the in-tree library (build it first if this is a source checkout)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build

        _build.build()
    path = os.environ.get("EF_LIB_OVERRIDE", LIB_PATH)  # experiment builds (tools/); default in-tree
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc == EF_OK:
        return
    msg = load().ef_last_error().decode(errors="replace")
    if rc == EF_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"{what}: {msg} (status {rc})")


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)
