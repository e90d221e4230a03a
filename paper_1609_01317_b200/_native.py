"""ctypes binding of the C ABI declared in include/voxelcast_b200.h.

The library is built in-tree by paper_1609_01317_b200/build.py
(nvcc, sm_100a).  There is no fallback: if the library is missing or no
CUDA device is visible, every compute call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

# VC_LIB overrides the library path (development variants, tools/kbench.py)
_LIB_PATH = Path(os.environ.get("VC_LIB") or Path(__file__).resolve().parent / "_lib" / "libvoxelcast_b200.so")

VC_OK = 0
VC_ERR_INVALID = 1
VC_ERR_CUDA = 2
VC_ERR_NOMEM = 3
VC_ERR_UNSUPPORTED = 4

VC_U8, VC_U16, VC_F32 = 0, 1, 2
VC_GRAD_TAPS, VC_GRAD_VOLUME = 0, 1
VC_SAMPLER_SOFTWARE, VC_SAMPLER_TEXTURE = 0, 1
MAX_LUT = 64
NUM_COUNTERS = 6

DTYPE_CODES = {np.dtype(np.uint8): VC_U8, np.dtype(np.uint16): VC_U16, np.dtype(np.float32): VC_F32}

# every symbol the header declares (tests check the library exports them)
EXPORTS = (
    "vc_abi_version", "vc_render_params_size", "vc_last_error", "vc_device_count",
    "vc_volume_create", "vc_volume_create_device", "vc_volume_destroy", "vc_volume_data",
    "vc_volume_set_octree",
    "vc_gradient_prepass", "vc_gradient_volume", "vc_gradient_prepass_into",
    "vc_render", "vc_render_profiled", "vc_render_host", "vc_render_to_peers", "vc_signal_flags", "vc_wait_flags",
    "vc_ipc_handle", "vc_ipc_open", "vc_ipc_close", "vc_device_alloc", "vc_device_free",
    "vc_memcpy_to_host", "vc_sample_peak", "vc_sample_peak_texture", "vc_encode_png",
    "vc_sample_points", "vc_gradient_points",
    "vc_box_interval_rays", "vc_first_hit_rays", "vc_bisect_rays",
)

_d3 = ctypes.c_double * 3


class RenderParams(ctypes.Structure):
    """Mirror of vc_render_params."""

    _fields_ = [
        ("eye", _d3), ("right", _d3), ("up", _d3), ("forward", _d3),
        ("half_w", ctypes.c_double), ("half_h", ctypes.c_double),
        ("width", ctypes.c_int32), ("height", ctypes.c_int32),
        ("band_rows", ctypes.c_int32), ("band_first", ctypes.c_int32),
        ("band_step", ctypes.c_int32), ("lut_n", ctypes.c_int32),
        ("clip_lo", _d3), ("clip_hi", _d3),
        ("light_pos", _d3), ("light_col", _d3),
        ("t_low", ctypes.c_double), ("t_high", ctypes.c_double),
        ("lut_hu", ctypes.c_double * MAX_LUT),
        ("lut_rgba", (ctypes.c_double * 4) * MAX_LUT),
        ("mu_water", ctypes.c_double),
        ("op", ctypes.c_int32), ("interp", ctypes.c_int32),
        ("mode", ctypes.c_int32), ("refine_iters", ctypes.c_int32),
        ("coarse", ctypes.c_double), ("fine", ctypes.c_double),
        ("bg", ctypes.c_double * 4),
        ("skip_empty", ctypes.c_int32), ("grad_source", ctypes.c_int32),
        ("use_adaptive", ctypes.c_int32), ("adapt_jump", ctypes.c_int32),
        ("detail_eps", ctypes.c_double),
        ("sampler", ctypes.c_int32), ("row_end", ctypes.c_int32),
    ]


class PeerFramesDesc(ctypes.Structure):
    """Mirror of vc_peer_frames."""

    _fields_ = [
        ("d_frames", ctypes.c_void_p), ("d_done", ctypes.c_void_p), ("frame_bytes", ctypes.c_uint64),
        ("n", ctypes.c_int32), ("self", ctypes.c_int32), ("dest", ctypes.c_int32), ("seq", ctypes.c_uint32),
    ]


MAX_PEERS = 64


class OctreeDesc(ctypes.Structure):
    """Mirror of vc_octree_desc."""

    _fields_ = [
        ("levels", ctypes.c_int32),
        ("dims", ctypes.POINTER(ctypes.c_int32)), ("axis_map", ctypes.POINTER(ctypes.c_int32)),
        ("ivl_off", ctypes.POINTER(ctypes.c_int32)), ("ivl", ctypes.POINTER(ctypes.c_int32)),
        ("box_off", ctypes.POINTER(ctypes.c_int64)), ("state", ctypes.POINTER(ctypes.c_uint8)),
        ("srange", ctypes.POINTER(ctypes.c_double)),
        ("n_ivl", ctypes.c_int64), ("n_boxes", ctypes.c_int64),
    ]


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def library_path() -> Path:
    return _LIB_PATH


def load(build_if_missing: bool = True):
    """Load the sm_100a library (building it in-tree if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not _LIB_PATH.exists():
            if not build_if_missing:
                raise NativeError(f"native library missing: {_LIB_PATH} (run __graft_entry__.build())")
            from .build import build

            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        vp, i64, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        sig = {
            "vc_abi_version": ([], ctypes.c_int),
            "vc_render_params_size": ([], ctypes.c_int),
            "vc_last_error": ([], ctypes.c_char_p),
            "vc_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
            "vc_volume_create": ([ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_int, dp, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_volume_create_device": ([ctypes.c_int, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, dp, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_volume_destroy": ([vp], ctypes.c_int),
            "vc_volume_data": ([vp, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_volume_set_octree": ([vp, ctypes.POINTER(OctreeDesc)], ctypes.c_int),
            "vc_gradient_prepass": ([vp, ctypes.c_int, vp], ctypes.c_int),
            "vc_gradient_volume": ([vp, ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_gradient_prepass_into": ([vp, ctypes.c_int, vp, vp], ctypes.c_int),
            "vc_render": ([vp, ctypes.POINTER(RenderParams), vp, vp, vp], ctypes.c_int),
            "vc_render_profiled": ([vp, ctypes.POINTER(RenderParams), vp, vp, vp,
                                    ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
            "vc_render_to_peers": ([vp, ctypes.POINTER(RenderParams), ctypes.POINTER(PeerFramesDesc), vp, vp],
                                   ctypes.c_int),
            "vc_signal_flags": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, vp], ctypes.c_int),
            "vc_wait_flags": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, vp, vp],
                              ctypes.c_int),
            "vc_device_alloc": ([ctypes.c_int, ctypes.c_size_t, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_device_free": ([vp], ctypes.c_int),
            "vc_sample_peak": ([ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "vc_sample_peak_texture": ([ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
            "vc_encode_png": ([vp, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_size_t,
                               ctypes.POINTER(ctypes.c_size_t)], ctypes.c_int),
            "vc_memcpy_to_host": ([vp, vp, ctypes.c_size_t, vp], ctypes.c_int),
            "vc_ipc_handle": ([vp, vp], ctypes.c_int),
            "vc_ipc_open": ([ctypes.c_int, vp, ctypes.POINTER(vp)], ctypes.c_int),
            "vc_ipc_close": ([vp], ctypes.c_int),
            "vc_render_host": ([vp, ctypes.POINTER(RenderParams), vp, u64p,
                                ctypes.POINTER(ctypes.c_float)], ctypes.c_int),
            "vc_sample_points": ([vp, ctypes.c_int, dp, i64, dp], ctypes.c_int),
            "vc_gradient_points": ([vp, ctypes.c_int, dp, i64, dp], ctypes.c_int),
            "vc_box_interval_rays": ([dp, i64, dp, dp, dp], ctypes.c_int),
            "vc_first_hit_rays": ([vp, dp, i64, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int, dp, u64p], ctypes.c_int),
            "vc_bisect_rays": ([vp, dp, i64, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                                ctypes.c_int, dp, u64p], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name, None)
            if fn is None:  # an older library variant (A/B tools); tests check the exports
                continue
            fn.argtypes = args
            fn.restype = res
        if hasattr(L, "vc_checked_violations"):  # the bounds-checked variant (_lib/checked)
            L.vc_checked_violations.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
            L.vc_checked_violations.restype = ctypes.c_ulonglong
        if L.vc_render_params_size() != ctypes.sizeof(RenderParams):
            raise NativeError("vc_render_params layout mismatch between header and binding")
        _lib = L
        return L


def check(rc: int) -> None:
    """Map a vc_status to the reference's exception types."""
    if rc == VC_OK:
        return
    msg = (_lib.vc_last_error() or b"").decode(errors="replace") if _lib else ""
    if rc == VC_ERR_INVALID:
        raise ValueError(msg)
    if rc == VC_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == VC_ERR_NOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def device_count() -> int:
    L = load()
    n = ctypes.c_int(0)
    check(L.vc_device_count(ctypes.byref(n)))
    return int(n.value)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
