"""voxelcast._kernels on the B200 path: the reference's kernel layer
(/root/reference/pkg/src/voxelcast/_kernels.py) with the same entry-point
names, argument lists, integer codes and return shapes, each one a call
through the C ABI (include/voxelcast_b200.h) into the sm_100a library.

The reference's kernels take the raw voxel array (`data`, x fastest) plus
its dims on every call; here the array is uploaded once and kept resident
in HBM while it lives (read-only arrays -- a `Volume.data` always is; a
writable array is re-uploaded on every call because the caller may have
changed it).  There is no CPU fallback: without the library or a device
every call raises.

  sample_any / sample_nearest / sample_linear / sample_trilinear
                        (_kernels.py:66-127)  -> vc_sample_points
  grad_raw              (_kernels.py:140-177) -> vc_gradient_points
  box_interval          (_kernels.py:206-224) -> vc_box_interval_rays
  render_tile           (_kernels.py:582-797) -> vc_render_host, rows [y0, y1)
                                                 (band_rows 1, row_end = y1)

render_tile is the band entry raycast.render_frame fans out to a thread
pool (raycast.py:476-505): with this module in place of the numba one the
reference's own host code renders on the GPU unchanged (INTEGRATION.md
Option B, tests/test_dropin_gpu.py).  Its `use_octree` runs the
output-neutral macrocell skipping; with 0 inside the window, or with
`use_adaptive`, the octree the caller passes (reference flat form) is
replayed on the device, as the reference walks it.  `stack`, `seg0` and
`seg1` are the reference's per-band scratch and are not touched.
"""

from __future__ import annotations

import ctypes
import math
import threading
import weakref

import numpy as np

from paper_1609_01317_b200 import _native
from paper_1609_01317_b200.octree import device_arrays_from_flat
from paper_1609_01317_b200.volume import DeviceVolume

INTERP_NEAREST = 0
INTERP_LINEAR = 1
INTERP_TRILINEAR = 2

OP_CENTRAL = 0
OP_SOBEL3D = 1
OP_ZUCKER_HUMMEL = 2

MODE_SURFACE = 0
MODE_COMPOSITED = 1

GRAD_EPS = 1e-8
OPAQUE_ALPHA = 1.0 - 1e-6
MIN_REMAINING = 0.01

# volume fetches per gradient evaluation, indexed by operator code
GRAD_SAMPLES = (6, 26, 26)

_NATIVE = {np.dtype(np.uint8), np.dtype(np.uint16), np.dtype(np.float32)}


class _Grid:
    """What DeviceVolume reads off a Volume."""

    def __init__(self, data: np.ndarray, dims, spacing):
        self.data = data
        self.dims = dims
        self.spacing = spacing


def _storage(data) -> np.ndarray:
    """The flat array in a storage type the device reads (u8 / u16 / f32),
    values unchanged; anything that would change a value raises."""
    a = np.asarray(data).ravel()
    if a.dtype in _NATIVE:
        return a
    if a.dtype.kind in "iu" and (a.size == 0 or (a.min() >= 0 and a.max() <= 65535)):
        return a.astype(np.uint16)
    f = a.astype(np.float32)
    if np.array_equal(f.astype(a.dtype), a):
        return f
    raise ValueError(f"voxel values of dtype {a.dtype} are not representable in uint8/uint16/float32 storage")


_cache: dict[int, tuple] = {}  # id(data) -> (weakref(data), {spacing: DeviceVolume})
_cache_lock = threading.Lock()


def _device(data, nx, ny, nz, spacing=(1.0, 1.0, 1.0), device: int = 0) -> DeviceVolume:
    """The resident device copy of `data` (dims nx, ny, nz) for `spacing`."""
    dims = (int(nx), int(ny), int(nz))
    sp = tuple(float(s) for s in spacing)
    arr = np.asarray(data)
    if arr.size != dims[0] * dims[1] * dims[2]:
        raise ValueError(f"data holds {arr.size} voxels, dims {dims} need {dims[0] * dims[1] * dims[2]}")
    if arr.flags.writeable or not isinstance(data, np.ndarray):
        return DeviceVolume(_Grid(_storage(arr), dims, sp), device)  # uncached: may change
    key = id(data)
    with _cache_lock:
        ent = _cache.get(key)
        if ent is not None and ent[0]() is not data:
            ent = None  # a recycled id
        if ent is None:
            ent = (weakref.ref(data), {})
            _cache[key] = ent

            def _drop(k=key, e=ent):
                with _cache_lock:
                    if _cache.get(k) is e:
                        del _cache[k]
                for dv in e[1].values():
                    dv.close()

            weakref.finalize(data, _drop)
        per = ent[1]
        dv = per.get((sp, dims, device))
        if dv is None:
            dv = per[(sp, dims, device)] = DeviceVolume(_Grid(_storage(arr), dims, sp), device)
        return dv


def _any_device(data, nx, ny, nz) -> DeviceVolume:
    """A resident copy for a point query (spacing plays no part there)."""
    with _cache_lock:
        ent = _cache.get(id(data))
        if ent is not None and ent[0]() is data:
            for (sp, dims, dev), dv in ent[1].items():
                if dims == (int(nx), int(ny), int(nz)):
                    return dv
    return _device(data, nx, ny, nz)


# ---------------------------------------------------------------- point kernels

def lerp(f0, f1, t):
    """f0 + (f1 - f0) * t (_kernels.py:35-37)."""
    return f0 + (f1 - f0) * t


def sample_any(data, nx, ny, nz, x, y, z, interp):
    """Field value at voxel-space (x, y, z); 0 outside [0, n-1]^3 (_kernels.py:118-127)."""
    if interp not in (INTERP_NEAREST, INTERP_LINEAR, INTERP_TRILINEAR):
        raise ValueError(f"interp must be 0, 1 or 2, got {interp}")
    dv = _any_device(data, nx, ny, nz)
    pts = np.array([[float(x), float(y), float(z)]], np.float64)
    out = np.empty(1, np.float64)
    _native.check(_native.load().vc_sample_points(dv.handle, int(interp), _native.dptr(pts), 1,
                                                  _native.dptr(out)))
    return float(out[0])


def sample_nearest(data, nx, ny, nz, x, y, z):
    return sample_any(data, nx, ny, nz, x, y, z, INTERP_NEAREST)


def sample_linear(data, nx, ny, nz, x, y, z):
    return sample_any(data, nx, ny, nz, x, y, z, INTERP_LINEAR)


def sample_trilinear(data, nx, ny, nz, x, y, z):
    return sample_any(data, nx, ny, nz, x, y, z, INTERP_TRILINEAR)


def grad_raw(data, nx, ny, nz, x, y, z, op):
    """Raw (unnormalized) gradient (gx, gy, gz) of operator `op` at a
    voxel-space point, taps trilinear with 0 outside (_kernels.py:140-177)."""
    if op not in (OP_CENTRAL, OP_SOBEL3D, OP_ZUCKER_HUMMEL):
        raise ValueError(f"op must be 0, 1 or 2, got {op}")
    dv = _any_device(data, nx, ny, nz)
    pts = np.array([[float(x), float(y), float(z)]], np.float64)
    out = np.empty((1, 3), np.float64)
    _native.check(_native.load().vc_gradient_points(dv.handle, int(op), _native.dptr(pts), 1,
                                                    _native.dptr(out)))
    return float(out[0, 0]), float(out[0, 1]), float(out[0, 2])


def normalize3(gx, gy, gz, eps):
    """g / |g|, or exactly 0 when |g| <= eps (_kernels.py:180-185): three
    doubles of host glue, the same IEEE operations in the same order."""
    n = math.sqrt(gx * gx + gy * gy + gz * gz)
    if n <= eps:
        return 0.0, 0.0, 0.0
    return gx / n, gy / n, gz / n


def box_interval(org, dirv, lo, hi):
    """(hit, t0, t1) of the slab test (_kernels.py:206-224)."""
    rays = np.ascontiguousarray(np.concatenate([np.asarray(org, np.float64).ravel()[:3],
                                                np.asarray(dirv, np.float64).ravel()[:3]])[None, :])
    out = np.empty((1, 3), np.float64)
    lo = np.ascontiguousarray(np.asarray(lo, np.float64).ravel()[:3])
    hi = np.ascontiguousarray(np.asarray(hi, np.float64).ravel()[:3])
    _native.check(_native.load().vc_box_interval_rays(_native.dptr(rays), 1, _native.dptr(lo),
                                                      _native.dptr(hi), _native.dptr(out)))
    return bool(out[0, 0] != 0.0), float(out[0, 1]), float(out[0, 2])


# ---------------------------------------------------------------- the band renderer

def _attach_tree(dv: DeviceVolume, nbounds, sminmax, nchildren) -> None:
    """Put the caller's (reference-form) octree on the device volume, once
    per tree object (raycast.render_frame builds it once per frame or
    receives it, raycast.py:455-462)."""
    key = ("flat", id(nbounds), id(sminmax), id(nchildren), np.asarray(nbounds).shape)
    ref = getattr(dv, "_flat_refs", None)
    if ref is not None and getattr(dv, "_octree_key", None) == key and ref[0]() is nbounds:
        return
    dv.set_octree_arrays(device_arrays_from_flat(dv.dims, nbounds, sminmax, nchildren), key)
    try:
        dv._flat_refs = (weakref.ref(nbounds),)
    except TypeError:  # not weak-referenceable: never trust the key again
        dv._octree_key = None


def render_tile(data, nx, ny, nz, spacing, eye, right, upv, fwd, half_w, half_h, width, height,
                clip_lo, clip_hi, light_pos, light_col, t_low, t_high, lut_hu, lut_rgba, mu_water,
                op, interp, mode, coarse, fine, refine_iters, bg, use_octree, nbounds, sminmax,
                nchildren, use_adaptive, adapt_jump, detail_eps, y0, y1, out, counter, stack, seg0,
                seg1):
    """Render scanline rows [y0, y1) of the frame into out[y0:y1]
    (_kernels.py:582-797) with one device launch pair; counter[0] grows by
    the band's sample count (the reference's fetch convention)."""
    y0, y1 = int(y0), int(y1)
    width, height = int(width), int(height)
    if y1 <= y0:
        return
    if not (0 <= y0 and y1 <= height):
        raise ValueError(f"rows [{y0}, {y1}) outside the {height}-row frame")
    if out.shape[0] < height or out.shape[1] != width or out.shape[2] != 4 or out.dtype != np.uint8:
        raise ValueError(f"out must be ({height}, {width}, 4) uint8")
    dv = _device(data, nx, ny, nz, spacing)
    P = _native.RenderParams()
    P.eye[:] = [float(v) for v in eye]
    P.right[:] = [float(v) for v in right]
    P.up[:] = [float(v) for v in upv]
    P.forward[:] = [float(v) for v in fwd]
    P.half_w, P.half_h = float(half_w), float(half_h)
    P.width, P.height = width, height
    P.band_rows, P.band_first, P.band_step, P.row_end = 1, y0, 1, y1
    P.clip_lo[:] = [float(v) for v in clip_lo]
    P.clip_hi[:] = [float(v) for v in clip_hi]
    P.light_pos[:] = [float(v) for v in light_pos]
    P.light_col[:] = [float(v) for v in light_col]
    P.t_low, P.t_high = float(t_low), float(t_high)
    hu = np.asarray(lut_hu, np.float64).ravel()
    rgba = np.asarray(lut_rgba, np.float64).reshape(-1, 4)
    if not 1 <= len(hu) <= _native.MAX_LUT or len(rgba) != len(hu):
        raise ValueError(f"transfer tables must hold 1..{_native.MAX_LUT} breakpoints")
    P.lut_n = len(hu)
    for i in range(len(hu)):
        P.lut_hu[i] = float(hu[i])
        for c in range(4):
            P.lut_rgba[i][c] = float(rgba[i, c])
    P.mu_water = float(mu_water)
    P.op, P.interp, P.mode, P.refine_iters = int(op), int(interp), int(mode), int(refine_iters)
    P.coarse, P.fine = float(coarse), float(fine)
    P.bg[:] = [float(v) for v in bg]
    P.skip_empty = 1 if use_octree else 0
    P.grad_source = _native.VC_GRAD_TAPS
    P.sampler = _native.VC_SAMPLER_SOFTWARE
    P.use_adaptive = 1 if use_adaptive else 0
    P.adapt_jump = int(adapt_jump)
    P.detail_eps = float(detail_eps)
    if use_adaptive or (use_octree and float(t_low) <= 0.0 <= float(t_high)):
        _attach_tree(dv, nbounds, sminmax, nchildren)
    rows = out[y0:y1]
    dst = rows if rows.flags.c_contiguous else np.empty(rows.shape, np.uint8)
    counters = np.zeros(_native.NUM_COUNTERS, np.uint64)
    ms = ctypes.c_float(0.0)
    _native.check(_native.load().vc_render_host(
        dv.handle, ctypes.byref(P), dst.ctypes.data,
        counters.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), ctypes.byref(ms)))
    if dst is not rows:
        rows[...] = dst
    counter[0] += int(counters[0]) + int(counters[1]) * (1 + GRAD_SAMPLES[int(op)])
