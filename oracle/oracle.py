"""ctypes front end of the C parity oracle (TEST INFRASTRUCTURE ONLY).

Scenes are passed as plain dicts ("scene specs", see tests/golden/README.md)
so the same description drives the reference (when generating goldens),
this oracle and the B200 product path.

Host-side arithmetic restated here follows the reference exactly:
  * camera_basis        -> /root/reference/pkg/src/voxelcast/raycast.py:238-268
  * clip box            -> raycast.py:448-452
  * transfer tables     -> raycast.py:150-153
  * lattice stencils    -> _kernels.py:140-177 evaluated at integer points
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "vc_oracle.c"
_LIB_PATH = _HERE / "_build" / "libvcoracle.so"
MAX_LUT = 64

OP_CODES = {"central": 0, "sobel3d": 1, "zucker-hummel": 2}
INTERP_CODES = {"nearest": 0, "linear": 1, "trilinear": 2}
MODE_CODES = {"surface": 0, "composited": 1}
GRAD_SAMPLES = (6, 26, 26)
MAX_ELEVATION = 89.9


class _Params(ctypes.Structure):
    _fields_ = [
        ("spacing", ctypes.c_double * 3),
        ("eye", ctypes.c_double * 3),
        ("right", ctypes.c_double * 3),
        ("up", ctypes.c_double * 3),
        ("fwd", ctypes.c_double * 3),
        ("half_w", ctypes.c_double),
        ("half_h", ctypes.c_double),
        ("width", ctypes.c_int32),
        ("height", ctypes.c_int32),
        ("clip_lo", ctypes.c_double * 3),
        ("clip_hi", ctypes.c_double * 3),
        ("light_pos", ctypes.c_double * 3),
        ("light_col", ctypes.c_double * 3),
        ("t_low", ctypes.c_double),
        ("t_high", ctypes.c_double),
        ("lut_n", ctypes.c_int32),
        ("lut_hu", ctypes.c_double * MAX_LUT),
        ("lut_rgba", ctypes.c_double * (MAX_LUT * 4)),
        ("mu_water", ctypes.c_double),
        ("op", ctypes.c_int32),
        ("interp", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("coarse", ctypes.c_double),
        ("fine", ctypes.c_double),
        ("refine_iters", ctypes.c_int32),
        ("bg", ctypes.c_double * 4),
        ("use_adaptive", ctypes.c_int32),
        ("adapt_jump", ctypes.c_int32),
        ("detail_eps", ctypes.c_double),
        ("nbounds", ctypes.POINTER(ctypes.c_int32)),
        ("sminmax", ctypes.POINTER(ctypes.c_double)),
        ("nchildren", ctypes.POINTER(ctypes.c_int32)),
        ("use_octree", ctypes.c_int32),
    ]


def build(force: bool = False) -> Path:
    """Compile the oracle with strict IEEE float64 (no FMA contraction)."""
    if _LIB_PATH.exists() and not force and _LIB_PATH.stat().st_mtime >= _SRC.stat().st_mtime:
        return _LIB_PATH
    _LIB_PATH.parent.mkdir(parents=True, exist_ok=True)
    cmd = [
        "gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
        "-pthread", str(_SRC), "-o", str(_LIB_PATH), "-lm",
    ]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = build()
        L = ctypes.CDLL(str(path))
        dp = ctypes.POINTER(ctypes.c_double)
        L.vco_sample.restype = ctypes.c_double
        L.vco_sample.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_int]
        L.vco_sample_many.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, dp, ctypes.c_int64, ctypes.c_int, dp]
        L.vco_grad_raw_many.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, dp, ctypes.c_int64,
                                        ctypes.c_int, dp]
        L.vco_grad_volume.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_float), ctypes.c_int]
        L.vco_render.restype = ctypes.c_int64
        L.vco_render.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.POINTER(_Params), ctypes.c_int,
                                 ctypes.c_int, ctypes.POINTER(ctypes.c_uint8), ctypes.c_int]
        L.vco_box_interval.restype = ctypes.c_int
        L.vco_box_interval.argtypes = [dp, dp, dp, dp, dp]
        L.vco_first_hit.restype = ctypes.c_int
        L.vco_first_hit.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, dp, dp, dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int, dp,
                                    ctypes.POINTER(ctypes.c_int64)]
        L.vco_bisect.restype = ctypes.c_double
        L.vco_bisect.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, dp, dp, dp, ctypes.c_double, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_int64)]
        L.vco_params_size.restype = ctypes.c_int
        assert L.vco_params_size() == ctypes.sizeof(_Params), "oracle struct layout mismatch"
        _lib = L
    return _lib


# ---------------------------------------------------------------- volumes

_DTYPE_CODES = {np.dtype(np.uint8): 0, np.dtype(np.uint16): 1, np.dtype(np.float32): 2}


def _vol(arr: np.ndarray):
    arr = np.ascontiguousarray(arr)
    if arr.dtype not in _DTYPE_CODES:
        raise TypeError(f"oracle volumes are uint8/uint16/float32, got {arr.dtype}")
    nz, ny, nx = arr.shape
    return arr, _DTYPE_CODES[arr.dtype], nx, ny, nz


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def sample(arr, points, interp="trilinear") -> np.ndarray:
    """sample_any at voxel-space points (N,3) -> (N,)  (_kernels.py:118-127)."""
    arr, code, nx, ny, nz = _vol(arr)
    pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
    out = np.empty(len(pts), np.float64)
    lib().vco_sample_many(arr.ctypes.data, code, nx, ny, nz, _dp(pts), len(pts),
                          INTERP_CODES[interp], _dp(out))
    return out


def grad_raw(arr, points, op="central") -> np.ndarray:
    """Raw gradient (N,3) at voxel-space points (_kernels.py:140-177)."""
    arr, code, nx, ny, nz = _vol(arr)
    pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 3))
    out = np.empty((len(pts), 3), np.float64)
    lib().vco_grad_raw_many(arr.ctypes.data, code, nx, ny, nz, _dp(pts), len(pts),
                            OP_CODES[op], _dp(out))
    return out


def normalize3(g) -> np.ndarray:
    """normalize3 with EPS 1e-8 (_kernels.py:180-185)."""
    gx, gy, gz = (float(c) for c in g)
    n = math.sqrt(gx * gx + gy * gy + gz * gz)
    if n <= 1e-8:
        return np.zeros(3)
    return np.array([gx / n, gy / n, gz / n])


def grad_volume(arr, op="central", threads=None) -> np.ndarray:
    """grad_raw at every lattice point -> (nz,ny,nx,4) float32 (gx,gy,gz,value)."""
    arr, code, nx, ny, nz = _vol(arr)
    out = np.empty((nz, ny, nx, 4), np.float32)
    lib().vco_grad_volume(arr.ctypes.data, code, nx, ny, nz, OP_CODES[op],
                          out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                          int(threads or os.cpu_count() or 1))
    return out


def grad_volume_numpy(arr, op="central") -> np.ndarray:
    """Vectorised zero-padded 3x3x3 stencil in the reference's i->j->k term
    order, float64.  Bit-identical to grad_raw at lattice points (the
    trilinear tap at an integer point returns the voxel value exactly and
    out-of-range taps read 0, _kernels.py:52-64, :118-127).  Returns
    (nz,ny,nx,3) float64."""
    a = np.asarray(arr).astype(np.float64)
    nz, ny, nx = a.shape
    p = np.zeros((nz + 2, ny + 2, nx + 2))
    p[1:-1, 1:-1, 1:-1] = a

    def tap(i, j, k):
        return p[1 + k:1 + k + nz, 1 + j:1 + j + ny, 1 + i:1 + i + nx]

    g = np.zeros((nz, ny, nx, 3))
    if op == "central":
        g[..., 0] = tap(1, 0, 0) - tap(-1, 0, 0)
        g[..., 1] = tap(0, 1, 0) - tap(0, -1, 0)
        g[..., 2] = tap(0, 0, 1) - tap(0, 0, -1)
        return g

    def sw(u, v):
        if u == 0 and v == 0:
            return 6.0
        if u == 0 or v == 0:
            return 3.0
        return 1.0

    for i in (-1, 0, 1):
        for j in (-1, 0, 1):
            for k in (-1, 0, 1):
                if i == 0 and j == 0 and k == 0:
                    continue
                s = tap(i, j, k)
                if op == "sobel3d":
                    wx, wy, wz = i * sw(j, k), j * sw(i, k), k * sw(i, j)
                else:
                    inv = 1.0 / math.sqrt(float(i * i + j * j + k * k))
                    wx, wy, wz = i * inv, j * inv, k * inv
                g[..., 0] += wx * s
                g[..., 1] += wy * s
                g[..., 2] += wz * s
    return g


# ---------------------------------------------------------------- scenes

def camera_basis(cam: dict, width: int, height: int):
    """Restatement of raycast.camera_basis (raycast.py:238-268)."""
    eye = np.asarray(cam["eye"], np.float64)
    target = np.asarray(cam["target"], np.float64)
    az_deg = float(cam.get("azimuth", 0.0))
    el_deg = float(cam.get("elevation", 0.0))
    zoom = float(cam.get("zoom", 1.0))
    offset = eye - target
    if az_deg == 0.0 and el_deg == 0.0 and zoom == 1.0:
        eye_eff = eye.copy()
    else:
        r0 = float(np.linalg.norm(offset))
        az = math.atan2(offset[0], offset[2]) + math.radians(az_deg)
        el = math.asin(max(-1.0, min(1.0, offset[1] / r0))) + math.radians(el_deg)
        el = max(-math.radians(MAX_ELEVATION), min(math.radians(MAX_ELEVATION), el))
        dist = r0 / zoom
        eye_eff = target + dist * np.array(
            [math.cos(el) * math.sin(az), math.sin(el), math.cos(el) * math.cos(az)]
        )
    forward = target - eye_eff
    forward /= np.linalg.norm(forward)
    up = np.asarray(cam.get("up", (0.0, 1.0, 0.0)), np.float64)
    right = np.cross(forward, up)
    rn = np.linalg.norm(right)
    if rn < 1e-12:
        alt = np.array([1.0, 0.0, 0.0]) if abs(forward[0]) < 0.9 else np.array([0.0, 0.0, 1.0])
        right = np.cross(forward, alt)
        rn = np.linalg.norm(right)
    right /= rn
    up_cam = np.cross(right, forward)
    half_h = math.tan(math.radians(float(cam.get("fov_y", 60.0))) / 2.0)
    half_w = half_h * width / height
    return eye_eff, right, up_cam, forward, half_w, half_h


DEFAULT_CT = [
    (-1000.0, (0.0, 0.0, 0.0, 0.0)),
    (-100.0, (0.80, 0.30, 0.25, 0.35)),
    (500.0, (0.95, 0.93, 0.88, 1.0)),
    (1500.0, (1.0, 1.0, 1.0, 1.0)),
]


def default_scene_spec(dims, spacing=(1.0, 1.0, 1.0)) -> dict:
    """raycast.default_scene (raycast.py:421-428) as a spec dict."""
    ext = tuple(n * s for n, s in zip(dims, spacing))
    center = tuple(e / 2.0 for e in ext)
    dist = 1.1 * max(ext) / 2.0
    eye = (center[0], center[1], center[2] - dist)
    return {
        "camera": {"eye": eye, "target": center},
        "light": {"position": eye},
    }


def make_params(dims, spacing, spec: dict) -> _Params:
    s = spec.get("settings", {})
    width = int(s.get("width", 640))
    height = int(s.get("height", 480))
    eye, right, up, fwd, half_w, half_h = camera_basis(spec["camera"], width, height)
    ext = np.array([n * sp for n, sp in zip(dims, spacing)], np.float64)
    clip_lo = np.zeros(3)
    clip_hi = ext.copy()
    clip = spec.get("clip")
    if clip is not None:
        clip_lo = np.maximum(clip_lo, np.asarray(clip[0], np.float64))
        clip_hi = np.minimum(clip_hi, np.asarray(clip[1], np.float64))
    tf = spec.get("transfer") or {}
    points = tf.get("points", DEFAULT_CT)
    if len(points) > MAX_LUT:
        raise ValueError("too many transfer breakpoints for the oracle")
    win = spec.get("window", (500.0, 4095.0))
    light = spec["light"]
    P = _Params()
    P.spacing[:] = [float(x) for x in spacing]
    P.eye[:] = list(eye)
    P.right[:] = list(right)
    P.up[:] = list(up)
    P.fwd[:] = list(fwd)
    P.half_w = half_w
    P.half_h = half_h
    P.width = width
    P.height = height
    P.clip_lo[:] = list(clip_lo)
    P.clip_hi[:] = list(clip_hi)
    P.light_pos[:] = [float(x) for x in light["position"]]
    P.light_col[:] = [float(x) for x in light.get("color", (1.0, 1.0, 1.0))]
    P.t_low = float(win[0])
    P.t_high = float(win[1])
    P.lut_n = len(points)
    for i, (hu, rgba) in enumerate(points):
        P.lut_hu[i] = float(hu)
        for c in range(4):
            P.lut_rgba[4 * i + c] = float(rgba[c])
    P.mu_water = float(tf.get("mu_water", 1000.0))
    P.op = OP_CODES[s.get("operator", "central")]
    P.interp = INTERP_CODES[s.get("interpolation", "trilinear")]
    P.mode = MODE_CODES[s.get("mode", "surface")]
    P.coarse = float(s.get("coarse_step", 1.0))
    P.fine = float(s.get("fine_step", 0.125))
    P.refine_iters = int(s.get("refine_iters", 6))
    P.bg[:] = [float(x) for x in s.get("background", (0.0, 0.0, 0.0, 1.0))]
    return P


# ---------------------------------------------------------------- octree (adaptive mode)

def build_octree_flat(arr, min_block=4, max_depth=8):
    """Restatement of octree.build_octree + flat_arrays (octree.py:52-136):
    returns (nbounds (N,6) int32, sminmax (N,2) float64, nchildren (N,8)
    int32) in the reference's node order.  Plain recursion; for the small
    grids the tests use."""
    a = np.asarray(arr)
    nz, ny, nx = a.shape

    def ranges(lo, hi):
        blk = a[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        pad = a[max(lo[2] - 1, 0):min(hi[2] + 1, nz), max(lo[1] - 1, 0):min(hi[1] + 1, ny),
                max(lo[0] - 1, 0):min(hi[0] + 1, nx)]
        return int(blk.min()), int(blk.max()), int(pad.min()), int(pad.max())

    def make(lo, hi, depth):
        vmin, vmax, smin, smax = ranges(lo, hi)
        return {"lo": lo, "hi": hi, "vmin": vmin, "vmax": vmax, "smin": smin, "smax": smax,
                "depth": depth, "children": []}

    root = make((0, 0, 0), (nx, ny, nz), 0)
    stack = [root]
    while stack:
        node = stack.pop()
        ext = tuple(h - l for l, h in zip(node["lo"], node["hi"]))
        if node["vmin"] == node["vmax"] or max(ext) <= min_block or node["depth"] >= max_depth:
            continue
        cuts = []
        for ax in range(3):
            if ext[ax] >= 2:
                cuts.append([(node["lo"][ax], node["lo"][ax] + ext[ax] // 2),
                             (node["lo"][ax] + ext[ax] // 2, node["hi"][ax])])
            else:
                cuts.append([(node["lo"][ax], node["hi"][ax])])
        for zc in cuts[2]:
            for yc in cuts[1]:
                for xc in cuts[0]:
                    ch = make((xc[0], yc[0], zc[0]), (xc[1], yc[1], zc[1]), node["depth"] + 1)
                    node["children"].append(ch)
                    stack.append(ch)
    nodes = []
    stack = [root]
    while stack:
        n = stack.pop()
        nodes.append(n)
        stack.extend(n["children"])
    index = {id(n): i for i, n in enumerate(nodes)}
    nb = np.empty((len(nodes), 6), np.int32)
    sm = np.empty((len(nodes), 2), np.float64)
    ch = np.full((len(nodes), 8), -1, np.int32)
    for i, n in enumerate(nodes):
        nb[i, :3] = n["lo"]
        nb[i, 3:] = n["hi"]
        sm[i] = (n["smin"], n["smax"])
        for c, kid in enumerate(n["children"]):
            ch[i, c] = index[id(kid)]
    return nb, sm, ch


def render(arr, spacing, spec: dict, threads=None, rows=None, octree: bool = False):
    """Brute-force frame (render_frame(..., use_octree=False)); with
    settings.use_adaptive the reference's adaptive stride over its octree.
    octree=True honours settings.use_octree as the reference does: only the
    merged octree segments are marched (collect_segments), which changes the
    sample count (and, with use_adaptive, where the stride restarts).

    Returns (pixels (H,W,4) uint8, sample_count).  `rows` = (y0, y1)
    restricts the work to a row range (other rows stay zero)."""
    arr, code, nx, ny, nz = _vol(arr)
    P = make_params((nx, ny, nz), spacing, spec)
    s = spec.get("settings", {})
    keep = None
    use_octree = bool(octree and s.get("use_octree", True))
    if use_octree and not s.get("use_adaptive"):
        nb, sm, ch = build_octree_flat(arr, s.get("octree_min_block", 4), s.get("octree_max_depth", 8))
        keep = (nb, sm, ch)
        P.nbounds = nb.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        P.sminmax = sm.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        P.nchildren = ch.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    P.use_octree = 1 if use_octree else 0
    if s.get("use_adaptive"):
        nb, sm, ch = build_octree_flat(arr, s.get("octree_min_block", 4), s.get("octree_max_depth", 8))
        keep = (nb, sm, ch)
        P.use_adaptive = 1
        P.adapt_jump = int(s.get("adaptive_factor", 4))
        eps = s.get("detail_epsilon")
        if eps is None:
            eps = 0.01 * max(1, int(arr.max()) - int(arr.min()))
        P.detail_eps = float(eps)
        P.nbounds = nb.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        P.sminmax = sm.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        P.nchildren = ch.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    out = np.zeros((P.height, P.width, 4), np.uint8)
    y0, y1 = rows if rows is not None else (0, P.height)
    count = lib().vco_render(arr.ctypes.data, code, nx, ny, nz, ctypes.byref(P), int(y0),
                             int(y1), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                             int(threads or os.cpu_count() or 1))
    del keep
    return out, int(count)


def work_counts(arr, spacing, spec: dict, threads=None):
    """Brute-force work split: W ray samples and K shades,
    recovered from the CD and ZH sample counts like the reference would be
    measured: K = (count_ZH - count_CD)/20, W = count_CD - 6K."""
    s = dict(spec.get("settings", {}))
    cd = dict(spec, settings=dict(s, operator="central"))
    zh = dict(spec, settings=dict(s, operator="zucker-hummel"))
    _, c_cd = render(arr, spacing, cd, threads)
    _, c_zh = render(arr, spacing, zh, threads)
    k = (c_zh - c_cd) // 20
    w = c_cd - 6 * k
    return w, k


def box_interval(org, dirv, lo, hi):
    o, d = (np.ascontiguousarray(x, np.float64) for x in (org, dirv))
    lo, hi = (np.ascontiguousarray(x, np.float64) for x in (lo, hi))
    out = np.zeros(2)
    hit = lib().vco_box_interval(_dp(o), _dp(d), _dp(lo), _dp(hi), _dp(out))
    return (float(out[0]), float(out[1])) if hit else None


def first_hit(arr, spacing, org, dirv, interval, coarse, fine, window, interp="trilinear"):
    arr, code, nx, ny, nz = _vol(arr)
    sp = np.ascontiguousarray(spacing, np.float64)
    o, d = (np.ascontiguousarray(x, np.float64) for x in (org, dirv))
    out = np.zeros(3)
    cnt = ctypes.c_int64(0)
    found = lib().vco_first_hit(arr.ctypes.data, code, nx, ny, nz, _dp(sp), _dp(o), _dp(d),
                                float(interval[0]), float(interval[1]), float(coarse),
                                float(fine), float(window[0]), float(window[1]),
                                INTERP_CODES[interp], _dp(out), ctypes.byref(cnt))
    if not found:
        return None
    return float(out[0]), float(out[1]), bool(out[2])


def bisect(arr, spacing, org, dirv, t_before, t_after, window, iters=6, interp="trilinear"):
    arr, code, nx, ny, nz = _vol(arr)
    sp = np.ascontiguousarray(spacing, np.float64)
    o, d = (np.ascontiguousarray(x, np.float64) for x in (org, dirv))
    cnt = ctypes.c_int64(0)
    return float(lib().vco_bisect(arr.ctypes.data, code, nx, ny, nz, _dp(sp), _dp(o), _dp(d),
                                  float(t_before), float(t_after), float(window[0]),
                                  float(window[1]), int(iters), INTERP_CODES[interp],
                                  ctypes.byref(cnt)))
