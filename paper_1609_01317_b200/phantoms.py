"""Synthetic datasets of the BASELINE configurations.

None of these exist in the reference (its phantoms are sphere / shell /
ramp / empty, volume.py:113-181); they are deterministic numpy generators
so the oracle and the device render identical grids.

  C1  sphere_c1(64)            uint8 sphere, value 200, radius 0.35 n
  C2  marschner_lobb(256)      uint8 Marschner-Lobb, round(255 rho)
  C3  ct_phantom(512)          uint16 3-D Shepp-Logan (Kak-Slaney ellipsoids), raw = 1000 + HU
  C4  fbm_noise(1024)          float32 5-octave value-noise fBm in [0, 4095]
  C5  gradient sweep           ct_phantom / fbm_noise at 128^3 .. 1024^3

plus the scene for each (camera, window, transfer function, settings).
"""

from __future__ import annotations

import math

import numpy as np

from .gradients import OperatorKind
from .raycast import (
    Camera,
    Light,
    RenderMode,
    RenderSettings,
    Scene,
    ThresholdWindow,
    TransferFunction,
    default_scene,
)
from .volume import Volume, make_phantom

# ------------------------------------------------------------------ volumes


def sphere_c1(n: int = 64) -> Volume:
    """C1: make_phantom("sphere", n, radius=0.35 n, value=200) stored as uint8."""
    return make_phantom("sphere", n, radius=0.35 * n, value=200, dtype=np.uint8)


def _centers(n: int) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 0.5) * (2.0 / n) - 1.0


def marschner_lobb(n: int = 256, alpha: float = 0.25, f_m: float = 6.0) -> Volume:
    """C2: Marschner-Lobb test signal on [-1,1]^3 at voxel centres,
    rho = (1 - sin(pi z / 2) + alpha (1 + cos(2 pi f_M cos(pi r / 2)))) / (2 (1 + alpha)),
    r = sqrt(x^2 + y^2), quantised round(255 rho) to uint8."""
    c = _centers(n)
    z = c[:, None, None]
    y = c[None, :, None]
    x = c[None, None, :]
    r = np.sqrt(x * x + y * y)
    rho_r = np.cos(2.0 * math.pi * f_m * np.cos(math.pi * r / 2.0))
    rho = (1.0 - np.sin(math.pi * z / 2.0) + alpha * (1.0 + rho_r)) / (2.0 * (1.0 + alpha))
    arr = np.clip(np.rint(255.0 * rho), 0, 255).astype(np.uint8)
    return Volume.from_array(arr, dtype=np.uint8)


# Kak & Slaney 3-D Shepp-Logan: (a, b, c, x0, y0, z0, phi_deg, density),
# densities of the "modified" (higher-contrast) variant.
SHEPP_LOGAN_3D = (
    (0.6900, 0.920, 0.810, 0.00, 0.000, 0.00, 0.0, 1.0),
    (0.6624, 0.874, 0.780, 0.00, -0.0184, 0.00, 0.0, -0.8),
    (0.1100, 0.310, 0.220, 0.22, 0.000, 0.00, -18.0, -0.2),
    (0.1600, 0.410, 0.280, -0.22, 0.000, 0.00, 18.0, -0.2),
    (0.2100, 0.250, 0.410, 0.00, 0.350, -0.15, 0.0, 0.1),
    (0.0460, 0.046, 0.050, 0.00, 0.100, 0.25, 0.0, 0.1),
    (0.0460, 0.046, 0.050, 0.00, -0.100, 0.25, 0.0, 0.1),
    (0.0460, 0.023, 0.050, -0.08, -0.605, 0.00, 0.0, 0.1),
    (0.0230, 0.023, 0.020, 0.00, -0.606, 0.00, 0.0, 0.1),
    (0.0230, 0.046, 0.020, 0.06, -0.605, 0.00, 0.0, 0.1),
)


def ct_phantom(n: int = 512, skull_hu: float = 300.0) -> Volume:
    """C3: uint16 3-D Shepp-Logan head.  Summed density v inside the head
    maps to raw = 1000 + (v - 0.2) / 0.8 * skull_hu (brain v = 0.2 -> 0 HU,
    bone v = 1.0 -> skull_hu), 0 (air, -1000 HU) outside, clamped to 12 bits.
    skull_hu = 300 keeps bone translucent under TransferFunction.default_ct
    so the composite loop and early ray termination are exercised
    (SURVEY.md §8(d), C3)."""
    c = _centers(n)
    out = np.empty((n, n, n), np.uint16)
    h = 2.0 / n
    boxes = []  # conservative voxel-index bounding box of each ellipsoid
    for (a, b, cc, x0, y0, z0, phi, dens) in SHEPP_LOGAN_3D:
        ph = math.radians(phi)
        ex = math.sqrt((a * math.cos(ph)) ** 2 + (b * math.sin(ph)) ** 2)
        ey = math.sqrt((a * math.sin(ph)) ** 2 + (b * math.cos(ph)) ** 2)
        box = []
        for lo, hi in ((x0 - ex, x0 + ex), (y0 - ey, y0 + ey), (z0 - cc, z0 + cc)):
            i0 = max(int(math.floor((lo + 1.0) / h - 0.5)) - 1, 0)
            i1 = min(int(math.ceil((hi + 1.0) / h - 0.5)) + 2, n)
            box.append((i0, i1))
        boxes.append(box)
    for kz in range(n):  # slice by slice keeps peak memory at O(n^2)
        z = c[kz]
        v = np.zeros((n, n), np.float64)
        head = np.zeros((n, n), bool)
        for idx, (a, b, cc, x0, y0, z0, phi, dens) in enumerate(SHEPP_LOGAN_3D):
            (xa, xb), (ya, yb), (za, zb) = boxes[idx]
            if not za <= kz < zb or xa >= xb or ya >= yb:
                continue
            ph = math.radians(phi)
            cp, sp = math.cos(ph), math.sin(ph)
            y = c[ya:yb, None]
            x = c[None, xa:xb]
            dx, dy, dz = x - x0, y - y0, z - z0
            xr = dx * cp + dy * sp
            yr = -dx * sp + dy * cp
            inside = (xr / a) ** 2 + (yr / b) ** 2 + (dz / cc) ** 2 <= 1.0
            v[ya:yb, xa:xb] += np.where(inside, dens, 0.0)
            if idx == 0:
                head[ya:yb, xa:xb] = inside
        raw = 1000.0 + (v - 0.2) / 0.8 * skull_hu
        raw = np.where(head, np.clip(np.rint(raw), 0, 4095), 0.0)
        out[kz] = raw.astype(np.uint16)
    return Volume.from_array(out)


def _hash3(ix, iy, iz, seed: int) -> np.ndarray:
    """Integer lattice hash -> [0, 1) (uint32 arithmetic, wraps)."""
    h = (ix.astype(np.uint32) * np.uint32(0x8DA6B343)
         ^ iy.astype(np.uint32) * np.uint32(0xD8163841)
         ^ iz.astype(np.uint32) * np.uint32(0xCB1AB31F)
         ^ np.uint32(seed * 0x9E3779B9 & 0xFFFFFFFF))
    h ^= h >> np.uint32(15)
    h *= np.uint32(0x2C1B3C6D)
    h ^= h >> np.uint32(12)
    h *= np.uint32(0x297A2D39)
    h ^= h >> np.uint32(15)
    return (h >> np.uint32(8)).astype(np.float64) * (1.0 / (1 << 24))


def _smooth(t: np.ndarray) -> np.ndarray:
    return t * t * (3.0 - 2.0 * t)


def _lerp_axis(lo: np.ndarray, hi: np.ndarray, w: np.ndarray) -> np.ndarray:
    return lo * (1.0 - w) + hi * w


def fbm_noise(n: int = 1024, octaves: int = 5, seed: int = 1609, base_cells: int = 8,
              dtype=np.float32, slab: int = 64, device: str | None = None) -> Volume:
    """C4: seeded fBm of trilinear value noise with smoothstep weights,
    octave k on a lattice of base_cells * 2^k cells per axis (integer hash
    values in [0, 1)) with amplitude 2^-k, normalised to [0, 4095].  The
    interpolation is evaluated separably (x, then y, then z), slab by slab,
    so 1024^3 takes seconds, not hours.  device="cuda" evaluates the same
    formula with torch on the GPU (last-bit differences from numpy are
    possible; oracle and device always receive the same returned grid)."""
    if device is not None:
        return _fbm_noise_torch(n, octaves, seed, base_cells, dtype, device)
    c = (np.arange(n, dtype=np.float64) + 0.5) / n
    out = np.empty((n, n, n), np.float32)
    total_amp = sum(0.5 ** k for k in range(octaves))
    axes = []
    for o in range(octaves):
        cells = base_cells << o
        f = c * cells
        i = np.floor(f).astype(np.int64)
        w = _smooth(f - i)
        g = np.arange(cells + 1, dtype=np.int64)
        lat = _hash3(g[:, None, None], g[None, :, None], g[None, None, :], seed + o)  # [z, y, x]
        # x then y interpolation is independent of z: (cells+1, n, n) per octave
        tx = _lerp_axis(lat[:, :, i], lat[:, :, i + 1], w)                 # (C, C, n)
        txy = _lerp_axis(tx[:, i, :], tx[:, i + 1, :], w[:, None])        # (C, n, n)
        axes.append((i, w, txy))
    for z0 in range(0, n, slab):
        z1 = min(z0 + slab, n)
        acc = np.zeros((z1 - z0, n, n), np.float64)
        for o, (i, w, txy) in enumerate(axes):
            iz, wz = i[z0:z1], w[z0:z1, None, None]
            acc += (0.5 ** o) * _lerp_axis(txy[iz], txy[iz + 1], wz)
        out[z0:z1] = (acc / total_amp * 4095.0).astype(np.float32)
    return Volume.from_array(out, dtype=dtype)


def _fbm_noise_torch(n, octaves, seed, base_cells, dtype, device) -> Volume:
    out = fbm_noise_tensor(n, octaves, seed, base_cells, device).cpu().numpy()
    return Volume.from_array(out, dtype=dtype)


def fbm_noise_tensor(n: int = 1024, octaves: int = 5, seed: int = 1609, base_cells: int = 8,
                     device: str = "cuda"):
    """fbm_noise evaluated with torch on `device`, returned as the (n, n, n)
    float32 device tensor itself (no host copy): bench.py's C4 side config
    hands it to the library with vc_volume_create_device."""
    import torch

    c = (torch.arange(n, dtype=torch.float64, device=device) + 0.5) / n
    acc = torch.zeros((n, n, n), dtype=torch.float64, device=device)
    total_amp = sum(0.5 ** k for k in range(octaves))
    for o in range(octaves):
        cells = base_cells << o
        f = c * cells
        i = torch.floor(f).long()
        t = f - i
        w = t * t * (3.0 - 2.0 * t)
        g = np.arange(cells + 1, dtype=np.int64)
        lat = torch.as_tensor(_hash3(g[:, None, None], g[None, :, None], g[None, None, :], seed + o),
                              device=device)
        tx = lat[:, :, i] * (1.0 - w) + lat[:, :, i + 1] * w
        txy = tx[:, i, :] * (1.0 - w[:, None]) + tx[:, i + 1, :] * w[:, None]
        for z0 in range(0, n, 64):
            z1 = min(z0 + 64, n)
            wz = w[z0:z1, None, None]
            acc[z0:z1] += (0.5 ** o) * (txy[i[z0:z1]] * (1.0 - wz) + txy[i[z0:z1] + 1] * wz)
        del tx, txy
    out = (acc / total_amp * 4095.0).to(torch.float32)
    del acc
    return out


# ------------------------------------------------------------------ scenes


def scene_c1(vol: Volume, op=OperatorKind.CENTRAL_DIFFERENCE, width=256, height=256):
    """C1: default_scene framing; u8 data needs a scaled window and mu_water
    (the default [500, 4095] renders nothing on 8-bit data)."""
    base = default_scene(vol)
    sc = Scene(camera=base.camera, light=base.light, window=ThresholdWindow(100.0, 255.0),
               transfer=TransferFunction(TransferFunction.default_ct().points, mu_water=100.0))
    return sc, RenderSettings(width=width, height=height, operator=op, mode=RenderMode.SURFACE)


def scene_c2(vol: Volume, op=OperatorKind.SOBEL3D, width=1024, height=1024, azimuth=0.0):
    """C2: Marschner-Lobb rho = 0.5 isosurface (raw >= 128), orbit by azimuth."""
    base = default_scene(vol)
    cam = Camera(eye=base.camera.eye, target=base.camera.target, azimuth=azimuth)
    sc = Scene(camera=cam, light=base.light, window=ThresholdWindow(128.0, 255.0),
               transfer=TransferFunction(TransferFunction.default_ct().points, mu_water=100.0))
    return sc, RenderSettings(width=width, height=height, operator=op, mode=RenderMode.SURFACE)


def scene_c3(vol: Volume, op=OperatorKind.ZUCKER_HUMMEL, width=1920, height=1080, azimuth=0.0,
             mode=RenderMode.COMPOSITED):
    """C3: CT head, default window [500, 4095] and default_ct transfer,
    composited with early ray termination, orbit by azimuth."""
    base = default_scene(vol)
    cam = Camera(eye=base.camera.eye, target=base.camera.target, azimuth=azimuth)
    sc = Scene(camera=cam, light=base.light)
    return sc, RenderSettings(width=width, height=height, operator=op, mode=mode)


def scene_c4(vol: Volume, op=OperatorKind.SOBEL3D, width=3840, height=2160, azimuth=0.0):
    """C4: noise volume with a narrow window on the top ~10% of values, so
    rays march into the interior instead of stopping at the front face."""
    base = default_scene(vol)
    cam = Camera(eye=base.camera.eye, target=base.camera.target, azimuth=azimuth)
    tf = TransferFunction(points=[(-1000.0, (0.2, 0.4, 0.9, 0.0)), (2000.0, (0.9, 0.8, 0.3, 0.6)),
                                  (3095.0, (1.0, 1.0, 1.0, 1.0))], mu_water=1000.0)
    sc = Scene(camera=cam, light=base.light, window=ThresholdWindow(2600.0, 4095.0), transfer=tf)
    return sc, RenderSettings(width=width, height=height, operator=op, mode=RenderMode.COMPOSITED)
