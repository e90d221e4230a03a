"""The first-hit kernel's fixed-point lattice walk (raycast.cu, "fixed-point
lattice walk") against the float64 oracle, on the cases its exactness
argument singles out:

* positions exactly on cell faces (axis-aligned rays through voxel
  centres): every such sample sits inside the 2^-20 guard band and must
  take the reference's float64 path;
* rays fx_setup does not admit -- a camera so far away that the float64
  rounding bound (|o| / s > 2^24) fails, a step count above 2^19 -- where
  every sample takes the float64 path;
* a large but admitted eye distance (the bound's slack);
* more than 64 bisection steps (the bisection falls back to float64);
* float32 and uint8 grids, anisotropic spacing.

Pixels and sample counts must equal the oracle's (brute force), and
empty-space skipping must not change the pixels.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from oracle import oracle
from paper_1609_01317_b200 import phantoms
from tests.specs import spec_of

pytestmark = pytest.mark.gpu


def _check(vol, sc, st, counts=True):
    want, want_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), threads=8)
    fb = vc.render_frame(vol, sc, replace(st, use_octree=False))
    d = int(np.abs(fb.pixels.astype(int) - want.astype(int)).max())
    assert d == 0, f"brute force: max|d|={d}"
    if counts:
        assert fb.sample_count == want_count
    fb = vc.render_frame(vol, sc, replace(st, use_octree=True))
    d = int(np.abs(fb.pixels.astype(int) - want.astype(int)).max())
    assert d == 0, f"skipping: max|d|={d}"


def _ct(n=64):
    return phantoms.ct_phantom(n)


@pytest.mark.parametrize("axis", [0, 1, 2])
@pytest.mark.parametrize("coarse", [1.0, 0.5, 0.75])
@pytest.mark.parametrize("mode", ["surface", "composited"])
def test_axis_aligned_rays_through_voxel_centres(axis, coarse, mode):
    vol = _ct(64)
    c = [32.5, 32.5, 32.5]  # voxel coordinate 32.0 (p = w / s - 0.5)
    eye = list(c)
    eye[axis] = -40.0
    up = (0.0, 0.0, 1.0) if axis == 1 else (0.0, 1.0, 0.0)
    cam = vc.Camera(eye=tuple(eye), target=tuple(c), up=up, fov_y=40.0)
    sc = vc.Scene(camera=cam, light=phantoms.default_scene(vol).light)
    # odd sizes: the centre row and column are exactly axis-parallel planes
    st = vc.RenderSettings(width=33, height=31, mode=mode, coarse_step=coarse, fine_step=coarse / 8.0,
                           operator=vc.OperatorKind.SOBEL3D)
    _check(vol, sc, st)


def test_integer_eye_and_unit_steps_every_sample_on_a_lattice_plane():
    """Eye at a voxel-centre position, unit steps along an axis direction:
    all three coordinates of the centre ray are integers at every step."""
    vol = _ct(48)
    cam = vc.Camera(eye=(24.5, 24.5, -30.5), target=(24.5, 24.5, 24.5), fov_y=30.0)
    sc = vc.Scene(camera=cam, light=phantoms.default_scene(vol).light)
    st = vc.RenderSettings(width=1, height=1, mode="composited", coarse_step=1.0, fine_step=0.25)
    _check(vol, sc, st)
    st = replace(st, width=5, height=5)
    _check(vol, sc, st)


@pytest.mark.parametrize("dist", [3.0e7, 1.0e6, 2.0e5])
def test_far_eye(dist):
    """3e7 and 1e6: beyond the frame-wide admission bound ((|o| + 2T) / s <=
    2^21), every sample takes the float64 path; 2e5: admitted with a large
    rounding scale."""
    vol = _ct(64)
    c = (32.0, 30.0, 33.0)
    cam = vc.Camera(eye=(c[0] + 0.3 * dist, c[1] + 0.1 * dist, c[2] - dist), target=c,
                    fov_y=float(np.degrees(2.0 * np.arctan(40.0 / dist))))
    sc = vc.Scene(camera=cam, light=phantoms.default_scene(vol).light)
    st = vc.RenderSettings(width=48, height=40, mode="composited")
    _check(vol, sc, st)


def test_step_count_above_walk_limit():
    """coarse steps small enough that k_last > 2^19: not admitted."""
    vol = _ct(40)
    sc, st = phantoms.scene_c3(vol, width=4, height=3, azimuth=17.0, mode="surface")
    st = replace(st, coarse_step=5.0e-5, fine_step=2.5e-5)  # ~ 40 / 5e-5 = 8e5 lattice steps
    _check(vol, sc, st)


def test_more_than_64_bisection_steps():
    vol = _ct(64)
    sc, st = phantoms.scene_c3(vol, width=64, height=48, azimuth=40.0)
    _check(vol, sc, replace(st, refine_iters=70))
    _check(vol, sc, replace(st, refine_iters=64))


@pytest.mark.parametrize("dtype", [np.uint8, np.float32])
def test_other_voxel_types(dtype):
    rng = np.random.default_rng(3)
    base = phantoms.ct_phantom(56).as_array().astype(np.float64)
    if dtype == np.uint8:
        arr = np.clip(base / 16.0, 0, 255).astype(np.uint8)
        win = vc.ThresholdWindow(30.0, 255.0)
    else:
        arr = (base + rng.normal(0.0, 3.0, base.shape)).astype(np.float32)
        win = vc.ThresholdWindow(500.0, 4095.0)
    vol = vc.Volume.from_array(arr, dtype=dtype)
    sc, st = phantoms.scene_c3(vol, width=80, height=60, azimuth=123.0)
    sc = vc.Scene(camera=sc.camera, light=sc.light, window=win, transfer=sc.transfer)
    _check(vol, sc, st)


@pytest.mark.parametrize("spacing", [(0.5, 0.5, 0.5), (0.7, 1.1, 0.9)])
def test_spacing_with_axis_aligned_centre_ray(spacing):
    """Voxel-centre axis rays under power-of-two and general spacing."""
    base = _ct(48).as_array()
    vol = vc.Volume.from_array(base, spacing=spacing)
    c = tuple((24 + 0.5) * s for s in spacing)
    cam = vc.Camera(eye=(c[0], c[1], -20.0), target=c, fov_y=35.0)
    sc = vc.Scene(camera=cam, light=phantoms.default_scene(vol).light)
    st = vc.RenderSettings(width=21, height=21, mode="composited", coarse_step=0.5 * min(spacing),
                           fine_step=0.0625 * min(spacing))
    _check(vol, sc, st)
