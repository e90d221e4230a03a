"""Randomised parity sweep: seeded random scenes (camera orbit / elevation /
zoom, threshold window, operator, interpolation, mode, storage type,
spacing, clip box, light, transfer function) on small CT / noise / sphere
volumes, each rendered on the device and by the C oracle.

Bars: reference taps bit-exact with and without empty-space skipping (and
the exact sample count without it); gradient-volume shading within 1/255.
The point is coverage of rare decisions -- float32 pre-test near a
threshold, skip boxes near faces, clamped cells, grazing rays."""

from __future__ import annotations

from dataclasses import replace

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from oracle import oracle
from paper_1609_01317_b200 import phantoms
from tests.specs import spec_of

pytestmark = pytest.mark.gpu

N_SCENES = 96


def _volumes():
    rng = np.random.default_rng(20261018)
    ct = phantoms.ct_phantom(56).as_array()
    noise = rng.integers(0, 4096, size=(20, 24, 28)).astype(np.uint16)
    smooth = phantoms.marschner_lobb(40).as_array()
    return {"ct": ct, "noise": noise, "ml": smooth}


def _scene(rng, arr, name):
    dtype = rng.choice(["u16", "u8", "f32"]) if name != "ct" else rng.choice(["u16", "f32"])
    a = arr
    if dtype == "u8":
        a = (arr.astype(np.float64) * (255.0 / max(1.0, float(arr.max())))).astype(np.uint8)
    spacing = tuple(float(x) for x in rng.choice([1.0, 0.5, 2.0, 0.7, 1.3], size=3)) \
        if rng.random() < 0.5 else (1.0, 1.0, 1.0)
    vol = vc.Volume.from_array(a, spacing=spacing, dtype={"u16": np.uint16, "u8": np.uint8,
                                                          "f32": np.float32}[dtype])
    base = vc.default_scene(vol)
    cam = vc.Camera(eye=base.camera.eye, target=base.camera.target,
                    azimuth=float(rng.uniform(0, 360)), elevation=float(rng.uniform(-80, 80)),
                    zoom=float(rng.uniform(0.7, 1.6)))
    vmax = float(a.max())
    lo = float(rng.uniform(0.05, 0.6)) * vmax
    hi = vmax if rng.random() < 0.6 else float(rng.uniform(lo, vmax))
    mu = float(rng.choice([1000.0, max(1.0, 0.25 * vmax)]))
    clip = None
    if rng.random() < 0.3:
        ext = vol.extent
        c0 = tuple(float(rng.uniform(0, 0.3)) * e for e in ext)
        c1 = tuple(float(rng.uniform(0.6, 1.0)) * e for e in ext)
        clip = vc.ClipBox(c0, c1)
    light = vc.Light(position=tuple(float(x) for x in rng.uniform(-2, 2, size=3) * max(vol.extent)))
    sc = vc.Scene(camera=cam, light=light, window=vc.ThresholdWindow(lo, hi),
                  transfer=vc.TransferFunction.default_ct() if mu == 1000.0 else vc.TransferFunction(
                      points=[(-1000.0, (0.0, 0.0, 0.0, 0.0)), (0.0, (0.8, 0.5, 0.4, 0.05)),
                              (2000.0, (1.0, 1.0, 0.9, 0.6))], mu_water=mu),
                  clip=clip)
    st = vc.RenderSettings(width=int(rng.integers(40, 90)), height=int(rng.integers(30, 70)),
                           operator=vc.OperatorKind(rng.choice(["central", "sobel3d", "zucker-hummel"])),
                           interpolation=vc.InterpolationMode(rng.choice(["trilinear", "trilinear", "linear",
                                                                          "nearest"])),
                           mode=str(rng.choice(["surface", "composited"])),
                           coarse_step=float(rng.choice([1.0, 0.75, 1.5])), fine_step=0.125,
                           refine_iters=int(rng.integers(0, 8)))
    return vol, sc, st


def zero_window_scene(rng, vol, sc):
    """The scene with a threshold window containing 0 (lower bound 0 or below):
    with use_octree the reference skips in-window border samples through its
    octree segments, which the device replays."""
    vmax = float(vol.as_array().max())
    lo = -float(rng.uniform(0.0, 0.3)) * vmax if rng.random() < 0.7 else 0.0
    hi = float(rng.uniform(0.02, 0.7)) * vmax
    return vc.Scene(camera=sc.camera, light=sc.light, window=vc.ThresholdWindow(lo, hi),
                    transfer=sc.transfer, clip=sc.clip)


@pytest.fixture(scope="module")
def volumes():
    return _volumes()


@pytest.mark.parametrize("i", range(N_SCENES))
def test_random_scene_vs_oracle(volumes, i):
    rng = np.random.default_rng(1000 + i)
    name = ["ct", "noise", "ml"][i % 3]
    vol, sc, st = _scene(rng, volumes[name], name)
    want, want_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), threads=8)
    fb = vc.render_frame(vol, sc, replace(st, use_octree=False))
    d = np.abs(fb.pixels.astype(int) - want.astype(int))
    assert d.max() == 0, f"brute force: {int((d > 0).any(axis=2).sum())} px differ, max {int(d.max())}"
    assert fb.sample_count == want_count
    fb = vc.render_frame(vol, sc, replace(st, use_octree=True))
    assert np.array_equal(fb.pixels, want), "empty-space skipping changed pixels"
    fb = vc.render_frame(vol, sc, replace(st, gradient_source="volume"))
    assert int(np.abs(fb.pixels.astype(int) - want.astype(int)).max()) <= 1


@pytest.mark.parametrize("i", range(32))
def test_random_adaptive_scene_vs_oracle(volumes, i):
    """use_adaptive on the same kind of random scenes (random stride factor,
    detail epsilon, octree block size), with and without the octree-segment
    walk: bit-exact, counts included."""
    rng = np.random.default_rng(5000 + i)
    name = ["ct", "noise", "ml"][i % 3]
    vol, sc, st = _scene(rng, volumes[name], name)
    vmax = float(vol.as_array().max())
    st = replace(st, use_adaptive=True, use_octree=False, adaptive_factor=int(rng.integers(1, 9)),
                 detail_epsilon=None if rng.random() < 0.3 else float(rng.uniform(0.001, 0.3)) * vmax,
                 octree_min_block=int(rng.choice([2, 4, 8])))
    # the reference's default use_octree=True restarts the stride at its
    # octree segments: odd scenes run that walk
    st = replace(st, use_octree=bool(i % 2))
    want, want_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), threads=8,
                                     octree=True)
    fb = vc.render_frame(vol, sc, st)
    d = np.abs(fb.pixels.astype(int) - want.astype(int))
    assert d.max() == 0, f"{int((d > 0).any(axis=2).sum())} px differ, max {int(d.max())}"
    assert fb.sample_count == want_count


def test_gradient_volume_cancellation_regression(volumes):
    """A scene from the 10 000-scene sweep (tools/parity_sweep.py, seed
    206744: f32 grid, nearest interpolation, CD) where the gradient field
    crosses zero at a shaded sample: the float32 interpolated gradient lost
    its direction (32 LSB off) until near-cancelling corners were routed to
    the exact taps."""
    rng = np.random.default_rng(206744)
    vol, sc, st = _scene(rng, volumes["ct"], "ct")
    want, _ = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), threads=8)
    fb = vc.render_frame(vol, sc, replace(st, gradient_source="volume"))
    assert int(np.abs(fb.pixels.astype(int) - want.astype(int)).max()) <= 1


@pytest.mark.parametrize("i", range(24))
def test_random_zero_window_scene_vs_oracle(volumes, i):
    """0 inside the window: use_octree=False is the brute-force march,
    use_octree=True the reference's octree-segment walk (oracle octree=True,
    pinned to the reference's zerowin goldens) -- pixels and counts."""
    rng = np.random.default_rng(9000 + i)
    name = ["ct", "noise", "ml"][i % 3]
    vol, sc, st = _scene(rng, volumes[name], name)
    sc = zero_window_scene(rng, vol, sc)
    for oct_on in (False, True):
        st2 = replace(st, use_octree=oct_on)
        want, want_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st2)), threads=8, octree=True)
        fb = vc.render_frame(vol, sc, st2)
        d = np.abs(fb.pixels.astype(int) - want.astype(int))
        assert d.max() == 0, (oct_on, int((d > 0).any(axis=2).sum()), int(d.max()))
        assert fb.sample_count == want_count, oct_on
        fb = vc.render_frame(vol, sc, replace(st2, gradient_source="volume"))
        assert int(np.abs(fb.pixels.astype(int) - want.astype(int)).max()) <= 1
