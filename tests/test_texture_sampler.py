"""The hardware-texture sampler (RenderSettings.sampler = "texture").

It is an approximation of the reference (8-bit texture-filter weights), so
it is held to the tolerance DESIGN.md states for it, not to the 1/255 bar:
on the CT scenes >= 99% of pixels within 1/255 of the reference and a mean
|d| <= 0.5/255; threshold-crossing pixels may differ more.  Properties that
hold exactly: empty-space skipping stays output-neutral (texture values are
convex combinations of the 8 corners) and the band partition reassembles the
whole frame.
"""

from __future__ import annotations

import ctypes
from dataclasses import replace

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import phantoms
from tests.specs import product_scene, product_settings, product_volume


def _stats(a, b):
    d = np.abs(a.astype(np.int32) - b.astype(np.int32)).max(axis=2)
    return float((d <= 1).mean()), float(d.mean())


def test_settings_validation():
    with pytest.raises(ValueError):
        vc.RenderSettings(sampler="tex3d")
    with pytest.raises(ValueError):
        vc.RenderSettings(sampler="texture", interpolation=vc.InterpolationMode.NEAREST)
    with pytest.raises(ValueError):
        vc.RenderSettings(sampler="texture", use_adaptive=True)
    assert vc.RenderSettings().sampler == "software"


@pytest.fixture(scope="module")
def ct192():
    return phantoms.ct_phantom(192)


@pytest.mark.gpu
@pytest.mark.parametrize("grad", ["volume", "taps"])
@pytest.mark.parametrize("mode", ["surface", "composited"])
def test_texture_sampler_within_stated_tolerance(ct192, grad, mode):
    for az in (0.0, 40.0):
        sc, st = phantoms.scene_c3(ct192, azimuth=az, width=480, height=270, mode=mode)
        ref = vc.render_frame(ct192, sc, replace(st, gradient_source=grad)).pixels
        tex = vc.render_frame(ct192, sc, replace(st, gradient_source=grad, sampler="texture")).pixels
        within1, mean = _stats(tex, ref)
        assert within1 >= 0.99 and mean <= 0.5, (within1, mean)


@pytest.mark.gpu
def test_texture_sampler_golden_frames_close(golden):
    """The reference goldens (all grids / operators / modes with trilinear
    interpolation).  These include binary-valued phantoms (spheres, shells)
    whose every surface pixel sits on a 0 -> value step, where the 8-bit
    filter weights move the surface most: the bar there is >= 90% within
    1/255 and mean <= 2/255 (C1's u8 sphere: ~94%, mean ~1)."""
    from tests.conftest import frame_names

    checked = 0
    bad = []
    for name in frame_names():
        arr, spacing, spec, want_px, _ = golden.frame(name)
        s = spec.get("settings", {})
        if s.get("interpolation", "trilinear") != "trilinear" or s.get("use_adaptive"):
            continue
        vol = product_volume(arr, spacing)
        fb = vc.render_frame(vol, product_scene(spec), product_settings(spec, sampler="texture"))
        within1, mean = _stats(fb.pixels, want_px)
        print(f"texture vs reference {name}: within 1/255 {within1:.4f}, mean {mean:.3f}")
        if not (within1 >= 0.90 and mean <= 2.0):
            bad.append((name, within1, mean))
        checked += 1
    assert checked >= 10
    assert not bad, bad


@pytest.mark.gpu
def test_texture_sampler_skipping_is_output_neutral(ct192):
    sc, st = phantoms.scene_c3(ct192, azimuth=25.0, width=320, height=180)
    for grad in ("volume", "taps"):
        base = replace(st, gradient_source=grad, sampler="texture")
        a = vc.render_frame(ct192, sc, replace(base, use_octree=True))
        b = vc.render_frame(ct192, sc, replace(base, use_octree=False))
        assert np.array_equal(a.pixels, b.pixels)
        assert a.sample_count <= b.sample_count


@pytest.mark.gpu
def test_texture_sampler_float_grid_and_u8():
    vol = phantoms.fbm_noise(64, seed=3)
    sc, st = phantoms.scene_c4(vol, width=160, height=96)
    ref = vc.render_frame(vol, sc, st).pixels
    tex = vc.render_frame(vol, sc, replace(st, sampler="texture")).pixels
    within1, mean = _stats(tex, ref)
    assert within1 >= 0.97 and mean <= 1.0, (within1, mean)
    ml = phantoms.marschner_lobb(64)
    sc, st = phantoms.scene_c2(ml, width=128, height=128)
    ref = vc.render_frame(ml, sc, st).pixels
    tex = vc.render_frame(ml, sc, replace(st, sampler="texture")).pixels
    within1, mean = _stats(tex, ref)
    assert within1 >= 0.99 and mean <= 0.5, (within1, mean)


@pytest.mark.gpu
def test_texture_sample_peak_reported():
    from paper_1609_01317_b200 import _native

    g = ctypes.c_double()
    _native.check(_native.load().vc_sample_peak_texture(0, ctypes.byref(g)))
    assert g.value > 1.0
