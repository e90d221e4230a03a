"""Host-side half of the reference's behavioural tests, restated against
this package (no device needed): parameter validation, the camera and
ray geometry, HU / transfer / compositing / shading helpers and gradient
normalisation (the clip-box interval runs on the device:
tests/test_reference_behaviour_gpu.py).

Sources: pkg/tests/test_render.py:203-224, test_raycast_geometry.py:13-108,
test_raycast_pipeline.py:193-302, test_gradients.py:199-205,
test_acceptance.py:223-226.  The
assertions and tolerances are the reference's; the structure is this
suite's."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1609_01317_b200 as vc


# ------------------------------------------------------------------ settings / scene


@pytest.mark.parametrize("bad", [dict(width=0), dict(fine_step=2.0, coarse_step=1.0), dict(mode="xray"),
                                 dict(adaptive_factor=0), dict(background=(2, 0, 0, 1))])
def test_render_settings_reject(bad):
    """test_render.py:203-213"""
    with pytest.raises(ValueError):
        vc.RenderSettings(**bad)


def test_default_scene_layout():
    """test_render.py:216-221: eye outside the box, light at the eye, the
    default [500, 4095] window."""
    sc = vc.default_scene(vc.make_phantom("sphere", 32, radius=10))
    assert sc.camera.eye[2] < 0
    assert tuple(sc.light.position) == tuple(sc.camera.eye)
    assert (sc.window.low, sc.window.high) == (500.0, 4095.0)


# ------------------------------------------------------------------ ray generation


def test_rays_are_unit_and_start_at_the_eye():
    """test_raycast_geometry.py:13-19"""
    cam = vc.Camera(eye=(0, 0, -10), target=(0, 0, 0))
    rng = np.random.default_rng(1)
    for px, py in rng.integers(0, 64, size=(50, 2)):
        r = vc.generate_ray(cam, int(px), int(py), 64, 64)
        assert np.linalg.norm(r.direction) == pytest.approx(1.0, abs=1e-12)
        assert np.array_equal(r.origin, [0, 0, -10])


def test_image_symmetries_and_centre_ray():
    """test_raycast_geometry.py:22-37"""
    fwd = vc.generate_ray(vc.Camera(eye=(0, 0, -10), target=(0, 0, 5)), 50, 50, 101, 101)
    assert fwd.direction == pytest.approx([0, 0, 1], abs=1e-12)
    cam = vc.Camera(eye=(1, 2, -10), target=(1, 2, 0), fov_y=45)
    n = 64
    a, b = vc.generate_ray(cam, 3, 10, n, n), vc.generate_ray(cam, n - 4, 10, n, n)
    assert a.direction[0] == pytest.approx(-b.direction[0], abs=1e-12)
    assert a.direction[1] == pytest.approx(b.direction[1], abs=1e-12)
    top, bot = vc.generate_ray(cam, 12, 0, n, n), vc.generate_ray(cam, 12, n - 1, n, n)
    assert top.direction[1] == pytest.approx(-bot.direction[1], abs=1e-12)


def test_vertical_field_of_view():
    """test_raycast_geometry.py:40-48"""
    r = vc.generate_ray(vc.Camera(eye=(0, 0, -10), target=(0, 0, 0), fov_y=60), 50, 0, 101, 101)
    want = math.atan((1.0 - 1.0 / 101) * math.tan(math.radians(30)))
    got = math.atan2(r.direction[1], r.direction[2])
    assert got == pytest.approx(want, abs=1e-12) and got < math.radians(30)


@pytest.mark.parametrize("px", [64, -1])
def test_pixel_outside_image_rejected(px):
    """test_raycast_geometry.py:51-56"""
    with pytest.raises(ValueError):
        vc.generate_ray(vc.Camera(eye=(0, 0, -10), target=(0, 0, 0)), px, 0, 64, 64)


def test_orbit_controls():
    """test_raycast_geometry.py:59-97: identity orbit, azimuth about the
    target's y axis, elevation clamped at 89.9 deg, zoom divides the
    distance, and orbit composes with zoom."""
    a = vc.generate_ray(vc.Camera(eye=(3, 4, -12), target=(1, 1, 1)), 7, 9, 32, 32)
    b = vc.generate_ray(vc.Camera(eye=(3, 4, -12), target=(1, 1, 1), azimuth=0.0, elevation=0.0, zoom=1.0),
                        7, 9, 32, 32)
    assert a.origin == pytest.approx(b.origin, abs=1e-9)
    assert a.direction == pytest.approx(b.direction, abs=1e-12)

    def eye(**kw):
        base = dict(eye=(0, 0, 10), target=(0, 0, 0))
        base.update(kw)
        return vc.generate_ray(vc.Camera(**base), 8, 8, 17, 17).origin

    assert eye(azimuth=90.0) == pytest.approx([10, 0, 0], abs=1e-9)
    assert eye(azimuth=180.0) == pytest.approx([0, 0, -10], abs=1e-9)
    e = eye(elevation=30.0)
    assert e[1] == pytest.approx(10 * math.sin(math.radians(30)), abs=1e-9)
    assert np.linalg.norm(e) == pytest.approx(10.0, abs=1e-9)
    e = eye(elevation=90.0)
    assert e[1] < 10.0 and e[1] == pytest.approx(10 * math.sin(math.radians(89.9)), abs=1e-9)
    assert np.linalg.norm(eye(zoom=2.0)) == pytest.approx(5.0, abs=1e-9)
    assert eye(eye=(0, 0, 8), azimuth=90.0, zoom=4.0) == pytest.approx([2, 0, 0], abs=1e-9)


@pytest.mark.parametrize("bad", [dict(eye=(1, 1, 1), target=(1, 1, 1)), dict(fov_y=0.0), dict(fov_y=180.0),
                                 dict(zoom=0.0)])
def test_camera_rejects(bad):
    """test_raycast_geometry.py:100-108"""
    kw = dict(eye=(0, 0, 1), target=(0, 0, 0))
    kw.update(bad)
    with pytest.raises(ValueError):
        vc.Camera(**kw)


# ------------------------------------------------------- HU, transfer, compositing, shading


def test_hounsfield():
    """test_raycast_pipeline.py:193-205"""
    assert vc.hounsfield(1000.0, 1000.0) == 0.0
    assert vc.hounsfield(0.0, 1000.0) == -1000.0
    assert vc.hounsfield(2000.0, 1000.0) == 1000.0
    assert vc.hounsfield(1200.0, 1000.0) == pytest.approx(200.0, abs=1e-12)
    assert vc.hounsfield(500.0, 500.0) == 0.0
    # default mu_water = 1000 (test_acceptance.py:223-226)
    assert (vc.hounsfield(1000.0), vc.hounsfield(0.0), vc.hounsfield(2000.0, mu_water=2000.0)) == (0.0, -1000.0, 0.0)
    for mu in (0.0, -5.0):
        with pytest.raises(ValueError):
            vc.hounsfield(100.0, mu)


def test_transfer_lookup():
    """test_raycast_pipeline.py:208-231: exact at breakpoints, linear in
    between, clamped outside, constant with one breakpoint."""
    ct = vc.TransferFunction.default_ct()
    for hu, rgba in ct.points:
        assert vc.transfer(ct, hu) == pytest.approx(rgba, abs=0.0)
    assert vc.transfer(ct, -5000.0) == pytest.approx(vc.transfer(ct, -1000.0), abs=0.0)
    assert vc.transfer(ct, 9000.0) == pytest.approx(vc.transfer(ct, 1500.0), abs=0.0)
    two = vc.TransferFunction(points=[(0.0, (0, 0, 0, 0)), (100.0, (1, 0.5, 0.25, 1))])
    assert vc.transfer(two, 50.0) == pytest.approx([0.5, 0.25, 0.125, 0.5], abs=1e-12)
    assert vc.transfer(two, 25.0) == pytest.approx([0.25, 0.125, 0.0625, 0.25], abs=1e-12)
    one = vc.TransferFunction(points=[(0.0, (0.2, 0.4, 0.6, 0.8))])
    for hu in (-100.0, 0.0, 250.0):
        assert vc.transfer(one, hu) == pytest.approx([0.2, 0.4, 0.6, 0.8], abs=0.0)


@pytest.mark.parametrize("kw", [dict(points=[]), dict(points=[(0.0, (0, 0, 0, 0)), (0.0, (1, 1, 1, 1))]),
                                dict(points=[(0.0, (0, 0, 2.0, 0))]),
                                dict(points=[(0.0, (0, 0, 0, 0))], mu_water=0.0)])
def test_transfer_rejects(kw):
    """test_raycast_pipeline.py:234-242"""
    with pytest.raises(ValueError):
        vc.TransferFunction(**kw)


def test_composite_step():
    """test_raycast_pipeline.py:245-262"""
    x, y = np.array([0.2, 0.4, 0.6]), np.array([1.0, 0.5, 0.0])
    assert vc.composite_step(x, y, 1.0) == pytest.approx(y, abs=0.0)
    assert vc.composite_step(x, y, 0.0) == pytest.approx(x, abs=0.0)
    assert vc.composite_step(x, y, 0.5) == pytest.approx(0.5 * x + 0.5 * y, abs=1e-15)
    rng = np.random.default_rng(4)
    for _ in range(50):
        a = float(rng.uniform(0, 1))
        p, q = rng.uniform(0, 1, (2, 3))
        assert vc.composite_step(p, q, a) == pytest.approx(p * (1 - a) + q * a, abs=1e-15)
    for a in (1.5, -0.1):
        with pytest.raises(ValueError):
            vc.composite_step((0, 0, 0), (1, 1, 1), a)


def test_diffuse_shading():
    """test_raycast_pipeline.py:265-291: full colour head-on, black at 90
    degrees / behind / zero normal / light on the point, half at 60."""
    o, up = (0, 0, 0), (0, 0, 1)
    assert vc.shade(o, up, vc.Light(position=(0, 0, 10), color=(1.0, 0.5, 0.25))) == \
        pytest.approx([1.0, 0.5, 0.25], abs=1e-12)
    assert vc.shade(o, up, vc.Light(position=(10, 0, 0))) == pytest.approx([0, 0, 0], abs=1e-12)
    assert vc.shade(o, up, vc.Light(position=(0, 0, -10))) == pytest.approx([0, 0, 0], abs=0.0)
    s60 = vc.Light(position=(10 * math.sin(math.radians(60)), 0, 10 * math.cos(math.radians(60))))
    assert vc.shade(o, up, s60) == pytest.approx([0.5, 0.5, 0.5], abs=1e-9)
    assert vc.shade(o, (0, 0, 0), vc.Light(position=(5, 5, 5))) == pytest.approx([0, 0, 0], abs=0.0)
    assert vc.shade((1, 2, 3), up, vc.Light(position=(1, 2, 3))) == pytest.approx([0, 0, 0], abs=0.0)


def test_light_and_window_rules():
    """test_raycast_pipeline.py:294-302"""
    with pytest.raises(ValueError):
        vc.Light(position=(0, 0, 0), color=(1.5, 0, 0))
    with pytest.raises(ValueError):
        vc.ThresholdWindow(10.0, 5.0)
    w = vc.ThresholdWindow(5.0, 10.0)
    assert w.contains(5.0) and w.contains(10.0) and not w.contains(10.001)


def test_normalize_gradient_cutoff():
    """test_gradients.py:199-205: exactly zero at or below EPS_GRADIENT."""
    assert np.array_equal(vc.normalize_gradient((0.0, 0.0, 0.0)), np.zeros(3))
    assert np.array_equal(vc.normalize_gradient((vc.EPS_GRADIENT * 0.5, 0, 0)), np.zeros(3))
    assert vc.normalize_gradient((3.0, 0.0, 4.0)) == pytest.approx([0.6, 0.0, 0.8], abs=1e-15)
    assert np.linalg.norm(vc.normalize_gradient((1e-7, 0, 0))) == pytest.approx(1.0)
