"""CPU tests: C-ABI library loads and exports the header's symbols, the host
mirror of the reference API validates like the reference, and the product
path refuses to run without a GPU (no CPU fallback)."""

from __future__ import annotations

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from oracle import oracle
from paper_1609_01317_b200 import _native
from paper_1609_01317_b200.raycast import render_params

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "voxelcast_b200.h").read_text()
    return sorted(set(re.findall(r"^VC_API\s+[\w\s\*]+?\b(vc_\w+)\s*\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    L = _native.load()
    syms = header_symbols()
    assert len(syms) >= 18
    assert set(syms) == set(_native.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    assert L.vc_abi_version() == 4
    assert L.vc_render_params_size() == ctypes.sizeof(_native.RenderParams)


def test_library_is_sm100a():
    """The shipped library carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess

    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(_native.library_path())], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    if _native.device_count() > 0:
        pytest.skip("a CUDA device is present")
    vol = vc.make_phantom("sphere", 8, radius=3)
    with pytest.raises(RuntimeError):
        vc.render_frame(vol, vc.default_scene(vol), vc.RenderSettings(width=4, height=4))
    with pytest.raises(RuntimeError):
        vc.sample(vol, (1.0, 1.0, 1.0))


def test_camera_basis_matches_oracle_restatement():
    rng = np.random.default_rng(11)
    for _ in range(50):
        eye = tuple(rng.uniform(-50, 50, 3))
        target = tuple(rng.uniform(-5, 5, 3))
        cam = vc.Camera(eye=eye, target=target, fov_y=float(rng.uniform(10, 120)),
                        azimuth=float(rng.uniform(-180, 180)), elevation=float(rng.uniform(-100, 100)),
                        zoom=float(rng.uniform(0.5, 3)))
        b = vc.camera_basis(cam, 320, 200)
        o = oracle.camera_basis({"eye": eye, "target": target, "fov_y": cam.fov_y,
                                 "azimuth": cam.azimuth, "elevation": cam.elevation,
                                 "zoom": cam.zoom}, 320, 200)
        for got, want in zip((b.eye, b.right, b.up, b.forward, b.half_w, b.half_h), o):
            assert np.array_equal(np.asarray(got), np.asarray(want))


def test_render_params_block_mirrors_scene():
    vol = vc.make_phantom("sphere", 16, radius=5)
    sc = vc.default_scene(vol)
    st = vc.RenderSettings(width=33, height=17, operator=vc.OperatorKind.ZUCKER_HUMMEL,
                           mode="composited", background=(0.1, 0.2, 0.3, 0.4), use_octree=False,
                           gradient_source="volume")
    P = render_params(vol, sc, st)
    assert (P.width, P.height, P.op, P.mode, P.interp) == (33, 17, 2, 1, 2)
    assert (P.band_rows, P.band_first, P.band_step) == (17, 0, 1)
    assert P.skip_empty == 0 and P.grad_source == _native.VC_GRAD_VOLUME
    assert P.lut_n == 4 and list(P.lut_hu[:4]) == [-1000.0, -100.0, 500.0, 1500.0]
    assert list(P.clip_hi) == [16.0, 16.0, 16.0]
    assert (P.t_low, P.t_high, P.mu_water) == (500.0, 4095.0, 1000.0)


def test_render_settings_validation_matches_reference():
    """test_render.py:197-207 plus the new gradient_source field."""
    with pytest.raises(ValueError):
        vc.RenderSettings(width=0)
    with pytest.raises(ValueError):
        vc.RenderSettings(fine_step=2.0, coarse_step=1.0)
    with pytest.raises(ValueError):
        vc.RenderSettings(mode="xray")
    with pytest.raises(ValueError):
        vc.RenderSettings(adaptive_factor=0)
    with pytest.raises(ValueError):
        vc.RenderSettings(background=(2, 0, 0, 1))
    with pytest.raises(ValueError):
        vc.RenderSettings(gradient_source="magic")


def test_scene_type_validation_matches_reference():
    with pytest.raises(ValueError):
        vc.Camera(eye=(1, 1, 1), target=(1, 1, 1))
    with pytest.raises(ValueError):
        vc.Camera(eye=(0, 0, 1), target=(0, 0, 0), fov_y=180.0)
    with pytest.raises(ValueError):
        vc.Camera(eye=(0, 0, 1), target=(0, 0, 0), zoom=0.0)
    with pytest.raises(ValueError):
        vc.Light(position=(0, 0, 0), color=(1.5, 0, 0))
    with pytest.raises(ValueError):
        vc.ThresholdWindow(10.0, 5.0)
    with pytest.raises(ValueError):
        vc.TransferFunction(points=[])
    with pytest.raises(ValueError):
        vc.TransferFunction(points=[(0.0, (0, 0, 0, 0)), (0.0, (1, 1, 1, 1))])
    with pytest.raises(ValueError):
        vc.TransferFunction(points=[(0.0, (0, 0, 0, 0))], mu_water=0.0)
    with pytest.raises(ValueError):
        vc.ClipBox(lo=(1, 0, 0), hi=(0, 1, 1))


def test_volume_from_array_matches_reference_semantics():
    arr = np.arange(24, dtype=np.int64).reshape(2, 3, 4)
    v = vc.Volume.from_array(arr, spacing=(1.0, 2.0, 0.5))
    assert v.dims == (4, 3, 2) and v.data.dtype == np.uint16
    assert v.extent == (4.0, 6.0, 1.0)
    assert v.value_at(3, 2, 1) == 23 and v.value_min == 0 and v.value_max == 23
    assert not v.data.flags.writeable
    with pytest.raises(ValueError):
        vc.Volume.from_array(np.zeros((2, 2)))
    with pytest.raises(ValueError):
        vc.Volume.from_array(np.zeros((0, 2, 2)))
    with pytest.raises(ValueError):
        vc.Volume.from_array(np.zeros((2, 2, 2)), spacing=(1, 0, 1))
    with pytest.raises(IndexError):
        v.value_at(4, 0, 0)
    v8 = vc.Volume.from_array(arr, dtype=np.uint8)
    assert v8.data.dtype == np.uint8
    with pytest.raises(ValueError):  # 1000 would wrap to 232 in uint8 storage
        vc.Volume.from_array(np.full((2, 2, 2), 1000), dtype=np.uint8)
    with pytest.raises(ValueError):
        vc.make_phantom("sphere", 16, radius=6, dtype=np.uint8)
    assert vc.Volume.from_array(np.full((2, 2, 2), 70000)).value_max == 70000 - 65536  # as the reference
    with pytest.raises(ValueError):
        vc.Volume.from_array(arr, dtype=np.int32)


def test_phantom_factory_matches_reference_rules():
    s = vc.make_phantom("sphere", 16, radius=6)
    assert s.value_max == 1000 and s.value_min == 0
    with pytest.raises(ValueError):
        vc.make_phantom("sphere", 16, radius=9)
    with pytest.raises(ValueError):
        vc.make_phantom("shell", 16, r_inner=5, r_outer=4)
    with pytest.raises(ValueError):
        vc.make_phantom("ramp", 8, axis=3)
    with pytest.raises(ValueError):
        vc.make_phantom("sphere", 8, radius=2, bogus=1)
    r = vc.make_phantom("ramp", 16, axis=1, scale=2.0)
    assert r.value_at(0, 5, 0) == 10


def test_host_helpers_known_answers():
    """test_raycast_pipeline.py:193-291 (host-side helpers)."""
    assert vc.hounsfield(1000.0, 1000.0) == 0.0
    assert vc.hounsfield(0.0, 1000.0) == -1000.0
    with pytest.raises(ValueError):
        vc.hounsfield(100.0, 0.0)
    tf = vc.TransferFunction.default_ct()
    for hu, rgba in tf.points:
        assert vc.transfer(tf, hu) == pytest.approx(rgba, abs=0.0)
    tf2 = vc.TransferFunction(points=[(0.0, (0, 0, 0, 0)), (100.0, (1, 0.5, 0.25, 1))])
    assert vc.transfer(tf2, 50.0) == pytest.approx([0.5, 0.25, 0.125, 0.5], abs=1e-12)
    assert vc.composite_step((0.2, 0.4, 0.6), (1.0, 0.5, 0.0), 1.0) == pytest.approx([1.0, 0.5, 0.0])
    light = vc.Light(position=(math.sin(math.radians(60)) * 10, 0, math.cos(math.radians(60)) * 10))
    assert vc.shade((0, 0, 0), (0, 0, 1), light) == pytest.approx([0.5, 0.5, 0.5], abs=1e-9)
    assert np.array_equal(vc.normalize_gradient((0.0, 0.0, 0.0)), np.zeros(3))
    assert vc.normalize_gradient((3.0, 0.0, 4.0)) == pytest.approx([0.6, 0.0, 0.8], abs=1e-15)
    assert vc.lerp(2.0, 10.0, 1.0) == 10.0


def test_generate_ray_matches_reference_kats():
    """test_raycast_geometry.py:13-56."""
    cam = vc.Camera(eye=(0, 0, -10), target=(0, 0, 5))
    r = vc.generate_ray(cam, 50, 50, 101, 101)
    assert r.direction == pytest.approx([0, 0, 1], abs=1e-12)
    cam = vc.Camera(eye=(0, 0, -10), target=(0, 0, 0), fov_y=60)
    r = vc.generate_ray(cam, 50, 0, 101, 101)
    want = math.atan((1.0 - 2.0 * 0.5 / 101) * math.tan(math.radians(30)))
    assert math.atan2(r.direction[1], r.direction[2]) == pytest.approx(want, abs=1e-12)
    with pytest.raises(ValueError):
        vc.generate_ray(cam, 101, 0, 101, 101)
    cam = vc.Camera(eye=(0, 0, 10), target=(0, 0, 0), azimuth=90.0)
    assert vc.generate_ray(cam, 8, 8, 17, 17).origin == pytest.approx([10, 0, 0], abs=1e-9)


def test_cross3_is_np_cross_bit_for_bit():
    """camera_basis's hand-written 3-vector cross product equals np.cross
    bit for bit (signed zeros included): the device consumes the basis."""
    from paper_1609_01317_b200.raycast import _cross3

    rng = np.random.default_rng(7)
    vecs = [rng.normal(size=3) * s for s in (1e-300, 1e-8, 1.0, 1e8, 1e300) for _ in range(400)]
    vecs += [np.array(v, np.float64) for v in ((0.0, -0.0, 1.0), (-0.0, 0.0, -0.0), (1.0, 0.0, 0.0),
                                               (0.0, 1.0, 0.0), (-1.0, -0.0, 2.0))]
    for a, b in zip(vecs, vecs[::-1]):
        want = np.cross(a, b)
        got = _cross3(a, b)
        assert np.array_equal(want.view(np.int64), got.view(np.int64)), (a, b)
