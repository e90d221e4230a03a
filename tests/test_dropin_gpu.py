"""The drop-in at the reference's kernel contract, on the device.

* voxelcast._kernels.{sample_any, grad_raw} against the reference's point
  goldens (bit-exact);
* voxelcast._kernels.render_tile driven the way raycast.render_frame
  drives it (raycast.py:476-505: 16-row bands from a thread pool, every
  argument in the reference's form and order) against the reference's
  frame goldens -- pixels and the summed sample count;
* the reference's OWN render_frame / sample / gradient host code,
  unmodified, from its install in baseline/_ref (bench.py's reference arm
  installs it; skipped where it is absent), with its kernel module swapped
  for voxelcast._kernels: the reference's Python renders on the GPU and
  gives the reference's pixels.  This is INTEGRATION.md's Option B as a
  running test.
"""

from __future__ import annotations

import importlib.util
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

import voxelcast
from voxelcast import _kernels as K
from paper_1609_01317_b200 import octree as impl_octree
from paper_1609_01317_b200.raycast import camera_basis
from tests.conftest import ROOT, frame_names, zero_window_frames
from tests.specs import product_scene, product_settings, product_volume

pytestmark = pytest.mark.gpu

REF_INSTALL = ROOT / "baseline" / "_ref" / "voxelcast"


@pytest.mark.parametrize("interp", ["nearest", "linear", "trilinear"])
def test_kernel_sample_any_bit_exact(golden, interp):
    data = np.ascontiguousarray(golden["points/noise16"]).ravel()
    data.setflags(write=False)
    code = {"nearest": 0, "linear": 1, "trilinear": 2}[interp]
    got = np.array([K.sample_any(data, 16, 16, 16, *p, code) for p in golden["points/pts"][:120]])
    assert np.array_equal(got, golden[f"points/sample_{interp}"][:120])


@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_kernel_grad_raw_bit_exact(golden, op):
    data = np.ascontiguousarray(golden["points/noise16"]).ravel()
    data.setflags(write=False)
    code = {"central": 0, "sobel3d": 1, "zucker-hummel": 2}[op]
    got = np.array([K.grad_raw(data, 16, 16, 16, *p, code) for p in golden["points/gpts"][:120]])
    assert np.array_equal(got, golden[f"points/grad_{op}"][:120])
    # a writable array is read afresh on every call
    w = data.copy()
    assert K.grad_raw(w, 16, 16, 16, 7.0, 7.0, 7.0, code) == K.grad_raw(data, 16, 16, 16, 7.0, 7.0, 7.0, code)
    w[:] = 0
    assert K.grad_raw(w, 16, 16, 16, 7.0, 7.0, 7.0, code) == (0.0, 0.0, 0.0)


def _render_like_reference(arr, spacing, spec, tile_rows=16, use_octree=None, workers=8):
    """raycast.render_frame's host side (raycast.py:441-514) over
    voxelcast._kernels.render_tile, argument for argument."""
    vol = product_volume(arr, spacing)
    scene = product_scene(spec)
    st = product_settings(spec)
    if use_octree is not None:
        from dataclasses import replace

        st = replace(st, use_octree=use_octree)
    nx, ny, nz = vol.dims
    sp = np.array(vol.spacing, np.float64)
    basis = camera_basis(scene.camera, st.width, st.height)
    clip_lo, clip_hi = np.zeros(3), np.array(vol.extent, np.float64)
    if scene.clip is not None:
        clip_lo = np.maximum(clip_lo, np.asarray(scene.clip.lo, np.float64))
        clip_hi = np.minimum(clip_hi, np.asarray(scene.clip.hi, np.float64))
    lut_hu, lut_rgba = scene.transfer.tables()
    if st.use_octree or st.use_adaptive:
        tree = impl_octree.build_octree(vol, min_block=st.octree_min_block, max_depth=st.octree_max_depth)
        nb, _, sm, ch = impl_octree.flat_arrays(tree)
    else:
        nb, sm, ch = np.zeros((1, 6), np.int32), np.zeros((1, 2)), np.full((1, 8), -1, np.int32)
    eps = st.detail_epsilon
    if eps is None:
        eps = 0.01 * max(1, vol.value_max - vol.value_min)
    pixels = np.zeros((st.height, st.width, 4), np.uint8)
    bands = [(y, min(y + tile_rows, st.height)) for y in range(0, st.height, tile_rows)]
    counters = [np.zeros(1, np.int64) for _ in bands]

    def run_band(i):
        y0, y1 = bands[i]
        K.render_tile(vol.data, nx, ny, nz, sp, basis.eye, basis.right, basis.up, basis.forward,
                      basis.half_w, basis.half_h, st.width, st.height, clip_lo, clip_hi,
                      np.array(scene.light.position, np.float64), np.array(scene.light.color, np.float64),
                      float(scene.window.low), float(scene.window.high), lut_hu, lut_rgba,
                      float(scene.transfer.mu_water), st.operator.code, st.interpolation.code,
                      K.MODE_SURFACE if st.mode == "surface" else K.MODE_COMPOSITED,
                      float(st.coarse_step), float(st.fine_step), int(st.refine_iters),
                      np.array(st.background, np.float64), 1 if st.use_octree else 0, nb, sm, ch,
                      1 if st.use_adaptive else 0, int(st.adaptive_factor), float(eps), y0, y1, pixels,
                      counters[i], np.empty(512, np.int32), np.empty(4096), np.empty(4096))

    with ThreadPoolExecutor(max_workers=workers) as pool:
        list(pool.map(run_band, range(len(bands))))
    return pixels, int(sum(int(c[0]) for c in counters))


@pytest.mark.parametrize("name", frame_names())
def test_render_tile_bands_match_reference_frames(golden, name):
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    s = spec.get("settings", {})
    octree = bool(s.get("use_octree")) and bool(s.get("use_adaptive"))  # as the reference rendered it
    px, count = _render_like_reference(arr, spacing, spec, use_octree=octree)
    assert np.array_equal(px, want_px)
    assert count == want_count
    # use_octree on: macrocell skipping, the same pixels
    px2, _ = _render_like_reference(arr, spacing, spec, tile_rows=7, use_octree=True)
    assert np.array_equal(px2, want_px)


@pytest.mark.parametrize("name", zero_window_frames())
def test_render_tile_replays_reference_octree_with_zero_in_window(golden, name):
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    px, count = _render_like_reference(arr, spacing, spec)
    assert np.array_equal(px, want_px)
    assert count == want_count


# ---------------------------------------------------------------- the reference's own host code

def _load_reference(alias: str = "voxelcast_reference"):
    if alias in sys.modules:
        return sys.modules[alias]
    spec = importlib.util.spec_from_file_location(alias, REF_INSTALL / "__init__.py",
                                                  submodule_search_locations=[str(REF_INSTALL)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules[alias] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.fixture(scope="module")
def reference_on_b200():
    """The installed reference package with its kernel module replaced by
    voxelcast._kernels in every module that calls it."""
    if not (REF_INSTALL / "raycast.py").exists():
        pytest.skip("reference install baseline/_ref absent (bench.py --impl reference installs it)")
    pytest.importorskip("numba")
    ref = _load_reference()
    saved = {}
    for sub in ("raycast", "volume", "gradients"):
        m = sys.modules[f"{ref.__name__}.{sub}"]
        saved[sub] = m._k
        m._k = K
    yield ref
    for sub, k in saved.items():
        sys.modules[f"{ref.__name__}.{sub}"]._k = k


def _ref_scene(ref, spec):
    cam = spec["camera"]
    tf = spec.get("transfer")
    return ref.Scene(
        camera=ref.Camera(eye=tuple(cam["eye"]), target=tuple(cam["target"]),
                          up=tuple(cam.get("up", (0.0, 1.0, 0.0))), fov_y=cam.get("fov_y", 60.0),
                          azimuth=cam.get("azimuth", 0.0), elevation=cam.get("elevation", 0.0),
                          zoom=cam.get("zoom", 1.0)),
        light=ref.Light(position=tuple(spec["light"]["position"]),
                        color=tuple(spec["light"].get("color", (1.0, 1.0, 1.0)))),
        window=ref.ThresholdWindow(*spec.get("window", (500.0, 4095.0))),
        transfer=ref.TransferFunction.default_ct() if tf is None else ref.TransferFunction(
            points=[(p[0], tuple(p[1])) for p in tf["points"]], mu_water=tf.get("mu_water", 1000.0)),
        clip=None if spec.get("clip") is None else ref.ClipBox(tuple(spec["clip"][0]), tuple(spec["clip"][1])))


def _ref_settings(ref, spec, **over):
    s = dict(spec.get("settings", {}))
    kw = {k: s[k] for k in ("width", "height", "coarse_step", "fine_step", "refine_iters", "mode",
                            "use_adaptive", "adaptive_factor", "detail_epsilon", "octree_min_block",
                            "octree_max_depth") if k in s}
    if "operator" in s:
        kw["operator"] = ref.OperatorKind(s["operator"])
    if "interpolation" in s:
        kw["interpolation"] = ref.InterpolationMode(s["interpolation"])
    if "background" in s:
        kw["background"] = tuple(s["background"])
    kw["use_octree"] = bool(s.get("use_octree", False))
    kw.update(over)
    return ref.RenderSettings(**kw)


@pytest.mark.parametrize("name", [n for n in frame_names() if "f32" not in n] + zero_window_frames())
def test_reference_render_frame_runs_on_the_b200_kernels(golden, reference_on_b200, name):
    """The reference's unmodified raycast.render_frame (validation, camera
    basis, clip box, LUT tables, octree build, 16-row bands on its thread
    pool) calling voxelcast._kernels.render_tile: the reference's pixels and
    sample count.  (Float32 grids cannot enter the reference's Volume,
    which stores uint16 -- volume.py:71.)"""
    ref = reference_on_b200
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    vol = ref.Volume.from_array(arr, spacing=spacing)
    fb = ref.render_frame(vol, _ref_scene(ref, spec), _ref_settings(ref, spec))
    assert np.array_equal(fb.pixels, want_px)
    s = spec.get("settings", {})
    if not s.get("use_octree") or s.get("use_adaptive") or name in zero_window_frames():
        assert fb.sample_count == want_count  # the device replays the reference's walk
    # the reference's default use_octree=True: its octree handed to the device
    fb2 = ref.render_frame(vol, _ref_scene(ref, spec), _ref_settings(ref, spec, use_octree=True))
    if name not in zero_window_frames():
        assert np.array_equal(fb2.pixels, want_px)


def test_reference_point_api_runs_on_the_b200_kernels(golden, reference_on_b200):
    ref = reference_on_b200
    vol = ref.Volume.from_array(golden["points/noise16"])
    for p, want in zip(golden["points/pts"][:50], golden["points/sample_trilinear"][:50]):
        assert ref.sample(vol, tuple(p), ref.InterpolationMode.TRILINEAR) == want
    for p, want in zip(golden["points/gpts"][:50], golden["points/grad_sobel3d"][:50]):
        g = ref.gradient(vol, tuple(p), "sobel3d")
        assert np.array_equal(g, np.array(K.normalize3(*want, K.GRAD_EPS)))
    assert voxelcast.gradient is not ref.gradient
