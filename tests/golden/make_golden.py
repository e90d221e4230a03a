"""Generate golden fixtures by running the REFERENCE implementation.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Runs only in the build container (the reference does not exist on the GPU
box).  Writes tests/golden/golden.npz: for every case the input volume, the
scene spec (JSON), and the reference outputs -- frame pixels and
sample_count from render_frame(..., use_octree=False), raw gradients from
_kernels.grad_raw, samples from _kernels.sample_any, lattice gradient
volumes.  The float32 case calls _kernels.render_tile directly because
Volume.from_array truncates to uint16 (volume.py:71).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import voxelcast as vc  # noqa: E402  (the reference, via PYTHONPATH)
from voxelcast import _kernels as K  # noqa: E402
from voxelcast import raycast as R  # noqa: E402

assert "reference" in vc.__file__, f"expected the reference package, got {vc.__file__}"

from paper_1609_01317_b200 import phantoms  # noqa: E402  (numpy generators only)

OUT = Path(__file__).resolve().parent / "golden.npz"


def ref_scene(spec, dims, spacing):
    cam = spec["camera"]
    camera = vc.Camera(eye=tuple(cam["eye"]), target=tuple(cam["target"]),
                       up=tuple(cam.get("up", (0.0, 1.0, 0.0))), fov_y=cam.get("fov_y", 60.0),
                       azimuth=cam.get("azimuth", 0.0), elevation=cam.get("elevation", 0.0),
                       zoom=cam.get("zoom", 1.0))
    light = vc.Light(position=tuple(spec["light"]["position"]),
                     color=tuple(spec["light"].get("color", (1.0, 1.0, 1.0))))
    win = spec.get("window", (500.0, 4095.0))
    tf = spec.get("transfer")
    transfer = vc.TransferFunction.default_ct() if tf is None else vc.TransferFunction(
        points=[(p[0], tuple(p[1])) for p in tf["points"]], mu_water=tf.get("mu_water", 1000.0))
    clip = spec.get("clip")
    return vc.Scene(camera=camera, light=light, window=vc.ThresholdWindow(*win),
                    transfer=transfer,
                    clip=None if clip is None else vc.ClipBox(tuple(clip[0]), tuple(clip[1])))


def ref_settings(spec):
    s = dict(spec.get("settings", {}))
    kw = {}
    for key in ("width", "height", "coarse_step", "fine_step", "refine_iters", "mode"):
        if key in s:
            kw[key] = s[key]
    if "operator" in s:
        kw["operator"] = vc.OperatorKind(s["operator"])
    if "interpolation" in s:
        kw["interpolation"] = vc.InterpolationMode(s["interpolation"])
    if "background" in s:
        kw["background"] = tuple(s["background"])
    for key in ("use_adaptive", "adaptive_factor", "detail_epsilon", "octree_min_block",
                "octree_max_depth"):
        if key in s:
            kw[key] = s[key]
    return vc.RenderSettings(use_octree=bool(s.get("use_octree", False)), **kw)


def render_ref(arr, spacing, spec):
    """render_frame(use_octree=False) for integer grids; a direct
    _kernels.render_tile call for float32 grids (mirrors raycast.py:441-514)."""
    nz, ny, nx = arr.shape
    if arr.dtype != np.float32:
        vol = vc.Volume.from_array(arr, spacing=spacing)
        fb = vc.render_frame(vol, ref_scene(spec, (nx, ny, nz), spacing), ref_settings(spec), workers=8)
        return fb.pixels, fb.sample_count
    scene = ref_scene(spec, (nx, ny, nz), spacing)
    st = ref_settings(spec)
    sp = np.array(spacing, np.float64)
    basis = R.camera_basis(scene.camera, st.width, st.height)
    ext = np.array([n * s for n, s in zip((nx, ny, nz), spacing)])
    clip_lo, clip_hi = np.zeros(3), ext.copy()
    if scene.clip is not None:
        clip_lo = np.maximum(clip_lo, np.asarray(scene.clip.lo, np.float64))
        clip_hi = np.minimum(clip_hi, np.asarray(scene.clip.hi, np.float64))
    lut_hu, lut_rgba = scene.transfer.tables()
    nb, sm, ch = R._dummy_tree()
    pixels = np.zeros((st.height, st.width, 4), np.uint8)
    counter = np.zeros(1, np.int64)
    K.render_tile(arr.ravel(), nx, ny, nz, sp, basis.eye, basis.right, basis.up, basis.forward,
                  basis.half_w, basis.half_h, st.width, st.height, clip_lo, clip_hi,
                  np.array(scene.light.position, np.float64), np.array(scene.light.color, np.float64),
                  float(scene.window.low), float(scene.window.high), lut_hu, lut_rgba,
                  float(scene.transfer.mu_water), st.operator.code, st.interpolation.code,
                  K.MODE_SURFACE if st.mode == "surface" else K.MODE_COMPOSITED,
                  float(st.coarse_step), float(st.fine_step), int(st.refine_iters),
                  np.array(st.background, np.float64), 0, nb, sm, ch, 0, 1, 1.0,
                  0, st.height, pixels, counter, np.empty(512, np.int32), np.empty(4096), np.empty(4096))
    return pixels, int(counter[0])


def default_spec(dims, spacing=(1.0, 1.0, 1.0)):
    ext = tuple(n * s for n, s in zip(dims, spacing))
    center = tuple(e / 2.0 for e in ext)
    dist = 1.1 * max(ext) / 2.0
    eye = (center[0], center[1], center[2] - dist)
    return {"camera": {"eye": eye, "target": center}, "light": {"position": eye}}


def with_(spec, **kw):
    out = json.loads(json.dumps(spec))
    for k, v in kw.items():
        if k == "settings":
            out.setdefault("settings", {}).update(v)
        elif k == "camera":
            out["camera"].update(v)
        else:
            out[k] = v
    return out


CT_TF = {"points": [[-1000.0, [0.0, 0.0, 0.0, 0.0]], [-100.0, [0.8, 0.3, 0.25, 0.35]],
                    [500.0, [0.95, 0.93, 0.88, 1.0]], [1500.0, [1.0, 1.0, 1.0, 1.0]]]}
U8_TF = dict(CT_TF, mu_water=100.0)


def frame_cases():
    cases = []
    rng = np.random.default_rng(99)
    noise16 = rng.integers(0, 4096, size=(16, 16, 16), dtype=np.uint16)
    sphere32 = vc.make_phantom("sphere", 32, radius=10).as_array().copy()
    shell32 = vc.make_phantom("shell", 32, r_inner=8, r_outer=12).as_array().copy()
    d32 = default_spec((32, 32, 32))

    cases.append(("sphere32_cd_surface", sphere32, (1.0, 1.0, 1.0),
                  with_(d32, settings={"width": 64, "height": 64})))
    cases.append(("sphere32_zh_composited", sphere32, (1.0, 1.0, 1.0),
                  with_(d32, settings={"width": 64, "height": 64, "operator": "zucker-hummel",
                                       "mode": "composited"})))
    cases.append(("sphere32_sobel_orbit", sphere32, (1.0, 1.0, 1.0),
                  with_(d32, camera={"azimuth": 37.0, "elevation": 21.0, "zoom": 1.3},
                        settings={"width": 48, "height": 40, "operator": "sobel3d",
                                  "background": [0.25, 0.5, 0.75, 1.0]})))
    cases.append(("shell32_sobel_band", shell32, (1.0, 1.0, 1.0),
                  with_(d32, window=[400.0, 600.0],
                        settings={"width": 64, "height": 48, "operator": "sobel3d"})))
    cases.append(("shell32_zh_composited_band", shell32, (1.0, 1.0, 1.0),
                  with_(d32, window=[400.0, 600.0],
                        settings={"width": 48, "height": 48, "operator": "zucker-hummel",
                                  "mode": "composited", "background": [0.1, 0.2, 0.3, 0.0]})))
    # camera inside the shell material, light elsewhere (test_render.py:175-187)
    c = 16.0
    cases.append(("shell32_inside_camera", shell32, (1.0, 1.0, 1.0),
                  {"camera": {"eye": [c + 12.0, c, c], "target": [c, c, c]},
                   "light": {"position": [100.0, 100.0, 100.0]},
                   "settings": {"width": 32, "height": 32, "background": [0.0, 0.0, 0.25, 1.0]}}))
    d16 = default_spec((16, 16, 16))
    for op in ("central", "sobel3d", "zucker-hummel"):
        cases.append((f"noise16_{op}_composited", noise16, (1.0, 1.0, 1.0),
                      with_(d16, window=[1500.0, 4095.0], camera={"azimuth": 30.0, "elevation": 20.0},
                            settings={"width": 40, "height": 32, "operator": op,
                                      "mode": "composited"})))
    for interp in ("nearest", "linear"):
        cases.append((f"sphere32_{interp}", sphere32, (1.0, 1.0, 1.0),
                      with_(d32, camera={"azimuth": 15.0},
                            settings={"width": 40, "height": 40, "interpolation": interp,
                                      "operator": "sobel3d", "mode": "composited"})))
    # anisotropic spacing (division path), clip box, coarse/fine/refine variants
    sp = (1.0, 0.75, 1.25)
    dsp = default_spec((32, 32, 32), sp)
    cases.append(("sphere32_spacing_clip", sphere32, sp,
                  with_(dsp, clip=[[0.0, 0.0, 0.0], [18.0, 1e9, 1e9]], camera={"azimuth": 10.0},
                        settings={"width": 48, "height": 48, "operator": "central",
                                  "coarse_step": 0.7, "fine_step": 0.1, "refine_iters": 9,
                                  "background": [0.0, 0.0, 0.25, 1.0]})))
    cases.append(("sphere32_pow2_spacing", sphere32, (0.5, 2.0, 1.0),
                  with_(default_spec((32, 32, 32), (0.5, 2.0, 1.0)), camera={"elevation": -25.0},
                        settings={"width": 40, "height": 40, "operator": "zucker-hummel",
                                  "mode": "composited", "refine_iters": 0})))
    # BASELINE config C1 at full size: 64^3 u8 sphere, 256^2, CD, surface
    c1 = phantoms.sphere_c1(64).as_array().copy()
    cases.append(("c1_sphere64_u8", c1, (1.0, 1.0, 1.0),
                  with_(default_spec((64, 64, 64)), window=[100.0, 255.0], transfer=U8_TF,
                        settings={"width": 256, "height": 256, "operator": "central"})))
    ml = phantoms.marschner_lobb(32).as_array().copy()
    cases.append(("ml32_u8_sobel", ml, (1.0, 1.0, 1.0),
                  with_(d32, window=[128.0, 255.0], transfer=U8_TF, camera={"azimuth": 30.0},
                        settings={"width": 64, "height": 64, "operator": "sobel3d"})))
    ct = phantoms.ct_phantom(48).as_array().copy()
    d48 = default_spec((48, 48, 48))
    cases.append(("ct48_zh_composited", ct, (1.0, 1.0, 1.0),
                  with_(d48, camera={"azimuth": 20.0, "elevation": 10.0},
                        settings={"width": 64, "height": 48, "operator": "zucker-hummel",
                                  "mode": "composited"})))
    for az in (0.0, 90.0, 180.0, 270.0):
        cases.append((f"ct48_cd_surface_az{int(az)}", ct, (1.0, 1.0, 1.0),
                      with_(d48, camera={"azimuth": az},
                            settings={"width": 32, "height": 24, "operator": "central"})))
    fb = phantoms.fbm_noise(24, octaves=3, base_cells=2).as_array().copy()
    assert fb.dtype == np.float32 and not np.all(fb == np.round(fb))
    cases.append(("fbm24_f32_sobel_composited", fb, (1.0, 1.0, 1.0),
                  with_(default_spec((24, 24, 24)), window=[2600.0, 4095.0],
                        camera={"azimuth": 45.0},
                        settings={"width": 40, "height": 40, "operator": "sobel3d",
                                  "mode": "composited"})))
    # adaptive stride (use_adaptive, _kernels.py:437-463) -- test_render.py:142-152 scene
    sph8 = vc.make_phantom("sphere", 64, radius=8).as_array().copy()
    d64 = default_spec((64, 64, 64))
    for oct_on in (False, True):
        cases.append((f"adaptive_sphere64_octree{int(oct_on)}", sph8, (1.0, 1.0, 1.0),
                      with_(d64, settings={"width": 64, "height": 64, "use_adaptive": True,
                                           "adaptive_factor": 4, "use_octree": oct_on})))
        cases.append((f"adaptive_ct48_zh_composited_octree{int(oct_on)}", ct, (1.0, 1.0, 1.0),
                      with_(d48, camera={"azimuth": 20.0, "elevation": 10.0},
                            settings={"width": 64, "height": 48, "operator": "zucker-hummel",
                                      "mode": "composited", "use_adaptive": True,
                                      "adaptive_factor": 3, "use_octree": oct_on})))
    cases.append(("adaptive_noise16_detail", noise16, (1.0, 1.0, 1.0),
                  with_(d16, window=[3000.0, 4095.0], camera={"azimuth": 30.0},
                        settings={"width": 40, "height": 32, "operator": "sobel3d",
                                  "use_adaptive": True, "adaptive_factor": 3,
                                  "detail_epsilon": 3500.0, "octree_min_block": 2})))
    # 0 inside the threshold window with use_octree (the reference default):
    # samples in the half-voxel border band read 0 (_kernels.py:121-122) and
    # are in-window, but collect_segments skips the border leaves whose padded
    # range misses the window -- the reference's octree image differs from
    # its brute-force image.  A 2000-valued block with a zero-valued hole.
    zc = np.arange(32, dtype=np.float64)
    zz, zy, zx = np.meshgrid(zc, zc, zc, indexing="ij")
    block = np.where((zx - 15.5) ** 2 + (zy - 15.5) ** 2 + (zz - 15.5) ** 2 <= 10.0 ** 2,
                     0, 2000).astype(np.uint16)
    zero_tf = {"points": [[-1000.0, [0.9, 0.6, 0.3, 0.6]], [0.0, [0.5, 0.7, 0.4, 0.8]],
                          [1000.0, [0.2, 0.4, 0.9, 1.0]]]}
    for oct_on in (False, True):
        for mode, op in (("surface", "sobel3d"), ("composited", "central")):
            cases.append((f"zerowin_block32_{mode}_octree{int(oct_on)}", block, (1.0, 1.0, 1.0),
                          with_(d32, window=[-100.0, 500.0], transfer=zero_tf,
                                camera={"azimuth": 8.0, "elevation": 5.0},
                                settings={"width": 48, "height": 40, "operator": op, "mode": mode,
                                          "use_octree": oct_on})))
    empty = np.zeros((16, 16, 16), np.uint16)
    cases.append(("empty16", empty, (1.0, 1.0, 1.0),
                  with_(d16, settings={"width": 24, "height": 24,
                                       "background": [0.25, 0.5, 0.75, 1.0]})))
    return cases


def main():
    store = {}
    index = []
    for name, arr, spacing, spec in frame_cases():
        px, cnt = render_ref(arr, spacing, spec)
        store[f"{name}/volume"] = arr
        store[f"{name}/pixels"] = px
        store[f"{name}/count"] = np.array(cnt, np.int64)
        index.append({"name": name, "kind": "frame", "spacing": list(spacing), "spec": spec})
        print(f"{name}: {arr.dtype}{arr.shape} -> {px.shape} count={cnt}")

    # point queries on noise16 (conftest.py noise_volume16) and the ramp
    rng = np.random.default_rng(20240817)
    noise16 = np.random.default_rng(99).integers(0, 4096, size=(16, 16, 16), dtype=np.uint16)
    pts = np.concatenate([
        rng.uniform(-1.0, 16.0, (400, 3)),
        rng.integers(0, 16, (100, 3)).astype(np.float64),
        np.array([[15.0, 7.2, 3.8], [0.0, 0.0, 0.0], [15.0, 15.0, 15.0], [1.5, 2.0, 3.0],
                  [7.5, 7.5, 7.5], [-0.0, 3.0, 3.0], [15.0000001, 3, 3], [2.5, 2.5, 2.5]]),
    ])
    store["points/noise16"] = noise16
    store["points/pts"] = pts
    data = noise16.ravel()
    for interp, code in (("nearest", 0), ("linear", 1), ("trilinear", 2)):
        store[f"points/sample_{interp}"] = np.array(
            [K.sample_any(data, 16, 16, 16, *p, code) for p in pts])
    gpts = np.concatenate([rng.uniform(-1.5, 16.5, (300, 3)),
                           rng.integers(0, 16, (100, 3)).astype(np.float64)])
    store["points/gpts"] = gpts
    for op, code in (("central", 0), ("sobel3d", 1), ("zucker-hummel", 2)):
        store[f"points/grad_{op}"] = np.array([K.grad_raw(data, 16, 16, 16, *p, code) for p in gpts])
        lat = np.zeros((16, 16, 16, 3))
        for k in range(16):
            for j in range(16):
                for i in range(16):
                    lat[k, j, i] = K.grad_raw(data, 16, 16, 16, float(i), float(j), float(k), code)
        store[f"lattice/noise16_{op}"] = lat
    json_index = json.dumps(index)
    store["index"] = np.frombuffer(json_index.encode(), np.uint8)
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB)")


if __name__ == "__main__":
    main()
