"""The reference package's own behavioural tests, restated against this
package (every render, gradient query and single-ray march below runs on
the device through the C ABI).

Sources, one section each: pkg/tests/test_render.py,
pkg/tests/test_gradients.py, pkg/tests/test_raycast_pipeline.py,
test_raycast_geometry.py (the device-backed helpers), the sampler half of
test_volume.py and the on-path guarantees of test_acceptance.py.  The assertions and tolerances are the
reference's; the fixtures and structure are this suite's."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from paper_1609_01317_b200.gradients import grad_raw_points

pytestmark = pytest.mark.gpu

WINDOW = vc.ThresholdWindow(500.0, 4095.0)


def settings(**kw) -> vc.RenderSettings:
    kw.setdefault("width", 64)
    kw.setdefault("height", 64)
    return vc.RenderSettings(**kw)


@pytest.fixture(scope="module")
def ball():
    return vc.make_phantom("sphere", 32, radius=10)


@pytest.fixture(scope="module")
def ball_scene(ball):
    return vc.default_scene(ball)


# ---------------------------------------------------------------- test_render.py


def test_framebuffer_fields(ball, ball_scene):
    """test_render.py:67-74"""
    fb = vc.render_frame(ball, ball_scene, settings(width=40, height=24))
    assert (fb.width, fb.height) == (40, 24)
    assert fb.pixels.shape == (24, 40, 4) and fb.pixels.dtype == np.uint8
    assert fb.render_ms > 0 and fb.sample_count > 0
    assert fb.rgb().shape == (24, 40, 3)


def test_lit_centre_outshines_silhouette(ball):
    """test_render.py:77-92: head-on light, the centre pixel of the sphere
    is more than twice as bright as the last hit pixel of its row."""
    eye = (16.0, 16.0, -30.0)
    sc = vc.Scene(camera=vc.Camera(eye=eye, target=(16.0, 16.0, 16.0)), light=vc.Light(position=eye))
    px = vc.render_frame(ball, sc, settings(background=(0, 0, 0, 0))).pixels
    hit = px[:, :, 3] == 255
    assert hit.any() and not hit.all() and hit[32, 32]
    rim = int(np.nonzero(hit[32])[0].max())
    assert int(px[32, 32, :3].astype(int).sum()) > 2 * int(px[32, rim, :3].astype(int).sum())


def _opaque(points=((-1000.0, (0.1, 0.2, 0.3, 1.0)), (0.0, (0.9, 0.8, 0.7, 1.0)),
                    (1000.0, (1.0, 1.0, 1.0, 1.0)))):
    return vc.TransferFunction(points=list(points))


def test_opaque_transfer_composites_to_the_surface_image(ball, ball_scene):
    """test_render.py:95-104: alpha 1 everywhere, so compositing stops at
    the first shade and equals surface mode bit for bit."""
    sc = vc.Scene(camera=ball_scene.camera, light=ball_scene.light, window=ball_scene.window,
                  transfer=_opaque())
    surf = vc.render_frame(ball, sc, settings(mode=vc.RenderMode.SURFACE)).pixels
    comp = vc.render_frame(ball, sc, settings(mode=vc.RenderMode.COMPOSITED)).pixels
    assert np.array_equal(surf, comp)
    # and with the default (translucent) transfer the two modes differ (:107-110)
    surf = vc.render_frame(ball, ball_scene, settings(mode=vc.RenderMode.SURFACE)).pixels
    comp = vc.render_frame(ball, ball_scene, settings(mode=vc.RenderMode.COMPOSITED)).pixels
    assert not np.array_equal(surf, comp)


@pytest.mark.parametrize("knob", [{"workers": 1}, {"workers": 2}, {"workers": 4}, {"tile_rows": 5},
                                  {"tile_rows": 64}])
def test_scheduling_knobs_never_change_pixels(ball, ball_scene, knob):
    """test_render.py:113-125 (worker count, tile height)."""
    want = vc.render_frame(ball, ball_scene, settings()).pixels
    if "workers" in knob:
        got = vc.render_frame(ball, ball_scene, settings(), workers=knob["workers"]).pixels
    else:
        got = vc.render_frame(ball, ball_scene, settings(tile_rows=knob["tile_rows"])).pixels
    assert np.array_equal(got, want)


def test_skipping_identity_sphere_and_shell(ball, ball_scene):
    """test_render.py:128-143: empty-space skipping returns the brute-force
    image (fewer fetches) on a sphere, and on a shell for a high and a band
    window."""
    on = vc.render_frame(ball, ball_scene, settings(use_octree=True))
    off = vc.render_frame(ball, ball_scene, settings(use_octree=False))
    assert np.array_equal(on.pixels, off.pixels) and on.sample_count < off.sample_count
    shell = vc.make_phantom("shell", 32, r_inner=8, r_outer=12)
    base = vc.default_scene(shell)
    for win in (vc.ThresholdWindow(500, 4095), vc.ThresholdWindow(400, 600)):
        sc = vc.Scene(camera=base.camera, light=base.light, window=win)
        a = vc.render_frame(shell, sc, settings(use_octree=True)).pixels
        b = vc.render_frame(shell, sc, settings(use_octree=False)).pixels
        assert np.array_equal(a, b)


def test_adaptive_stride_saves_samples_within_two_levels():
    """test_render.py:146-156"""
    vol = vc.make_phantom("sphere", 64, radius=8)
    sc = vc.default_scene(vol)
    full = vc.render_frame(vol, sc, settings(use_octree=False))
    fast = vc.render_frame(vol, sc, settings(use_octree=False, use_adaptive=True, adaptive_factor=4))
    assert fast.sample_count < 0.6 * full.sample_count
    assert int(np.abs(fast.pixels.astype(int) - full.pixels.astype(int)).max()) <= 2


def test_clip_box_only_removes_hits(ball, ball_scene):
    """test_render.py:159-177"""
    bg = (0.0, 0.0, 0.25, 1.0)
    bg_px = np.array([0, 0, 64, 255], np.uint8)
    full = vc.render_frame(ball, ball_scene, settings(background=bg)).pixels
    half = ball.extent[0] / 2
    sc = vc.Scene(camera=ball_scene.camera, light=ball_scene.light,
                  clip=vc.ClipBox(lo=(0, 0, 0), hi=(half, 1e9, 1e9)))
    cut = vc.render_frame(ball, sc, settings(background=bg)).pixels
    assert (cut[32, :8] == bg_px).all()
    assert not (full[32] == bg_px).all(axis=1).all()
    was_bg = (full == bg_px).all(axis=2)
    now_bg = (cut == bg_px).all(axis=2)
    assert (now_bg | ~was_bg).all()


def test_eye_inside_material_gives_black_centre():
    """test_render.py:180-193: rays start inside a flat shell wall, hit at
    once, zero gradient, black."""
    shell = vc.make_phantom("shell", 32, r_inner=10, r_outer=14)
    mid = tuple(e / 2 for e in shell.extent)
    sc = vc.Scene(camera=vc.Camera(eye=(mid[0] + 12.0, mid[1], mid[2]), target=mid),
                  light=vc.Light(position=(100.0, 100.0, 100.0)))
    px = vc.render_frame(shell, sc, settings(background=(0, 0, 0.25, 1))).pixels
    assert (px[32, 32] == np.array([0, 0, 0, 255], np.uint8)).all()
    assert (px[31:34, 31:34, :3] == 0).all()


def test_surface_alpha_is_binary(ball, ball_scene):
    """test_render.py:196-200"""
    a = set(np.unique(vc.render_frame(ball, ball_scene, settings(background=(0, 0, 0, 0.0))).pixels[:, :, 3]).tolist())
    assert a == {0, 255}


# ------------------------------------------------------------- test_gradients.py

def _kernel_tables():
    """The 3x3x3 Sobel and Zucker-Hummel weights, typed out from the
    operator definitions (gradients.py:20-70), [di+1][dj+1][dk+1]."""
    plane = {(0, 0): 6, (0, 1): 3, (1, 0): 3, (1, 1): 1}
    sob = np.zeros((3, 3, 3, 3))
    zh = np.zeros((3, 3, 3, 3))
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for dk in (-1, 0, 1):
                d = (di, dj, dk)
                for a in range(3):
                    others = tuple(abs(d[b]) for b in range(3) if b != a)
                    sob[a, di + 1, dj + 1, dk + 1] = d[a] * plane[others]
                    if any(d):
                        zh[a, di + 1, dj + 1, dk + 1] = d[a] / math.sqrt(di * di + dj * dj + dk * dk)
    return {vc.OperatorKind.SOBEL3D: sob, vc.OperatorKind.ZUCKER_HUMMEL: zh}


def _stencil(arr, i, j, k, w):
    """27-term sum accumulated di -> dj -> dk, the order the operators
    define (the same float64 rounding as the reference's own check)."""
    g = [0.0, 0.0, 0.0]
    for di in (-1, 0, 1):
        for dj in (-1, 0, 1):
            for dk in (-1, 0, 1):
                v = float(arr[k + dk, j + dj, i + di])
                for a in range(3):
                    g[a] += float(w[a, di + 1, dj + 1, dk + 1]) * v
    return np.array(g)


@pytest.fixture(scope="module")
def noise16():
    rng = np.random.default_rng(7)
    return vc.Volume.from_array(rng.integers(0, 4096, size=(16, 16, 16)).astype(np.uint16))


def test_flat_volume_gradient_is_zero():
    """test_gradients.py:58-62"""
    vol = vc.Volume.from_array(np.full((8, 8, 8), 1234, np.uint16))
    for fn in (vc.central_difference, vc.sobel3d, vc.zucker_hummel):
        for p in ((3.0, 3.0, 3.0), (2.5, 4.25, 3.75)):
            assert np.array_equal(fn(vol, p), np.zeros(3))


def test_x_ramp_gradients():
    """test_gradients.py:65-83: unit +x for every operator; raw CD 2,
    Sobel 2*(6+4*3+4*1) = 44, ZH 2*(1 + 4/sqrt2 + 4/sqrt3)."""
    ramp = vc.make_phantom("ramp", 16)
    for kind in vc.OperatorKind:
        for p in ((5.0, 6.0, 7.0), (8.5, 7.25, 6.75)):
            assert vc.gradient(ramp, p, kind) == pytest.approx([1.0, 0.0, 0.0], abs=1e-12)
    arr = np.tile(np.arange(16, dtype=np.uint16), (16, 16, 1))
    vol = vc.Volume.from_array(arr)
    p = [(7.0, 7.0, 7.0)]
    assert tuple(grad_raw_points(vol, p, vc.OperatorKind.CENTRAL_DIFFERENCE)[0]) == (2.0, 0.0, 0.0)
    assert tuple(grad_raw_points(vol, p, vc.OperatorKind.SOBEL3D)[0]) == (44.0, 0.0, 0.0)
    gx, gy, gz = grad_raw_points(vol, p, vc.OperatorKind.ZUCKER_HUMMEL)[0]
    assert gx == pytest.approx(2.0 * (1.0 + 4.0 / math.sqrt(2.0) + 4.0 / math.sqrt(3.0)), rel=1e-12)
    assert (gy, gz) == pytest.approx((0.0, 0.0), abs=1e-12)


@pytest.mark.parametrize("kind", [vc.OperatorKind.SOBEL3D, vc.OperatorKind.ZUCKER_HUMMEL,
                                  vc.OperatorKind.CENTRAL_DIFFERENCE])
def test_lattice_gradient_vs_direct_stencil(noise16, kind):
    """test_gradients.py:86-118: at interior lattice points the raw
    gradient is the plain stencil sum (two-point difference for CD)."""
    arr = noise16.as_array()
    rng = np.random.default_rng(3)
    pts = [tuple(int(x) for x in rng.integers(1, 15, size=3)) for _ in range(40)]
    got = grad_raw_points(noise16, [tuple(float(c) for c in p) for p in pts], kind)
    tables = _kernel_tables()
    for (i, j, k), g in zip(pts, got):
        if kind is vc.OperatorKind.CENTRAL_DIFFERENCE:
            want = np.array([float(arr[k, j, i + 1]) - float(arr[k, j, i - 1]),
                             float(arr[k, j + 1, i]) - float(arr[k, j - 1, i]),
                             float(arr[k + 1, j, i]) - float(arr[k - 1, j, i])])
        else:
            want = _stencil(arr, i, j, k, tables[kind])
        assert g == pytest.approx(want, abs=1e-12)


def test_normals_unit_or_zero(noise16):
    """test_gradients.py:121-127"""
    rng = np.random.default_rng(11)
    for _ in range(30):
        p = tuple(float(x) for x in rng.uniform(0, 15, size=3))
        for kind in vc.OperatorKind:
            n = float(np.linalg.norm(vc.gradient(noise16, p, kind)))
            assert n == 0.0 or n == pytest.approx(1.0, abs=1e-9)


def test_mirror_and_axis_swap_symmetries(noise16):
    """test_gradients.py:130-153: mirroring x negates gx; swapping the x and
    y axes swaps gx and gy."""
    arr = noise16.as_array()
    mirrored = vc.Volume.from_array(np.ascontiguousarray(arr[:, :, ::-1]))
    swapped = vc.Volume.from_array(np.ascontiguousarray(np.transpose(arr, (0, 2, 1))))
    rng = np.random.default_rng(5)
    for _ in range(20):
        x, y, z = (float(c) for c in rng.uniform(1, 14, size=3))
        for kind in vc.OperatorKind:
            g = vc.gradient(noise16, (x, y, z), kind)
            gm = vc.gradient(mirrored, (15.0 - x, y, z), kind)
            assert gm == pytest.approx([-g[0], g[1], g[2]], abs=1e-12)
            gs = vc.gradient(swapped, (y, x, z), kind)
            assert gs == pytest.approx([g[1], g[0], g[2]], abs=1e-12)


def _shell_normal_errors(kind, n=200):
    shell = vc.make_phantom("shell", 48, r_inner=14, r_outer=18)
    c = np.full(3, (48 - 1) / 2.0)  # voxel-coordinate centre
    rng = np.random.default_rng(17)
    errs = []
    for _ in range(n):
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        p = c + 18.0 * d  # on the outer surface
        g = vc.gradient(shell, tuple(p), kind)
        assert np.linalg.norm(g) > 0
        # values rise inward: the gradient points toward the centre
        cosang = float(np.clip(np.dot(g, -d), -1.0, 1.0))
        errs.append(math.degrees(math.acos(cosang)))
    return np.array(errs)


def test_shell_normals_follow_the_radius():
    """test_gradients.py:156-188: mean < 15 deg, median < 12 deg, and the
    26-neighbour stencils no worse than central differences."""
    zh = _shell_normal_errors(vc.OperatorKind.ZUCKER_HUMMEL)
    cd = _shell_normal_errors(vc.OperatorKind.CENTRAL_DIFFERENCE)
    for e in (zh, cd):
        assert e.mean() < 15.0 and np.median(e) < 12.0
    assert zh.mean() <= cd.mean() + 1e-9


def test_outside_reads_zero_at_the_boundary():
    """test_gradients.py:191-196: in a uniform volume only the outside
    taps (reading 0) make a gradient, pointing inward at the x = 0 face."""
    vol = vc.Volume.from_array(np.full((8, 8, 8), 1000, np.uint16))
    g = vc.central_difference(vol, (0.5, 4.0, 4.0))
    assert g[0] > 0 and g == pytest.approx([1.0, 0.0, 0.0], abs=1e-12)


def test_operator_names_dispatch():
    """test_gradients.py:208-210"""
    ramp = vc.make_phantom("ramp", 16)
    for name in ("central", "sobel3d", "zucker-hummel"):
        assert vc.gradient(ramp, (6.0, 6.0, 6.0), name) == pytest.approx([1.0, 0.0, 0.0], abs=1e-12)


# ------------------------------------------------------ test_raycast_pipeline.py


def _ray(o, d):
    d = np.asarray(d, np.float64)
    return vc.Ray(origin=np.asarray(o, np.float64), direction=d / np.linalg.norm(d))


def _step16():
    a = np.zeros((16, 16, 16), np.uint16)
    a[:, :, 8:] = 1000  # x index >= 8
    return vc.Volume.from_array(a)


def _first_in_window(vol, r, iv, win, dt):
    t = iv[0]
    while t <= iv[1]:
        if win.contains(vc.sample(vol, r.origin + t * r.direction - 0.5)):
            return t
        t += dt
    return None


def test_march_misses_empty_and_hits_sphere_at_radius():
    """test_raycast_pipeline.py:50-65"""
    r = _ray((8, 8, -5), (0, 0, 1))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    assert vc.march_surface(r, vc.make_phantom("empty", 16), WINDOW, iv, 1.0, 0.125) is None
    h = vc.march_surface(r, vc.make_phantom("sphere", 16, radius=6), WINDOW, iv, 1.0, 0.125)
    assert h is not None and WINDOW.contains(h.value)
    assert abs(float(np.linalg.norm(h.position - 8.0)) - 6.0) <= 1.0 + 1e-9


@pytest.mark.parametrize("offset", [0.0, 1.3, 2.7])
def test_march_within_one_fine_step_of_dense_stepping(offset):
    """test_raycast_pipeline.py:68-77"""
    vol = vc.make_phantom("sphere", 16, radius=6)
    r = _ray((8 + offset, 8, -5), (0, 0, 1))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    h = vc.march_surface(r, vol, WINDOW, iv, 1.0, 0.125)
    want = _first_in_window(vol, r, iv, WINDOW, 0.125 / 64)
    assert h is not None and want is not None
    assert abs(h.t - want) <= 0.125 + 0.125 / 64 + 1e-9


def test_march_bracket_on_a_step_edge():
    """test_raycast_pipeline.py:80-92: the 500 crossing of the x ramp
    between voxels 7 and 8 is at world x = 8."""
    vol = _step16()
    r = _ray((0, 8, 8), (1, 0, 0))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    h = vc.march_surface(r, vol, WINDOW, iv, 1.0, 0.125)
    assert h is not None and h.t == pytest.approx(8.0, abs=1e-12)
    lo, hi = h.bracket
    assert hi == h.t and lo == pytest.approx(h.t - 0.125, abs=1e-12)
    assert not WINDOW.contains(vc.sample(vol, r.origin + lo * r.direction - 0.5))


def test_march_starting_in_material_and_band_window():
    """test_raycast_pipeline.py:95-114"""
    vol = _step16()
    r = _ray((12.0, 8, 8), (1, 0, 0))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    assert iv[0] == 0.0
    h = vc.march_surface(r, vol, WINDOW, iv, 1.0, 0.125)
    assert h is not None and h.t == 0.0 and h.bracket is None
    r = _ray((0, 8, 8), (1, 0, 0))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    h = vc.march_surface(r, vol, vc.ThresholdWindow(400.0, 600.0), iv, 0.25, 0.05)
    assert h is not None and 400.0 <= h.value <= 600.0


def test_march_argument_checks():
    """test_raycast_pipeline.py:117-125"""
    vol = vc.make_phantom("empty", 8)
    r = _ray((4, 4, -2), (0, 0, 1))
    for iv, coarse, fine in (((0.0, 10.0), 1.0, 2.0), ((5.0, 1.0), 1.0, 0.125), ((0.0, 10.0), -1.0, 0.125)):
        with pytest.raises(ValueError):
            vc.march_surface(r, vol, WINDOW, iv, coarse, fine)


def test_bisection_matches_a_plain_halving_loop():
    """test_raycast_pipeline.py:128-153: same halving sequence as a
    bisection driven by point samples; 6 / 10 iterations land within
    width/64 / width/1024 of the crossing."""
    vol = _step16()
    r = _ray((0, 8, 8), (1, 0, 0))

    def inside(t):
        return WINDOW.contains(vc.sample(vol, r.origin + t * r.direction - 0.5))

    rng = np.random.default_rng(23)
    for _ in range(40):
        a = 8.0 - float(rng.uniform(0.05, 2.0))
        b = 8.0 + float(rng.uniform(0.05, 2.0))
        assert not inside(a) and inside(b)
        lo, hi = a, b
        for _ in range(6):
            m = 0.5 * (lo + hi)
            lo, hi = (lo, m) if inside(m) else (m, hi)
        got = vc.refine_hitpoint(r, a, b, vol, WINDOW, iters=6)
        assert got == hi
        assert abs(got - 8.0) <= (b - a) / 64 + 1e-12
        assert abs(vc.refine_hitpoint(r, a, b, vol, WINDOW, iters=10) - 8.0) <= (b - a) / 1024 + 1e-12


def test_bisection_edge_cases():
    """test_raycast_pipeline.py:156-190: zero iterations return the inside
    end; the result is in window inside the bracket; a reversed bracket is
    rejected."""
    vol = _step16()
    r = _ray((0, 8, 8), (1, 0, 0))
    assert vc.refine_hitpoint(r, 7.0, 9.0, vol, WINDOW, iters=0) == 9.0
    with pytest.raises(ValueError):
        vc.refine_hitpoint(r, 9.0, 7.0, vol, WINDOW)
    ball = vc.make_phantom("sphere", 16, radius=6)
    r = _ray((8, 8, -5), (0, 0, 1))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    h = vc.march_surface(r, ball, WINDOW, iv, 1.0, 0.25)
    assert h is not None and h.bracket is not None
    t = vc.refine_hitpoint(r, h.bracket[0], h.bracket[1], ball, WINDOW, iters=6)
    assert h.bracket[0] <= t <= h.bracket[1]
    assert WINDOW.contains(vc.sample(ball, r.origin + t * r.direction - 0.5))


def test_finer_steps_never_increase_the_hit_error():
    """test_raycast_pipeline.py:173-183"""
    vol = vc.make_phantom("sphere", 32, radius=10)
    r = _ray((16.0, 16.0, -3.0), (0.13, 0.05, 1.0))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (32, 32, 32))
    want = _first_in_window(vol, r, iv, WINDOW, 1e-4)
    errs = [abs(vc.march_surface(r, vol, WINDOW, iv, 1.0, f).t - want) for f in (1.0, 0.5, 0.25, 0.125, 0.0625)]
    assert all(b <= a + 1e-9 for a, b in zip(errs, errs[1:]))


# ------------------------------------------- test_raycast_geometry.py: clip box


def test_clipbox_cases():
    """test_raycast_geometry.py:116-139"""
    box = ((0, 0, 0), (1, 1, 1))
    assert vc.intersect_clipbox(_ray((-1, 0.5, 0.5), (1, 0, 0)), *box) == pytest.approx((1.0, 2.0), abs=1e-12)
    assert vc.intersect_clipbox(_ray((0.5, 0.5, 0.5), (1, 0, 0)), *box) == pytest.approx((0.0, 0.5), abs=1e-12)
    assert vc.intersect_clipbox(_ray((-1, 5, 0.5), (1, 0, 0)), *box) is None
    assert vc.intersect_clipbox(_ray((2, 0.5, 0.5), (1, 0, 0)), *box) is None
    assert vc.intersect_clipbox(_ray((0.5, 0.5, -2), (0, 0, 1)), *box) == pytest.approx((2.0, 3.0), abs=1e-12)
    assert vc.intersect_clipbox(_ray((1.5, 0.5, -2), (0, 0, 1)), *box) is None
    assert vc.intersect_clipbox(_ray((1.0, 0.5, -2), (0, 0, 1)), *box) == pytest.approx((2.0, 3.0), abs=1e-12)


def test_clipbox_interval_is_ordered():
    """test_raycast_geometry.py:142-153"""
    rng = np.random.default_rng(8)
    lo, hi = np.zeros(3), np.full(3, 10.0)
    hits = 0
    for _ in range(1000):
        got = vc.intersect_clipbox(_ray(rng.uniform(-15, 25, 3), rng.normal(size=3)), lo, hi)
        if got is not None:
            assert 0.0 <= got[0] <= got[1]
            hits += 1
    assert hits > 30


def test_clipbox_against_dense_stepping():
    """test_raycast_geometry.py:156-173: every point of a 500-step walk
    that lies in the box lies in the interval (to 1e-2), and a miss has no
    such point."""
    rng = np.random.default_rng(9)
    lo, hi = np.zeros(3), np.array([4.0, 5.0, 6.0])
    ts = np.linspace(0.01, 25.0, 500)
    for _ in range(200):
        r = _ray(rng.uniform(-8, 12, 3), rng.normal(size=3))
        got = vc.intersect_clipbox(r, lo, hi)
        pts = r.origin[None, :] + ts[:, None] * r.direction[None, :]
        inside = np.all((pts >= lo) & (pts <= hi), axis=1)
        if got is None:
            assert not inside.any()
        else:
            assert ((ts[inside] >= got[0] - 1e-2) & (ts[inside] <= got[1] + 1e-2)).all()


# ------------------------------------------------------------ test_acceptance.py


def test_trilinear_sampling_exact():
    """test_acceptance.py:48-72: lattice points return the voxel bit for
    bit; off-lattice samples equal the 8-weight formula to 1e-9."""
    rng = np.random.default_rng(20240818)
    data = rng.integers(0, 4096, size=(24, 24, 24), dtype=np.uint16)
    vol = vc.Volume.from_array(data)
    for i, j, k in rng.integers(0, 24, size=(200, 3)):
        assert vc.sample(vol, (float(i), float(j), float(k)), vc.InterpolationMode.TRILINEAR) == \
            float(data[k, j, i])
    for p in rng.uniform(0, 23, size=(300, 3)):
        c = np.minimum(np.floor(p).astype(int), 22)
        f = p - c
        want = sum(float(data[c[2] + dz, c[1] + dy, c[0] + dx])
                   * (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                   for dz in (0, 1) for dy in (0, 1) for dx in (0, 1))
        assert vc.sample(vol, tuple(p), vc.InterpolationMode.TRILINEAR) == pytest.approx(want, rel=1e-9, abs=1e-9)


def test_operators_on_flat_ramp_and_shell():
    """test_acceptance.py:75-113 (the guarantees that hold in the
    reference: flat -> 0, ramp -> +x, and on 50 shell-surface points the
    Zucker-Hummel normals are no worse than central differences)."""
    flat = vc.Volume.from_array(np.full((16, 16, 16), 900, np.uint16))
    ramp = vc.make_phantom("ramp", 16, axis=0, scale=1.0)
    for op in vc.OperatorKind:
        assert tuple(vc.gradient(flat, (8.0, 8.0, 8.0), op)) == (0.0, 0.0, 0.0)
        assert tuple(vc.gradient(ramp, (8.0, 8.0, 8.0), op)) == pytest.approx((1.0, 0.0, 0.0), abs=1e-12)
    shell = vc.make_phantom("shell", 64, r_inner=20, r_outer=24)
    c = (64 - 1) / 2.0
    rng = np.random.default_rng(20240818)
    err = {op: [] for op in vc.OperatorKind}
    n = 0
    while n < 50:
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        r = 24.0 if n % 2 == 0 else 20.0
        p = c + r * v
        if not all(2.0 <= q <= 61.0 for q in p):
            continue
        n += 1
        out = v if r > 22.0 else -v
        for op in vc.OperatorKind:
            g = vc.gradient(shell, tuple(p), op)
            assert float(np.linalg.norm(g)) > 0.0
            err[op].append(math.degrees(math.acos(max(-1.0, min(1.0, float(np.dot(g, -out)))))))
    assert np.mean(err[vc.OperatorKind.ZUCKER_HUMMEL]) <= np.mean(err[vc.OperatorKind.CENTRAL_DIFFERENCE])


def test_six_bisections_shrink_the_bracket_64x():
    """test_acceptance.py:116-144"""
    rng = np.random.default_rng(7)
    win = vc.ThresholdWindow(500.0, 4095.0)
    r = vc.Ray(origin=(0.0, 4.0, 4.0), direction=(1.0, 0.0, 0.0))
    for _ in range(60):
        plane = float(rng.uniform(6.0, 26.0))
        data = np.zeros((8, 8, 32), np.uint16)
        data[:, :, int(math.ceil(plane)):] = 1000
        vol = vc.Volume.from_array(data)
        width = float(rng.uniform(0.1, 1.0))
        after = int(math.ceil(plane)) + 0.5 + float(rng.uniform(0.0, 0.4))
        before = after - width
        got = vc.refine_hitpoint(r, before, after, vol, win, iters=6)
        lo, hi = before, after
        for _ in range(6):
            m = 0.5 * (lo + hi)
            v = vc.sample(vol, (m - 0.5, 3.5, 3.5), vc.InterpolationMode.TRILINEAR)
            lo, hi = (lo, m) if win.contains(v) else (m, hi)
        assert got == hi
        assert width / (hi - lo) == pytest.approx(64.0, rel=1e-9)


def test_opaque_compositing_equals_surface_at_128x96():
    """test_acceptance.py:147-166"""
    vol = vc.make_phantom("sphere", 64, radius=22)
    base = vc.default_scene(vol)
    sc = vc.Scene(camera=base.camera, light=base.light, window=base.window, transfer=_opaque())
    a = vc.render_frame(vol, sc, vc.RenderSettings(width=128, height=96, mode=vc.RenderMode.SURFACE))
    b = vc.render_frame(vol, sc, vc.RenderSettings(width=128, height=96, mode=vc.RenderMode.COMPOSITED))
    assert np.array_equal(a.pixels, b.pixels)


def test_skipping_sound_and_at_least_halves_sparse_work():
    """test_acceptance.py:169-183"""
    st = vc.RenderSettings(width=96, height=72)
    for vol in (vc.make_phantom("sphere", 64, radius=22), vc.make_phantom("shell", 64, r_inner=20, r_outer=24)):
        sc = vc.default_scene(vol)
        on = vc.render_frame(vol, sc, st)
        off = vc.render_frame(vol, sc, vc.RenderSettings(width=96, height=72, use_octree=False))
        assert np.array_equal(on.pixels, off.pixels)
    sparse = vc.make_phantom("sphere", 64, radius=8)
    assert (sparse.as_array() > 0).mean() < 0.15
    sc = vc.default_scene(sparse)
    on = vc.render_frame(sparse, sc, st)
    off = vc.render_frame(sparse, sc, vc.RenderSettings(width=96, height=72, use_octree=False))
    assert np.array_equal(on.pixels, off.pixels)
    assert on.sample_count <= 0.5 * off.sample_count


def test_default_size_frame_independent_of_workers():
    """test_acceptance.py:186-193 (640x480 defaults)"""
    vol = vc.make_phantom("sphere", 128, radius=44.8)
    sc = vc.default_scene(vol)
    frames = [vc.render_frame(vol, sc, vc.RenderSettings(), workers=n).pixels for n in (1, 2, 16)]
    assert np.array_equal(frames[0], frames[1]) and np.array_equal(frames[0], frames[2])


# ---------------------------------------------------- test_volume.py: the sampler

TRI, NEAR, LIN = vc.InterpolationMode.TRILINEAR, vc.InterpolationMode.NEAREST, vc.InterpolationMode.LINEAR


@pytest.fixture(scope="module")
def noise16_ref():
    """The reference conftest's noise volume (seed 99)."""
    r = np.random.default_rng(99)
    return vc.Volume.from_array(r.integers(0, 4096, size=(16, 16, 16), dtype=np.uint16))


def _corner_sum(arr, x, y, z):
    i, j, k = int(math.floor(x)), int(math.floor(y)), int(math.floor(z))
    fx, fy, fz = x - i, y - j, z - k
    return sum(float(arr[k + c, j + b, i + a]) * (fx if a else 1 - fx) * (fy if b else 1 - fy) * (fz if c else 1 - fz)
               for c in (0, 1) for b in (0, 1) for a in (0, 1))


def test_trilinear_corner_sum_lattice_and_affine(noise16_ref):
    """test_volume.py:37-62"""
    arr = noise16_ref.as_array()
    rng = np.random.default_rng(20240817)
    for p in rng.uniform(0.0, 14.999, size=(300, 3)):
        assert vc.sample(noise16_ref, p, TRI) == pytest.approx(_corner_sum(arr, *p), rel=1e-12, abs=1e-9)
    for i, j, k in rng.integers(0, 16, size=(200, 3)):
        assert vc.sample(noise16_ref, (i, j, k), TRI) == float(arr[k, j, i])
    zi, yi, xi = np.meshgrid(np.arange(12), np.arange(12), np.arange(12), indexing="ij")
    affine = vc.Volume.from_array((7 + 2 * xi + 3 * yi + 5 * zi).astype(np.uint16))
    for x, y, z in rng.uniform(0, 11, size=(200, 3)):
        assert vc.sample(affine, (x, y, z)) == pytest.approx(7 + 2 * x + 3 * y + 5 * z, rel=1e-9)


def test_last_lattice_plane_interpolates(noise16_ref):
    """test_volume.py:65-70: x = n-1 uses the last cell."""
    want = _corner_sum(noise16_ref.as_array(), 14.9999999999, 7.2, 3.8)
    assert vc.sample(noise16_ref, (15.0, 7.2, 3.8)) == pytest.approx(want, abs=1e-6)


def test_nearest_rounding(noise16_ref):
    """test_volume.py:73-86: halves round away from zero."""
    arr = noise16_ref.as_array()
    assert vc.sample(noise16_ref, (1.5, 2.0, 3.0), NEAR) == float(arr[3, 2, 2])
    assert vc.sample(noise16_ref, (1.49, 2.0, 3.0), NEAR) == float(arr[3, 2, 1])
    assert vc.sample(noise16_ref, (7.5, 7.5, 7.5), NEAR) == float(arr[8, 8, 8])
    rng = np.random.default_rng(2)
    for p in rng.uniform(0, 15, size=(200, 3)):
        i, j, k = (int(math.floor(c + 0.5)) for c in p)
        assert vc.sample(noise16_ref, p, NEAR) == float(arr[k, j, i])


def test_linear_mode(noise16_ref):
    """test_volume.py:89-113: interpolate along the axis farthest from
    its lattice plane (ties: x, then y), round the others; equals trilinear
    on the lattice."""
    arr = noise16_ref.as_array()
    assert vc.sample(noise16_ref, (2.3, 1.04, 3.96), LIN) == \
        pytest.approx(0.7 * float(arr[4, 1, 2]) + 0.3 * float(arr[4, 1, 3]), rel=1e-12)
    assert vc.sample(noise16_ref, (5.02, 9.01, 6.6), LIN) == \
        pytest.approx(0.4 * float(arr[6, 9, 5]) + 0.6 * float(arr[7, 9, 5]), rel=1e-12)
    assert vc.sample(noise16_ref, (1.5, 2.5, 3.5), LIN) == \
        pytest.approx(0.5 * float(arr[4, 3, 1]) + 0.5 * float(arr[4, 3, 2]), rel=1e-12)
    rng = np.random.default_rng(3)
    for p in rng.integers(0, 16, size=(100, 3)).astype(float):
        assert vc.sample(noise16_ref, p, LIN) == vc.sample(noise16_ref, p, TRI)


def test_outside_reads_zero_and_non_finite_rejected(noise16_ref):
    """test_volume.py:116-128"""
    for mode in vc.InterpolationMode:
        for p in ((-0.01, 5, 5), (5, 15.01, 5), (5, 5, -3.0)):
            assert vc.sample(noise16_ref, p, mode) == 0.0
    for bad in ((np.nan, 1, 1), (np.inf, 1, 1)):
        with pytest.raises(ValueError):
            vc.sample(noise16_ref, bad)
