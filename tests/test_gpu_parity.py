"""Parity of the sm_100a path against the reference goldens and the oracle.

Bars (BASELINE.json north_star): frames within max |d| <= 1/255 per RGBA
channel -- the float64 software-trilinear path with reference taps is held
to bit-exactness (and exact sample counts), the gradient-volume shading
path to <= 1 LSB; gradient volumes within 1e-5 relative
(max_a |g_gpu - g_ref| <= 1e-5 * max(|g_ref|_2, 1)).
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from oracle import oracle
from paper_1609_01317_b200 import phantoms
from tests.conftest import frame_names, zero_window_frames
from tests.specs import product_scene, product_settings, product_volume, spec_of

pytestmark = pytest.mark.gpu


def maxdiff(a, b) -> int:
    return int(np.abs(a.astype(np.int32) - b.astype(np.int32)).max()) if a.size else 0


# ---------------------------------------------------------------- frames vs reference goldens

@pytest.mark.parametrize("name", frame_names())
def test_frame_bit_exact_vs_reference_brute_force(golden, name):
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    vol = product_volume(arr, spacing)
    ref_octree = spec.get("settings", {}).get("use_octree", False)
    fb = vc.render_frame(vol, product_scene(spec), product_settings(spec, use_octree=False))
    assert np.array_equal(fb.pixels, want_px), f"max|d|={maxdiff(fb.pixels, want_px)}"
    if not ref_octree:  # the reference's octree segments change its count, not its pixels
        assert fb.sample_count == want_count


@pytest.mark.parametrize("name", frame_names())
def test_frame_bit_exact_with_empty_space_skipping(golden, name):
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    vol = product_volume(arr, spacing)
    fb = vc.render_frame(vol, product_scene(spec), product_settings(spec, use_octree=True))
    assert np.array_equal(fb.pixels, want_px), f"max|d|={maxdiff(fb.pixels, want_px)}"
    if not spec.get("settings", {}).get("use_adaptive"):  # adaptive mode never skips
        assert fb.sample_count <= want_count


def _reference_octree_frames():
    from tests.conftest import GOLDEN, Golden

    return [e["name"] for e in Golden(GOLDEN).frames() if e["spec"].get("settings", {}).get("use_octree")]


@pytest.mark.parametrize("name", _reference_octree_frames())
def test_frame_octree_segments_match_reference_count(golden, name):
    """Frames the reference rendered with use_octree=True (adaptive stride
    restarted at its octree segments): the device's segment walk gives the
    reference's pixels and the reference's own sample count."""
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    vol = product_volume(arr, spacing)
    fb = vc.render_frame(vol, product_scene(spec), product_settings(spec, use_octree=True))
    assert np.array_equal(fb.pixels, want_px), f"max|d|={maxdiff(fb.pixels, want_px)}"
    assert fb.sample_count == want_count


@pytest.mark.parametrize("name", zero_window_frames())
def test_zero_window_frames_match_reference(golden, name):
    """0 inside the threshold window: with use_octree the reference skips
    in-window border samples that brute force hits (its octree segments,
    _kernels.py:656-669), so the two reference images differ everywhere on
    these goldens.  The device follows the golden's own use_octree setting
    (the octree-segment walk when on): pixels and sample count."""
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    vol = product_volume(arr, spacing)
    fb = vc.render_frame(vol, product_scene(spec), product_settings(spec))
    assert np.array_equal(fb.pixels, want_px), f"max|d|={maxdiff(fb.pixels, want_px)}"
    assert fb.sample_count == want_count
    fb2 = vc.render_frame(vol, product_scene(spec), product_settings(spec, gradient_source="volume"))
    assert maxdiff(fb2.pixels, want_px) <= 1


@pytest.mark.parametrize("name", frame_names())
def test_frame_gradient_volume_within_one_lsb(golden, name):
    arr, spacing, spec, want_px, _ = golden.frame(name)
    vol = product_volume(arr, spacing)
    fb = vc.render_frame(vol, product_scene(spec),
                         product_settings(spec, use_octree=True, gradient_source="volume"))
    assert maxdiff(fb.pixels, want_px) <= 1


def test_empty_volume_skipping_fetches_nothing():
    """test_render.py:45-53: background only, and no fetch with skipping on."""
    vol = vc.make_phantom("empty", 16)
    bg = (0.25, 0.5, 0.75, 1.0)
    fb = vc.render_frame(vol, vc.default_scene(vol),
                         vc.RenderSettings(width=64, height=64, background=bg))
    assert (fb.pixels == np.array([64, 128, 191, 255], np.uint8)).all()
    assert fb.sample_count == 0
    fb2 = vc.render_frame(vol, vc.default_scene(vol),
                          vc.RenderSettings(width=64, height=64, background=bg, use_octree=False))
    assert np.array_equal(fb.pixels, fb2.pixels) and fb2.sample_count > 0


# ---------------------------------------------------------------- point queries

@pytest.mark.parametrize("interp", ["nearest", "linear", "trilinear"])
def test_sample_points_bit_exact(golden, interp):
    vol = vc.Volume.from_array(golden["points/noise16"])
    got = vc.sample_points(vol, golden["points/pts"], vc.InterpolationMode(interp))
    assert np.array_equal(got, golden[f"points/sample_{interp}"])


@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_grad_raw_points_bit_exact(golden, op):
    vol = vc.Volume.from_array(golden["points/noise16"])
    got = vc.grad_raw_points(vol, golden["points/gpts"], vc.OperatorKind(op))
    assert np.array_equal(got, golden[f"points/grad_{op}"])


def test_public_gradient_api_matches_reference_kats():
    """test_gradients.py:58-83 and :191-196 through the public API."""
    ramp = vc.make_phantom("ramp", 16)
    for kind in vc.OperatorKind:
        for p in [(7, 7, 7), (5.3, 8.6, 7.1), (2.5, 2.5, 2.5)]:
            assert vc.gradient(ramp, p, kind) == pytest.approx([1.0, 0.0, 0.0], abs=1e-12)
    flat = vc.Volume.from_array(np.full((8, 8, 8), 1000, np.uint16))
    g = vc.central_difference(flat, (0.5, 4.0, 4.0))
    assert g == pytest.approx([1.0, 0.0, 0.0], abs=1e-12)
    assert np.array_equal(vc.sobel3d(flat, (3.5, 4.0, 4.25)), np.zeros(3))
    with pytest.raises(ValueError):
        vc.gradient(ramp, (7, 7, 7), "laplace")


def test_single_ray_helpers_match_oracle():
    arr = np.zeros((16, 16, 16), np.uint16)
    arr[:, :, 8:] = 1000
    vol = vc.Volume.from_array(arr)
    r = vc.Ray(origin=np.array([0.0, 8.0, 8.0]), direction=np.array([1.0, 0.0, 0.0]))
    iv = vc.intersect_clipbox(r, (0, 0, 0), (16, 16, 16))
    assert iv == oracle.box_interval(r.origin, r.direction, (0, 0, 0), (16, 16, 16))
    win = vc.ThresholdWindow(500.0, 4095.0)
    hit = vc.march_surface(r, vol, win, iv, 1.0, 0.125)
    want = oracle.first_hit(arr, (1, 1, 1), r.origin, r.direction, iv, 1.0, 0.125, (500.0, 4095.0))
    assert hit.t == want[0] and hit.bracket == (want[1], want[0])
    assert hit.t == pytest.approx(8.0, abs=1e-12)
    rng = np.random.default_rng(5)
    for _ in range(20):
        before, after = 8.0 - rng.uniform(0.05, 2.0), 8.0 + rng.uniform(0.05, 2.0)
        got = vc.refine_hitpoint(r, before, after, vol, win, iters=6)
        assert got == oracle.bisect(arr, (1, 1, 1), r.origin, r.direction, before, after,
                                    (500.0, 4095.0), 6)
    assert vc.intersect_clipbox(vc.Ray(np.array([-1.0, 5, 0.5]), np.array([1.0, 0, 0])),
                                (0, 0, 0), (1, 1, 1)) is None


# ---------------------------------------------------------------- Kernel 1

def _grad_close(got, want):
    scale = np.maximum(np.linalg.norm(want, axis=-1), 1.0)
    return float((np.abs(got - want).max(axis=-1) / scale).max())


@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_gradient_volume_vs_reference_lattice(golden, op):
    noise = golden["points/noise16"]
    vol = vc.Volume.from_array(noise)
    g = vc.gradient_volume(vol, vc.OperatorKind(op)).cpu().numpy()
    want = golden[f"lattice/noise16_{op}"]
    assert np.array_equal(g[..., 3], noise.astype(np.float32))
    if op == "zucker-hummel":
        assert _grad_close(g[..., :3].astype(np.float64), want) <= 1e-5
    else:  # integer stencils are exact
        assert np.array_equal(g[..., :3], want.astype(np.float32))


@pytest.mark.parametrize("maker,n", [(phantoms.ct_phantom, 128), (phantoms.marschner_lobb, 96),
                                     (lambda n: phantoms.fbm_noise(n, octaves=3), 64)])
@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_gradient_volume_vs_numpy_stencil(maker, n, op):
    vol = maker(n)
    g = vc.gradient_volume(vol, vc.OperatorKind(op)).cpu().numpy()
    want = oracle.grad_volume_numpy(vol.as_array(), op)
    assert _grad_close(g[..., :3].astype(np.float64), want) <= 1e-5
    if op != "zucker-hummel" and vol.data.dtype != np.float32:
        assert np.array_equal(g[..., :3], want.astype(np.float32))


def test_gradient_volume_odd_dims_and_tiny():
    rng = np.random.default_rng(3)
    for shape in [(1, 1, 1), (2, 3, 5), (17, 9, 33), (40, 1, 7)]:
        arr = rng.integers(0, 4096, size=shape, dtype=np.uint16)
        vol = vc.Volume.from_array(arr)
        for op in ("central", "sobel3d", "zucker-hummel"):
            g = vc.gradient_volume(vol, vc.OperatorKind(op)).cpu().numpy()
            want = oracle.grad_volume_numpy(arr, op)
            assert _grad_close(g[..., :3].astype(np.float64), want) <= 1e-5, (shape, op)


# ---------------------------------------------------------------- larger scenes vs oracle

def _oracle_frame(vol, sc_st):
    return oracle.render(vol.as_array(), vol.spacing, spec_of(sc_st))


@pytest.mark.parametrize("op", list(vc.OperatorKind))
def test_ct128_composited_vs_oracle(op):
    vol = phantoms.ct_phantom(128)
    sc, st = phantoms.scene_c3(vol, op=op, width=192, height=108, azimuth=33.0)
    want_px, want_count = _oracle_frame(vol, (sc, st))
    for skip in (False, True):
        fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=skip))
        assert np.array_equal(fb.pixels, want_px), f"skip={skip} max|d|={maxdiff(fb.pixels, want_px)}"
        if not skip:
            assert fb.sample_count == want_count
    fb = vc.render_frame(vol, sc, product_settings_from(st, gradient_source="volume"))
    assert maxdiff(fb.pixels, want_px) <= 1


@pytest.mark.parametrize("spacing", [(0.7, 0.9, 1.3), (1.0 / 3.0, 0.6, 2.5)])
def test_anisotropic_spacing_vs_oracle(spacing):
    """Non power-of-two spacing takes the reciprocal division path
    (ddiv_rcp) for every ray position: still bit-exact, counts included."""
    base = phantoms.ct_phantom(80)
    vol = vc.Volume.from_array(base.as_array(), spacing=spacing)
    for mode in ("surface", "composited"):
        sc, st = phantoms.scene_c3(vol, width=160, height=90, azimuth=21.0, mode=mode)
        want_px, want_count = _oracle_frame(vol, (sc, st))
        fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=False))
        assert np.array_equal(fb.pixels, want_px), f"max|d|={maxdiff(fb.pixels, want_px)}"
        assert fb.sample_count == want_count
        fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=True))
        assert np.array_equal(fb.pixels, want_px)


def test_marschner_lobb_c2_orbit_vs_oracle():
    vol = phantoms.marschner_lobb(64)
    for az in (0.0, 45.0, 200.0):
        sc, st = phantoms.scene_c2(vol, width=128, height=128, azimuth=az)
        want_px, want_count = _oracle_frame(vol, (sc, st))
        fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=False))
        assert np.array_equal(fb.pixels, want_px) and fb.sample_count == want_count
        fb = vc.render_frame(vol, sc, product_settings_from(st, gradient_source="volume"))
        assert maxdiff(fb.pixels, want_px) <= 1


def test_fbm_float32_vs_oracle():
    vol = phantoms.fbm_noise(48, octaves=4)
    sc, st = phantoms.scene_c4(vol, width=96, height=64, azimuth=10.0)
    want_px, want_count = _oracle_frame(vol, (sc, st))
    fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=False))
    assert np.array_equal(fb.pixels, want_px) and fb.sample_count == want_count
    fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=True))
    assert np.array_equal(fb.pixels, want_px)


def product_settings_from(st: vc.RenderSettings, **over) -> vc.RenderSettings:
    from dataclasses import replace

    return replace(st, **over)


# ---------------------------------------------------------------- full size, size-independent properties

@pytest.fixture(scope="module")
def ct512():
    return phantoms.ct_phantom(512)


def test_c3_full_size_skip_and_gradient_volume_properties(ct512):
    """At BASELINE C3 size the oracle is too slow for a whole frame: check
    (a) skipping is pixel-identical to brute force, (b) the gradient-volume
    path is within 1 LSB of the bit-faithful taps path, (c) a band of rows
    is bit-identical to the oracle."""
    sc, st = phantoms.scene_c3(ct512, azimuth=17.0)
    brute = vc.render_frame(ct512, sc, product_settings_from(st, use_octree=False))
    skip = vc.render_frame(ct512, sc, product_settings_from(st, use_octree=True))
    assert np.array_equal(brute.pixels, skip.pixels)
    assert skip.sample_count < brute.sample_count
    fast = vc.render_frame(ct512, sc, product_settings_from(st, gradient_source="volume"))
    assert maxdiff(fast.pixels, brute.pixels) <= 1
    rows = (530, 538)
    want_px, _ = oracle.render(ct512.as_array(), ct512.spacing, spec_of((sc, st)), rows=rows)
    assert np.array_equal(brute.pixels[rows[0]:rows[1]], want_px[rows[0]:rows[1]])


def test_band_partition_reassembles_whole_frame(ct512):
    """Image-plane tiles (the multi-GPU partition) are bit-identical to the
    whole frame for any band height / owner count (test_render.py:111-122)."""
    import ctypes

    import torch

    from paper_1609_01317_b200 import _native
    from paper_1609_01317_b200.raycast import render_params

    sc, st = phantoms.scene_c3(ct512, width=640, height=360, azimuth=5.0)
    whole = vc.render_frame(ct512, sc, st).pixels
    dv = vc.device_volume(ct512)
    L = _native.load()
    for band_rows, owners in [(8, 3), (16, 8), (37, 2)]:
        img = np.zeros_like(whole)
        for r in range(owners):
            P = render_params(ct512, sc, st, band_rows=band_rows, band_first=r, band_step=owners)
            nb = -(-st.height // band_rows)
            bands = list(range(r, nb, owners))
            rows = [y for b in bands for y in range(b * band_rows, min((b + 1) * band_rows, st.height))]
            out = torch.empty((len(rows), st.width, 4), dtype=torch.uint8, device="cuda")
            _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()),
                                      None, None))
            torch.cuda.synchronize()
            img[rows] = out.cpu().numpy()
        assert np.array_equal(img, whole), (band_rows, owners)


def test_render_sequence_matches_render_frame():
    vol = phantoms.ct_phantom(96)
    frames = [phantoms.scene_c3(vol, width=160, height=90, azimuth=float(a)) for a in (0, 33, 71, 150, 299)]
    want = [vc.render_frame(vol, sc, st).pixels.copy() for sc, st in frames]
    got = [(fb.pixels.copy(), fb.sample_count) for fb in vc.render_sequence(vol, frames, depth=2)]
    assert len(got) == len(want)
    for (g, cnt), w in zip(got, want):
        assert np.array_equal(g, w) and cnt > 0


def test_window_changes_between_frames_use_their_own_distance_fields():
    """Several threshold windows in flight on one volume (the distance-field
    cache is keyed by window): every frame stays bit-exact vs the oracle."""
    vol = phantoms.ct_phantom(64)
    base_sc, st = phantoms.scene_c3(vol, width=64, height=48, azimuth=20.0, mode="surface")
    for lo in (500.0, 950.0, 1200.0, 500.0, 1290.0, 960.0, 400.0, 600.0, 700.0, 800.0, 500.0):
        sc = vc.Scene(camera=base_sc.camera, light=base_sc.light, window=vc.ThresholdWindow(lo, 4095.0))
        want, _ = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)))
        fb = vc.render_frame(vol, sc, st)
        assert np.array_equal(fb.pixels, want), lo


@pytest.mark.parametrize("mode", ["surface", "composited"])
def test_adaptive_stride_vs_oracle(mode):
    """use_adaptive (_kernels.py:437-463) over the device octree: bit-exact
    against the oracle's restatement over the reference-format octree."""
    from dataclasses import replace

    vol = phantoms.ct_phantom(96)
    sc, st = phantoms.scene_c3(vol, width=128, height=72, azimuth=40.0, mode=mode)
    for factor, eps in ((4, None), (3, 400.0)):
        st2 = replace(st, use_adaptive=True, adaptive_factor=factor, detail_epsilon=eps,
                      use_octree=False)
        want, want_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st2)))
        fb = vc.render_frame(vol, sc, st2)
        assert np.array_equal(fb.pixels, want), (factor, eps, maxdiff(fb.pixels, want))
        assert fb.sample_count == want_count
        fb2 = vc.render_frame(vol, sc, replace(st2, gradient_source="volume"))
        assert maxdiff(fb2.pixels, want) <= 1
        # use_octree=True as the reference runs it (segment restarts,
        # restated in the oracle and pinned to the reference's counts): the
        # device replays the same walk -- same pixels, same count
        st3 = replace(st2, use_octree=True)
        want3, want3_count = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st3)), octree=True)
        fb3 = vc.render_frame(vol, sc, st3)
        assert np.array_equal(fb3.pixels, want3)
        assert fb3.sample_count == want3_count
        fb4 = vc.render_frame(vol, sc, replace(st3, gradient_source="volume"))
        assert maxdiff(fb4.pixels, want3) <= 1


@pytest.mark.parametrize("shape", [(1, 8, 8), (8, 1, 8), (2, 2, 2), (3, 17, 5), (1, 1, 1)])
@pytest.mark.parametrize("mode", ["surface", "composited"])
def test_degenerate_grids_vs_oracle(shape, mode):
    """Cell clamping for n = 1 / 2 (_kernels.py:52-64) and thin slabs."""
    rng = np.random.default_rng(sum(shape))
    arr = rng.integers(0, 4096, size=shape, dtype=np.uint16)
    vol = vc.Volume.from_array(arr)
    for op in vc.OperatorKind:
        sc = vc.default_scene(vol)
        sc = vc.Scene(camera=vc.Camera(eye=sc.camera.eye, target=sc.camera.target, azimuth=23.0,
                                       elevation=11.0), light=sc.light,
                      window=vc.ThresholdWindow(1200.0, 4095.0))
        st = vc.RenderSettings(width=24, height=20, operator=op, mode=mode, use_octree=False)
        want, cnt = oracle.render(arr, vol.spacing, spec_of((sc, st)))
        fb = vc.render_frame(vol, sc, st)
        assert np.array_equal(fb.pixels, want) and fb.sample_count == cnt, (shape, op)
        fb = vc.render_frame(vol, sc, product_settings_from(st, use_octree=True, gradient_source="volume"))
        assert maxdiff(fb.pixels, want) <= 1


@pytest.mark.parametrize("gather", ["nccl", "peer"])
def test_distributed_render_single_rank(gather):
    """render_frame_distributed on a 1-rank NCCL group: the band plan, the
    fused peer-store path (vc_render_to_peers) and the NCCL path reproduce
    render_frame bit-exactly."""
    import socket

    import torch.distributed as dist

    from paper_1609_01317_b200.dispatch import render_frame_distributed

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        vol = phantoms.ct_phantom(96)
        sc, st = phantoms.scene_c3(vol, width=200, height=117, azimuth=12.0)
        want = vc.render_frame(vol, sc, st)
        got = render_frame_distributed(vol, sc, st, band_rows=8, gather=gather)
        assert np.array_equal(got.pixels, want.pixels)
        assert got.sample_count == want.sample_count
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("wh", [(1920, 1080), (257, 3), (1, 1), (640, 480)])
def test_device_png_round_trip(wh):
    """Frame egress: the device PNG decodes (zlib, CRC and Adler-32 checked
    by the decoders) to exactly the frame's RGB (image_io.png_bytes drops
    alpha the same way)."""
    import io
    import zlib

    from PIL import Image

    from paper_1609_01317_b200 import egress

    W, H = wh
    rng = np.random.default_rng(W * 7 + H)
    img = np.zeros((H, W, 4), np.uint8)
    img[..., 3] = 255
    img[H // 3:, : max(W // 2, 1), :3] = rng.integers(0, 256, (H - H // 3, max(W // 2, 1), 3))
    img[: H // 4, :, 0] = 200  # long runs
    png = egress.png_bytes(img)
    assert png[:8] == b"\x89PNG\r\n\x1a\n"
    dec = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
    assert np.array_equal(dec, img[..., :3])
    # the IDAT payload is a valid zlib stream
    pos = 8
    while pos < len(png):
        n = int.from_bytes(png[pos:pos + 4], "big")
        typ = png[pos + 4:pos + 8]
        # every chunk's CRC-32 (the IDAT one is combined from per-row CRCs
        # computed on the device)
        assert int.from_bytes(png[pos + 8 + n:pos + 12 + n], "big") == zlib.crc32(png[pos + 4:pos + 8 + n])
        if typ == b"IDAT":
            raw = zlib.decompress(png[pos + 8:pos + 8 + n])
            assert len(raw) == H * (1 + 3 * W)
        pos += 12 + n
    assert pos == len(png)


@pytest.mark.parametrize("kind", ["skewed", "ramp", "noise", "flat"])
def test_device_png_code_construction(kind):
    """Symbol statistics that drive the shared dynamic Huffman code to its
    corners: nearly all one symbol with rare outliers (length limiting at
    15 bits), smooth ramps, uniform noise, a single colour (one literal)."""
    import io

    from PIL import Image

    from paper_1609_01317_b200 import egress

    H, W = 97, 211
    rng = np.random.default_rng({"skewed": 1, "ramp": 2, "noise": 3, "flat": 4}[kind])
    img = np.zeros((H, W, 4), np.uint8)
    img[..., 3] = 255
    if kind == "skewed":
        m = rng.random((H, W)) < 0.002
        img[m, :3] = rng.integers(0, 256, (int(m.sum()), 3))
    elif kind == "ramp":
        img[..., 0] = (np.arange(W)[None, :] * 255 // W).astype(np.uint8)
        img[..., 1] = (np.arange(H)[:, None] * 255 // H).astype(np.uint8)
    elif kind == "noise":
        img[..., :3] = rng.integers(0, 256, (H, W, 3))
    else:
        img[..., :3] = 77
    png = egress.png_bytes(img)
    dec = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
    assert np.array_equal(dec, img[..., :3])


def test_render_frame_png_matches_render_frame():
    import io

    from PIL import Image

    from paper_1609_01317_b200 import egress

    vol = phantoms.ct_phantom(128)
    sc, st = phantoms.scene_c3(vol, width=480, height=270, azimuth=21.0)
    fb = vc.render_frame(vol, sc, st)
    png, meta = egress.render_frame_png(vol, sc, st)
    dec = np.asarray(Image.open(io.BytesIO(png)).convert("RGB"))
    assert np.array_equal(dec, fb.pixels[..., :3])
    assert meta.sample_count == fb.sample_count and meta.pixels is None
    assert len(png) < 0.6 * fb.pixels[..., :3].nbytes  # it compresses
    pkt = egress.frame_packet(7, png)
    assert int.from_bytes(pkt[:8], "big") == 7 and int.from_bytes(pkt[8:12], "big") == len(png)


def test_many_streams_share_bounded_scratch():
    """Renders on more streams than the library keeps scratch for (LRU of 8)
    all produce the same frame."""
    import ctypes

    import torch

    from paper_1609_01317_b200 import _native
    from paper_1609_01317_b200.raycast import render_params

    vol = phantoms.ct_phantom(64)
    sc, st = phantoms.scene_c3(vol, width=96, height=64, azimuth=10.0)
    want = vc.render_frame(vol, sc, st).pixels
    dv = vc.device_volume(vol)
    P = render_params(vol, sc, st)
    L = _native.load()
    outs = []
    for _ in range(12):
        s = torch.cuda.Stream()
        out = torch.empty((64, 96, 4), dtype=torch.uint8, device="cuda")
        _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), None,
                                  ctypes.c_void_p(s.cuda_stream)))
        outs.append((s, out))
    for s, out in outs:
        s.synchronize()
        assert np.array_equal(out.cpu().numpy(), want)


def test_render_sequence_reuses_resources():
    vol = phantoms.ct_phantom(64)
    frames = [phantoms.scene_c3(vol, width=96, height=64, azimuth=float(a)) for a in range(5)]
    want = [vc.render_frame(vol, sc, st).pixels for sc, st in frames]
    for _ in range(3):  # pooled streams / buffers across calls
        got = [fb.pixels.copy() for fb in vc.render_sequence(vol, iter(frames))]
        assert all(np.array_equal(a, b) for a, b in zip(got, want))
