"""Pin the C oracle to the reference: bit-exact against golden fixtures
that tests/golden/make_golden.py produced by running the reference
(voxelcast numba kernels) itself.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import oracle
from tests.conftest import frame_names, zero_window_frames


@pytest.mark.parametrize("name", frame_names())
def test_oracle_frame_matches_reference(golden, name):
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    got_px, got_count = oracle.render(arr, spacing, spec, threads=4)
    if not spec.get("settings", {}).get("use_octree"):  # octree segments change the count only
        assert got_count == want_count
    assert np.array_equal(got_px, want_px), (
        f"{int((got_px != want_px).any(axis=2).sum())} pixels differ, "
        f"max |d| = {int(np.abs(got_px.astype(int) - want_px.astype(int)).max())}")


def _octree_frames():
    from tests.conftest import GOLDEN, Golden

    return [e["name"] for e in Golden(GOLDEN).frames() if e["spec"].get("settings", {}).get("use_octree")]


@pytest.mark.parametrize("name", _octree_frames())
def test_oracle_octree_segments_match_reference_counts(golden, name):
    """use_octree=True as the reference runs it (collect_segments,
    _kernels.py:267-342, and the segment loop of first_hit): pixels AND
    sample counts equal the reference's."""
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    got_px, got_count = oracle.render(arr, spacing, spec, threads=4, octree=True)
    assert np.array_equal(got_px, want_px)
    assert got_count == want_count


@pytest.mark.parametrize("name", zero_window_frames())
def test_oracle_zero_window_frames_match_reference(golden, name):
    """0 inside the window: the reference's image depends on use_octree
    (its segments skip in-window border samples); the oracle follows the
    setting each golden was rendered with -- pixels and counts."""
    arr, spacing, spec, want_px, want_count = golden.frame(name)
    got_px, got_count = oracle.render(arr, spacing, spec, threads=4, octree=True)
    assert np.array_equal(got_px, want_px)
    assert got_count == want_count


@pytest.mark.parametrize("interp", ["nearest", "linear", "trilinear"])
def test_oracle_sample_matches_reference(golden, interp):
    got = oracle.sample(golden["points/noise16"], golden["points/pts"], interp)
    assert np.array_equal(got, golden[f"points/sample_{interp}"])


@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_oracle_grad_raw_matches_reference(golden, op):
    got = oracle.grad_raw(golden["points/noise16"], golden["points/gpts"], op)
    assert np.array_equal(got, golden[f"points/grad_{op}"])


@pytest.mark.parametrize("op", ["central", "sobel3d", "zucker-hummel"])
def test_lattice_stencil_restatement_is_bit_exact(golden, op):
    """The numpy zero-padded stencil (used at sizes where looping grad_raw
    is too slow) equals grad_raw at every lattice point."""
    want = golden[f"lattice/noise16_{op}"]
    got = oracle.grad_volume_numpy(golden["points/noise16"], op)
    assert np.array_equal(got, want)
    got4 = oracle.grad_volume(golden["points/noise16"], op, threads=2)
    assert np.array_equal(got4[..., :3], want.astype(np.float32))
    assert np.array_equal(got4[..., 3], golden["points/noise16"].astype(np.float32))


def test_oracle_ramp_known_answers():
    """Raw KATs of pkg/tests/test_gradients.py:72-83 on ramp16 at (7,7,7)."""
    zi, yi, xi = np.meshgrid(np.arange(16), np.arange(16), np.arange(16), indexing="ij")
    ramp = np.floor(1.0 * xi).astype(np.uint16)
    g = oracle.grad_raw(ramp, [(7.0, 7.0, 7.0)], "central")[0]
    assert tuple(g) == (2.0, 0.0, 0.0)
    g = oracle.grad_raw(ramp, [(7.0, 7.0, 7.0)], "sobel3d")[0]
    assert tuple(g) == (44.0, 0.0, 0.0)
    g = oracle.grad_raw(ramp, [(7.0, 7.0, 7.0)], "zucker-hummel")[0]
    want = 2.0 + 4.0 * 2.0 / np.sqrt(2.0) + 8.0 / np.sqrt(3.0)
    assert g[0] == pytest.approx(want, rel=1e-12)
    assert abs(g[1]) < 1e-12 and abs(g[2]) < 1e-12


def test_oracle_u8_equals_u16_rendering(golden):
    """The reference kernels are type-generic: integer data renders the
    same whether stored as uint8 or uint16."""
    arr, spacing, spec, want_px, want_count = golden.frame("c1_sphere64_u8")
    px16, c16 = oracle.render(arr.astype(np.uint16), spacing, spec, threads=4)
    px8, c8 = oracle.render(arr, spacing, spec, threads=4)
    assert np.array_equal(px8, px16) and c8 == c16


def test_oracle_box_interval_known_answers():
    """test_raycast_geometry.py:116-140."""
    assert oracle.box_interval((-1, 0.5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1)) == (1.0, 2.0)
    assert oracle.box_interval((0.5, 0.5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1)) == (0.0, 0.5)
    assert oracle.box_interval((-1, 5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1)) is None
    assert oracle.box_interval((2, 0.5, 0.5), (1, 0, 0), (0, 0, 0), (1, 1, 1)) is None
    assert oracle.box_interval((1.0, 0.5, -2), (0, 0, 1), (0, 0, 0), (1, 1, 1)) == (2.0, 3.0)


def test_oracle_march_step_plane_known_answer():
    """test_raycast_pipeline.py:80-92: step plane at x index 8 -> hit.t == 8.0."""
    arr = np.zeros((16, 16, 16), np.uint16)
    arr[:, :, 8:] = 1000
    iv = oracle.box_interval((0, 8, 8), (1, 0, 0), (0, 0, 0), (16, 16, 16))
    t_hit, t_before, bracket = oracle.first_hit(arr, (1, 1, 1), (0, 8, 8), (1, 0, 0), iv, 1.0,
                                                0.125, (500.0, 4095.0))
    assert t_hit == pytest.approx(8.0, abs=1e-12) and bracket
    assert t_before == pytest.approx(8.0 - 0.125, abs=1e-12)
