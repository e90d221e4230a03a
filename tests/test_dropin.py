"""The drop-in at the reference's module name (pkg/src/voxelcast) and the
vendored reference suite: import surface, kernel-layer signatures, the
reference-form octree conversion.  CPU only (no compute calls)."""

from __future__ import annotations

import hashlib
import inspect
from pathlib import Path

import numpy as np
import pytest

import voxelcast
from paper_1609_01317_b200 import octree as impl_octree
from tests.conftest import PKG_SRC, REFERENCE_SUITE

REFERENCE_TESTS = Path("/root/reference/pkg/tests")
REFERENCE_SRC = Path("/root/reference/pkg/src/voxelcast")

# reference __all__ (voxelcast/__init__.py:48-96) minus the PPM I/O, which is
# out of scope
REFERENCE_ALL = [
    "Camera", "ClipBox", "EPS_GRADIENT", "FrameBuffer", "Hit", "InterpolationMode", "Light", "Octree",
    "OctreeNode", "OperatorKind", "PhantomKind", "Ray", "RenderMode", "RenderSettings", "Scene",
    "ThresholdWindow", "TransferFunction", "Volume", "adaptive_step", "build_octree",
    "central_difference", "composite_step", "default_scene", "generate_ray", "gradient", "hounsfield",
    "intersect_clipbox", "lerp", "load_raw_slices", "make_phantom", "march_surface",
    "normalize_gradient", "png_bytes", "refine_hitpoint", "render_frame", "sample", "save_raw_slices",
    "shade", "skip_empty", "sobel3d", "transfer", "write_png", "zucker_hummel", "__version__",
]

# _kernels.render_tile's argument list (_kernels.py:583-626)
RENDER_TILE_ARGS = [
    "data", "nx", "ny", "nz", "spacing", "eye", "right", "upv", "fwd", "half_w", "half_h", "width",
    "height", "clip_lo", "clip_hi", "light_pos", "light_col", "t_low", "t_high", "lut_hu", "lut_rgba",
    "mu_water", "op", "interp", "mode", "coarse", "fine", "refine_iters", "bg", "use_octree", "nbounds",
    "sminmax", "nchildren", "use_adaptive", "adapt_jump", "detail_eps", "y0", "y1", "out", "counter",
    "stack", "seg0", "seg1",
]


def test_voxelcast_resolves_to_the_dropin():
    assert Path(voxelcast.__file__).resolve().parent == (PKG_SRC / "voxelcast").resolve()
    for name in REFERENCE_ALL:
        assert hasattr(voxelcast, name), name
    import voxelcast.raycast as r
    import voxelcast.volume as v
    from voxelcast.octree import flat_arrays  # noqa: F401  (test_octree.py:18)
    from voxelcast.bench import BenchMatrix, fit_time_vs_pixels, run_benchmark  # noqa: F401
    from voxelcast._kernels import grad_raw, render_tile, sample_any  # noqa: F401

    assert r.Ray is voxelcast.Ray and v.Volume is voxelcast.Volume
    assert r.render_frame is voxelcast.render_frame


def test_kernel_layer_signatures_and_codes():
    from voxelcast import _kernels as k

    assert list(inspect.signature(k.render_tile).parameters) == RENDER_TILE_ARGS
    assert list(inspect.signature(k.grad_raw).parameters) == ["data", "nx", "ny", "nz", "x", "y", "z", "op"]
    assert list(inspect.signature(k.sample_any).parameters) == ["data", "nx", "ny", "nz", "x", "y", "z",
                                                                "interp"]
    assert (k.OP_CENTRAL, k.OP_SOBEL3D, k.OP_ZUCKER_HUMMEL) == (0, 1, 2)
    assert (k.INTERP_NEAREST, k.INTERP_LINEAR, k.INTERP_TRILINEAR) == (0, 1, 2)
    assert (k.MODE_SURFACE, k.MODE_COMPOSITED) == (0, 1)
    assert k.GRAD_SAMPLES == (6, 26, 26)


@pytest.mark.skipif(not REFERENCE_SRC.exists(), reason="reference tree not present (GPU box)")
def test_kernel_layer_matches_reference_source():
    import ast

    tree = ast.parse((REFERENCE_SRC / "_kernels.py").read_text())
    fns = {n.name: [a.arg for a in n.args.args] for n in tree.body if isinstance(n, ast.FunctionDef)}
    from voxelcast import _kernels as k

    for name in ("render_tile", "grad_raw", "sample_any", "sample_trilinear", "sample_nearest",
                 "sample_linear", "box_interval", "lerp", "normalize3"):
        assert list(inspect.signature(getattr(k, name)).parameters) == fns[name], name
    consts = {t.id: ast.literal_eval(n.value) for n in tree.body if isinstance(n, ast.Assign)
              for t in n.targets if isinstance(t, ast.Name) and t.id.isupper() and not t.id.startswith("_")
              and isinstance(n.value, (ast.Constant, ast.Tuple))}
    for name, val in consts.items():
        assert getattr(k, name) == val, name


def test_vendored_suite_is_byte_identical():
    sums = {}
    for line in (REFERENCE_SUITE / "SHA256SUMS").read_text().splitlines():
        digest, name = line.split()
        sums[name] = digest
    assert len(sums) == 8
    for name, digest in sums.items():
        assert hashlib.sha256((REFERENCE_SUITE / name).read_bytes()).hexdigest() == digest, name
        if REFERENCE_TESTS.exists():
            assert hashlib.sha256((REFERENCE_TESTS / name).read_bytes()).hexdigest() == digest, name


@pytest.mark.parametrize("shape,min_block,max_depth", [((32, 32, 32), 4, 8), ((17, 9, 23), 2, 8),
                                                        ((40, 24, 8), 4, 2), ((16, 16, 16), 4, 0),
                                                        ((33, 31, 29), 3, 5)])
def test_reference_form_octree_converts_to_the_device_form(shape, min_block, max_depth):
    """A tree handed over in the reference's flat form (what render_tile
    receives) becomes the same level grid build_octree uploads."""
    rng = np.random.default_rng(sum(shape))
    z, y, x = np.meshgrid(*(np.arange(n) for n in shape), indexing="ij")
    c = np.array(shape) / 2.0
    arr = np.where((z - c[0]) ** 2 + (y - c[1]) ** 2 + (x - c[2]) ** 2 <= (min(shape) / 3.0) ** 2,
                   rng.integers(500, 1500, size=shape), 0).astype(np.uint16)
    vol = voxelcast.Volume.from_array(arr)
    tree = impl_octree.build_octree(vol, min_block=min_block, max_depth=max_depth)
    nb, vmm, smm, ch = impl_octree.flat_arrays(tree)
    assert nb.shape == (tree.node_count, 6) and ch.shape == (tree.node_count, 8)
    want = tree.device_arrays()
    got = impl_octree.device_arrays_from_flat(vol.dims, nb, smm, ch)
    levels = got["levels"]
    assert levels <= want["levels"]
    for key in ("dims", "ivl_off", "box_off"):
        assert np.array_equal(got[key], want[key].reshape(want["levels"], -1)[:levels].ravel()), key
    n_ivl = got["ivl"].size
    assert np.array_equal(got["ivl"], want["ivl"][:n_ivl])
    n_box = got["state"].size
    assert np.array_equal(got["state"], want["state"][:n_box])
    assert not want["state"][n_box:].any()  # deeper levels of the build hold no node
    live = np.repeat(got["state"] > 0, 2)
    assert np.array_equal(got["srange"][live], want["srange"][: 2 * n_box][live])
    with pytest.raises(ValueError):
        bad = nb.copy()
        bad[-1, 0] += 1
        impl_octree.device_arrays_from_flat(vol.dims, bad, smm, ch)
