"""CPU tests of the level-grid octree (paper_1609_01317_b200.octree) against
the oracle's restatement of the reference build (octree.py:52-136) and the
reference's own octree invariants (pkg/tests/test_octree.py)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from oracle import oracle
from paper_1609_01317_b200 import phantoms


def walk(node):
    out = [node]
    i = 0
    while i < len(out):
        out.extend(out[i].children)
        i += 1
    return out


def volumes():
    rng = np.random.default_rng(99)
    return [
        vc.make_phantom("sphere", 32, radius=10),
        vc.make_phantom("shell", 33, r_inner=8, r_outer=12),
        vc.Volume.from_array(rng.integers(0, 4096, size=(16, 17, 19), dtype=np.uint16)),
        phantoms.ct_phantom(40),
        vc.make_phantom("empty", 16),
        vc.Volume.from_array(rng.integers(0, 3, size=(5, 9, 2), dtype=np.uint16)),
    ]


@pytest.mark.parametrize("idx", range(6))
@pytest.mark.parametrize("min_block,max_depth", [(4, 8), (2, 3), (1, 16), (8, 0)])
def test_tree_matches_reference_build(idx, min_block, max_depth):
    vol = volumes()[idx]
    tree = vc.build_octree(vol, min_block=min_block, max_depth=max_depth)
    nb, sm, ch = oracle.build_octree_flat(vol.as_array(), min_block, max_depth)
    assert tree.node_count == len(nb)
    mine = sorted((n.lo, n.hi, n.smin, n.smax, n.is_leaf) for n in walk(tree.root))
    ref = sorted((tuple(int(x) for x in nb[i, :3]), tuple(int(x) for x in nb[i, 3:]),
                  int(sm[i, 0]), int(sm[i, 1]), bool(ch[i, 0] < 0)) for i in range(len(nb)))
    assert mine == ref


def test_reference_invariants_on_sphere():
    """test_octree.py:52-109: extrema, partition, stop rules."""
    vol = vc.make_phantom("sphere", 32, radius=10)
    tree = vc.build_octree(vol, min_block=4)
    a = vol.as_array()
    nx, ny, nz = vol.dims
    total = 0
    for node in walk(tree.root):
        lo, hi = node.lo, node.hi
        blk = a[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]]
        assert (node.vmin, node.vmax) == (int(blk.min()), int(blk.max()))
        pad = a[max(lo[2] - 1, 0):min(hi[2] + 1, nz), max(lo[1] - 1, 0):min(hi[1] + 1, ny),
                max(lo[0] - 1, 0):min(hi[0] + 1, nx)]
        assert (node.smin, node.smax) == (int(pad.min()), int(pad.max()))
        if node.is_leaf:
            total += int(np.prod([h - l for l, h in zip(lo, hi)]))
        else:
            assert max(h - l for l, h in zip(lo, hi)) > tree.min_block
            assert node.vmin < node.vmax and node.depth < tree.max_depth
            assert 2 <= len(node.children) <= 8
    assert total == nx * ny * nz
    assert vc.build_octree(vc.make_phantom("empty", 16)).node_count == 1
    with pytest.raises(ValueError):
        vc.build_octree(vol, min_block=0)
    with pytest.raises(ValueError):
        vc.build_octree(vol, max_depth=-1)


def test_adaptive_step_and_skip_empty_api():
    """octree.py:139-181 helpers (test_octree.py:129-200 properties)."""
    vol = vc.make_phantom("sphere", 32, radius=10)
    tree = vc.build_octree(vol, min_block=4)
    assert vc.adaptive_step(tree, (1.0, 1.0, 1.0), 0.5, 4) == 2.0  # empty corner leaf
    assert vc.adaptive_step(tree, (15.5, 15.5, 5.6), 0.5, 4) == 0.5  # on the sphere surface
    with pytest.raises(ValueError):
        vc.adaptive_step(tree, (1, 1, 1), 0.0)
    ray = vc.Ray(origin=(16.0, 16.0, -5.0), direction=(0.0, 0.0, 1.0))
    assert vc.skip_empty(ray, tree, vc.ThresholdWindow(2000.0, 4095.0), (0.0, 37.0)) == []
    segs = vc.skip_empty(ray, tree, vc.ThresholdWindow(500.0, 4095.0), (0.0, 37.0))
    assert segs and all(0.0 <= a <= b <= 37.0 for a, b in segs)
    flat = vc.Volume.from_array(np.full((16, 16, 16), 600, np.uint16))
    segs = vc.skip_empty(vc.Ray(origin=(8.0, 8.0, -4.0), direction=(0.0, 0.0, 1.0)),
                         vc.build_octree(flat), vc.ThresholdWindow(500.0, 4095.0), (4.0, 20.0))
    assert segs == [(4.0, 20.0)]


def test_device_arrays_are_consistent():
    vol = phantoms.ct_phantom(40)
    tree = vc.build_octree(vol)
    d = tree.device_arrays()
    assert d["levels"] == tree.depth + 1
    assert d["state"].size == sum(e.size for e in tree.exists)
    assert (d["state"] == 2).sum() == sum(int(l.sum()) for l in tree.leaf)
    assert d["srange"].size == 2 * d["state"].size
