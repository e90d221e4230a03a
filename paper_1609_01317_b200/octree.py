"""Min/max octree (reference octree.py) in a level-grid form the device can walk.

The reference builds its octree top-down (octree.py:52-108): a node covers
a half-open voxel box, splits each axis of extent >= 2 at lo + ext // 2,
and stops when its voxels are uniform, its longest side is <= min_block, or
it reaches max_depth.  Because every split depends only on the node's own
interval on each axis, the candidate nodes of depth L form a product grid
of per-axis intervals; the tree is that grid pyramid plus, per level, which
boxes exist and which of them are leaves.  This module builds exactly that
(vectorised, seconds for 512^3 instead of a Python walk over millions of
nodes) and exposes the reference API on top of it:

  build_octree(volume, min_block=4, max_depth=8) -> Octree   (octree.py:52)
  Octree.root / OctreeNode (lo, hi, vmin, vmax, smin, smax, depth, children)
  skip_empty(ray, tree, window, interval, spacing)           (octree.py:139)
  adaptive_step(tree, position, base_step, coarse_factor, detail_epsilon)
                                                             (octree.py:158)

Ranges follow the reference: (vmin, vmax) over the node's voxels, (smin,
smax) over the box padded by one voxel on every side (octree.py:4-8).  The
renderer needs the tree only for adaptive stepping (use_adaptive,
_kernels.py:437-463); the level grid is uploaded to the device volume with
vc_volume_set_octree.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .volume import Volume


@dataclass
class OctreeNode:
    lo: tuple[int, int, int]
    hi: tuple[int, int, int]
    vmin: int
    vmax: int
    smin: int
    smax: int
    depth: int
    children: list["OctreeNode"] = field(default_factory=list)

    @property
    def is_leaf(self) -> bool:
        return not self.children


def _axis_levels(n: int, depth: int):
    """Per-level interval lists of one axis plus child index ranges."""
    levels = [np.array([[0, n]], np.int64)]
    kids = []
    for _ in range(depth):
        prev = levels[-1]
        ext = prev[:, 1] - prev[:, 0]
        split = ext >= 2
        mid = prev[:, 0] + ext // 2
        counts = np.where(split, 2, 1)
        start = np.concatenate([[0], np.cumsum(counts)[:-1]])
        nxt = np.empty((int(counts.sum()), 2), np.int64)
        nxt[start, 0] = prev[:, 0]
        nxt[start, 1] = np.where(split, mid, prev[:, 1])
        s2 = start[split] + 1
        nxt[s2, 0] = mid[split]
        nxt[s2, 1] = prev[split, 1]
        levels.append(nxt)
        parent = np.repeat(np.arange(len(prev)), counts)
        kids.append((start, counts, parent))
    return levels, kids


def _box_reduce(arr: np.ndarray, zs, ys, xs, fn):
    m = fn.reduceat(arr, xs[:, 0], axis=2)
    m = fn.reduceat(m, ys[:, 0], axis=1)
    return fn.reduceat(m, zs[:, 0], axis=0)


def _neighbour_filter(arr: np.ndarray, fn) -> np.ndarray:
    """fn over the (clipped) 3x3x3 neighbourhood, separably."""
    out = arr.copy()
    for ax in range(3):
        src = out.copy()
        sl_lo = [slice(None)] * 3
        sl_hi = [slice(None)] * 3
        sl_lo[ax], sl_hi[ax] = slice(0, -1), slice(1, None)
        fn(out[tuple(sl_lo)], src[tuple(sl_hi)], out=out[tuple(sl_lo)])
        fn(out[tuple(sl_hi)], src[tuple(sl_lo)], out=out[tuple(sl_hi)])
    return out


class Octree:
    """Level-grid octree; `root` materialises reference-style nodes on demand."""

    def __init__(self, volume: Volume, min_block: int, max_depth: int):
        if min_block < 1:
            raise ValueError(f"min_block must be >= 1, got {min_block}")
        if not 0 <= max_depth <= 16:
            raise ValueError(f"max_depth must be within [0, 16], got {max_depth}")
        arr = volume.as_array()
        nx, ny, nz = volume.dims
        self.volume_dims = volume.dims
        self.value_range = (volume.value_min, volume.value_max)
        self.min_block = min_block
        self.max_depth = max_depth
        # deepest level any node can reach: stop once every interval is <= min_block
        depth = 0
        while depth < max_depth:
            longest = max(math.ceil(n / (1 << depth)) for n in (nx, ny, nz))
            if longest <= min_block:
                break
            depth += 1
        self.depth = depth
        self.ax = [_axis_levels(n, depth) for n in (nx, ny, nz)]  # x, y, z
        D = depth
        xs, ys, zs = (self.ax[a][0][D] for a in range(3))
        # min / max never overflow: reduce in the storage type, widen the small grids
        wide = np.float64 if arr.dtype == np.float32 else np.int64
        fine = {
            "vmin": _box_reduce(arr, zs, ys, xs, np.minimum).astype(wide),
            "vmax": _box_reduce(arr, zs, ys, xs, np.maximum).astype(wide),
            "smin": _box_reduce(_neighbour_filter(arr, np.minimum), zs, ys, xs, np.minimum).astype(wide),
            "smax": _box_reduce(_neighbour_filter(arr, np.maximum), zs, ys, xs, np.maximum).astype(wide),
        }
        # coarser levels from their children (boxes nest)
        self.ranges = [None] * (D + 1)
        self.ranges[D] = fine
        for L in range(D - 1, -1, -1):
            xk, yk, zk = (self.ax[a][1][L] for a in range(3))
            child = self.ranges[L + 1]
            lvl = {}
            for key, fn in (("vmin", np.minimum), ("vmax", np.maximum), ("smin", np.minimum),
                            ("smax", np.maximum)):
                m = fn.reduceat(child[key], xk[0], axis=2)
                m = fn.reduceat(m, yk[0], axis=1)
                lvl[key] = fn.reduceat(m, zk[0], axis=0)
            self.ranges[L] = lvl
        # which boxes exist / split (octree.py:93-96 stop rules)
        self.exists = [np.ones((1, 1, 1), bool)]
        self.leaf = []
        for L in range(D + 1):
            xsL, ysL, zsL = (self.ax[a][0][L] for a in range(3))
            ext = np.maximum.outer(np.maximum.outer(zsL[:, 1] - zsL[:, 0], ysL[:, 1] - ysL[:, 0]),
                                   xsL[:, 1] - xsL[:, 0])
            r = self.ranges[L]
            split = self.exists[L] & (r["vmin"] != r["vmax"]) & (ext > min_block) & (L < max_depth)
            self.leaf.append(self.exists[L] & ~split)
            if L < D:
                px, py, pz = (self.ax[a][1][L][2] for a in range(3))
                self.exists.append(split[pz][:, py][:, :, px])
            else:
                assert not split.any()
        self.node_count = int(sum(e.sum() for e in self.exists))
        self._root = None
        self._flat = None

    # ------------------------------------------------------------ reference API

    @property
    def root(self) -> OctreeNode:
        if self._root is None:
            self._root = self._node(0, 0, 0, 0)
        return self._root

    def _node(self, L, iz, iy, ix) -> OctreeNode:
        xs, ys, zs = (self.ax[a][0][L] for a in range(3))
        r = self.ranges[L]
        conv = float if isinstance(r["vmin"].flat[0], np.floating) else int
        node = OctreeNode(lo=(int(xs[ix, 0]), int(ys[iy, 0]), int(zs[iz, 0])),
                          hi=(int(xs[ix, 1]), int(ys[iy, 1]), int(zs[iz, 1])),
                          vmin=conv(r["vmin"][iz, iy, ix]), vmax=conv(r["vmax"][iz, iy, ix]),
                          smin=conv(r["smin"][iz, iy, ix]), smax=conv(r["smax"][iz, iy, ix]), depth=L)
        if not self.leaf[L][iz, iy, ix]:
            (sx, cx, _), (sy, cy, _), (sz, cz, _) = (self.ax[a][1][L] for a in range(3))
            for kz in range(sz[iz], sz[iz] + cz[iz]):
                for ky in range(sy[iy], sy[iy] + cy[iy]):
                    for kx in range(sx[ix], sx[ix] + cx[ix]):
                        node.children.append(self._node(L + 1, kz, ky, kx))
        return node

    def leaf_box(self, ix: int, iy: int, iz: int):
        """(level, (bz, by, bx)) of the leaf containing voxel (ix, iy, iz)."""
        for L in range(self.depth + 1):
            xs, ys, zs = (self.ax[a][0][L] for a in range(3))
            bx = int(np.searchsorted(xs[:, 1], ix, side="right"))
            by = int(np.searchsorted(ys[:, 1], iy, side="right"))
            bz = int(np.searchsorted(zs[:, 1], iz, side="right"))
            if self.leaf[L][bz, by, bx]:
                return L, (bz, by, bx)
        raise AssertionError("no leaf contains the voxel")

    # ------------------------------------------------------------ device form

    def device_arrays(self):
        """Flat arrays of vc_octree_desc (include/voxelcast_b200.h)."""
        states = [np.where(self.leaf[L], 2, np.where(self.exists[L], 1, 0)).astype(np.uint8)
                  for L in range(self.depth + 1)]
        sranges = [np.stack([r["smin"], r["smax"]], axis=-1).astype(np.float64) for r in self.ranges]
        return _pack_levels(self.volume_dims, self.ax, states, sranges)


def _pack_levels(volume_dims, ax, states, sranges):
    """vc_octree_desc arrays from per-level axis intervals, box states
    (0 absent, 1 internal, 2 leaf; [bz, by, bx]) and padded ranges."""
    nx, ny, nz = volume_dims
    levels = len(states)
    dims = np.zeros((levels, 3), np.int32)
    amap = np.zeros((levels, nx + ny + nz), np.int32)
    ivl_off = np.zeros((levels, 3), np.int32)
    box_off = np.zeros(levels, np.int64)
    ivl, state, srange = [], [], []
    off = 0
    boff = 0
    for L in range(levels):
        for a, n in enumerate((nx, ny, nz)):
            iv = ax[a][0][L]
            dims[L, a] = len(iv)
            ivl_off[L, a] = off
            ivl.append(iv.astype(np.int32).ravel())
            off += 2 * len(iv)
            base = (0, nx, nx + ny)[a]
            amap[L, base:base + n] = np.repeat(np.arange(len(iv), dtype=np.int32), iv[:, 1] - iv[:, 0])
        box_off[L] = boff
        boff += states[L].size
        state.append(states[L].ravel())
        srange.append(np.asarray(sranges[L], np.float64).ravel())
    return {
        "levels": levels, "dims": dims.ravel(), "axis_map": amap.ravel(),
        "ivl_off": ivl_off.ravel(), "ivl": np.concatenate(ivl), "box_off": box_off,
        "state": np.concatenate(state), "srange": np.concatenate(srange),
    }


def flat_arrays(tree: Octree):
    """The reference's array form of the tree (octree.py:114-135): per node
    voxel bounds (lo, hi), exact and padded ranges, child indices (-1
    padded), nodes in the reference's depth-first order.  Cached on the tree."""
    cached = getattr(tree, "_flat", None)
    if cached is not None:
        return cached
    nodes: list[OctreeNode] = []
    stack = [tree.root]
    while stack:
        n = stack.pop()
        nodes.append(n)
        stack.extend(n.children)
    index = {id(n): i for i, n in enumerate(nodes)}
    cnt = len(nodes)
    nbounds = np.empty((cnt, 6), np.int32)
    vminmax = np.empty((cnt, 2), np.float64)
    sminmax = np.empty((cnt, 2), np.float64)
    nchildren = np.full((cnt, 8), -1, np.int32)
    for i, n in enumerate(nodes):
        nbounds[i] = (*n.lo, *n.hi)
        vminmax[i] = (n.vmin, n.vmax)
        sminmax[i] = (n.smin, n.smax)
        for c, ch in enumerate(n.children):
            nchildren[i, c] = index[id(ch)]
    tree._flat = (nbounds, vminmax, sminmax, nchildren)
    return tree._flat


def device_arrays_from_flat(volume_dims, nbounds, sminmax, nchildren):
    """vc_octree_desc arrays of a tree given in the reference's flat form
    (what _kernels.render_tile receives, _kernels.py:582-627).  Every split
    halves an axis interval the same way wherever it sits (octree.py:93-107),
    so the nodes of depth L lie on the level-L interval grid; this places
    each node there.  Raises ValueError for arrays that are not such a tree."""
    nb = np.asarray(nbounds, np.int64).reshape(-1, 6)
    sm = np.asarray(sminmax, np.float64).reshape(-1, 2)
    ch = np.asarray(nchildren, np.int64).reshape(-1, 8)
    n = len(nb)
    if n == 0 or len(sm) < n or len(ch) < n:
        raise ValueError("octree arrays are empty or of unequal length")
    depth = np.full(n, -1, np.int64)
    depth[0] = 0
    order = [0]
    for i in order:  # breadth first from the root
        for c in ch[i]:
            if c < 0:
                break
            if not 0 < c < n or depth[c] >= 0:
                raise ValueError("octree child index out of range or repeated")
            depth[c] = depth[i] + 1
            order.append(int(c))
    if len(order) != n:
        raise ValueError("octree has unreachable nodes")
    D = int(depth.max())
    if D > 16:
        raise ValueError("octree deeper than 16 levels")
    ax = [_axis_levels(d, D) for d in volume_dims]
    states, sranges = [], []
    for L in range(D + 1):
        sel = np.nonzero(depth == L)[0]
        idx = []
        for a in range(3):
            iv = ax[a][0][L]
            k = np.searchsorted(iv[:, 0], nb[sel, a])
            k = np.minimum(k, len(iv) - 1)
            if not (np.array_equal(iv[k, 0], nb[sel, a]) and np.array_equal(iv[k, 1], nb[sel, 3 + a])):
                raise ValueError(f"octree node bounds at depth {L} are not the reference's halving split")
            idx.append(k)
        shape = (len(ax[2][0][L]), len(ax[1][0][L]), len(ax[0][0][L]))
        st = np.zeros(shape, np.uint8)
        sr = np.zeros(shape + (2,), np.float64)
        st[idx[2], idx[1], idx[0]] = np.where(ch[sel, 0] < 0, 2, 1)
        sr[idx[2], idx[1], idx[0]] = sm[sel]
        states.append(st)
        sranges.append(sr)
    return _pack_levels(tuple(int(d) for d in volume_dims), ax, states, sranges)


def build_octree(volume: Volume, min_block: int = 4, max_depth: int = 8) -> Octree:
    """Top-down subdivision of the full grid (octree.py:52-108)."""
    return Octree(volume, min_block, max_depth)


def _node_interval(lo, hi, spacing, org, dirv):
    """_kernels._node_interval (_kernels.py:227-264) for one box."""
    tmin, tmax = -1e300, 1e300
    for a in range(3):
        l, h = lo[a] * spacing[a], hi[a] * spacing[a]
        o, d = float(org[a]), float(dirv[a])
        if d == 0.0:
            if o < l or o > h:
                return None
        else:
            inv = 1.0 / d
            ta, tb = (l - o) * inv, (h - o) * inv
            if ta > tb:
                ta, tb = tb, ta
            tmin = max(tmin, ta) if ta > tmin else tmin
            tmax = min(tmax, tb) if tb < tmax else tmax
    if tmin > tmax:
        return None
    return tmin, tmax


def skip_empty(ray, tree: Octree, window, interval, spacing=(1.0, 1.0, 1.0)) -> list[tuple[float, float]]:
    """Merged, ascending t-intervals of leaves whose padded value range
    overlaps the window, clipped to interval (octree.py:139-155,
    _kernels.collect_segments :267-342).  Host-side API helper; the renderer
    skips empty space with its own macrocell grid."""
    org = np.asarray(ray.origin, np.float64)
    dirv = np.asarray(ray.direction, np.float64)
    t0, t1 = float(interval[0]), float(interval[1])
    segs: list[list[float]] = []
    stack = [tree.root]
    while stack:
        node = stack.pop()
        iv = _node_interval(node.lo, node.hi, spacing, org, dirv)
        if iv is None:
            continue
        a0, b0 = max(iv[0], t0), min(iv[1], t1)
        if b0 < a0:
            continue
        if node.is_leaf:
            if node.smin <= window.high and node.smax >= window.low:
                if segs and a0 <= segs[-1][1] + 1e-9:
                    if b0 > segs[-1][1]:
                        segs[-1][1] = b0
                elif len(segs) < 4096:
                    segs.append([a0, b0])
                else:
                    segs[-1][1] = b0
        else:
            kids = []
            for ch in node.children:
                civ = _node_interval(ch.lo, ch.hi, spacing, org, dirv)
                if civ is None or civ[1] < t0 or civ[0] > t1:
                    continue
                kids.append((civ[0], ch))
            kids.sort(key=lambda x: -x[0])  # farthest first, nearest pops first
            stack.extend(ch for _, ch in kids)
    return [(float(a), float(b)) for a, b in segs]


def adaptive_step(tree: Octree, position, base_step: float, coarse_factor: int = 4,
                  detail_epsilon: float | None = None) -> float:
    """Step length at a voxel-space position: base_step in detailed regions,
    coarse_factor times that inside low-variation leaves (octree.py:158-181)."""
    if base_step <= 0:
        raise ValueError(f"base_step must be positive, got {base_step}")
    if coarse_factor < 1:
        raise ValueError(f"coarse_factor must be >= 1, got {coarse_factor}")
    if detail_epsilon is None:
        detail_epsilon = 0.01 * max(1, tree.value_range[1] - tree.value_range[0])
    nx, ny, nz = tree.volume_dims
    ix = min(max(int(np.floor(position[0])), 0), nx - 1)
    iy = min(max(int(np.floor(position[1])), 0), ny - 1)
    iz = min(max(int(np.floor(position[2])), 0), nz - 1)
    L, (bz, by, bx) = tree.leaf_box(ix, iy, iz)
    r = tree.ranges[L]
    if float(r["smax"][bz, by, bx]) - float(r["smin"][bz, by, bx]) < detail_epsilon:
        return float(base_step * coarse_factor)
    return float(base_step)
