"""Large randomised parity sweep (development evidence, not a test): the
scene generator of tests/test_gpu_random.py over many more seeds, each
scene rendered by the device and the C oracle.  Prints one JSON summary
(written to profiles/ by hand).

usage: python tools/parity_sweep.py [--scenes N] [--adaptive N] [--first-seed S] [--big]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from dataclasses import replace

sys.path.insert(0, os.getcwd())

import numpy as np  # noqa: E402

import paper_1609_01317_b200 as vc  # noqa: E402
from oracle import oracle  # noqa: E402
from tests.specs import spec_of  # noqa: E402
from tests.test_gpu_random import _scene, _volumes, zero_window_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenes", type=int, default=1000)
    ap.add_argument("--adaptive", type=int, default=300)
    ap.add_argument("--first-seed", type=int, default=100000)
    ap.add_argument("--zero-window", type=int, default=0,
                    help="scenes with 0 inside the threshold window (use_octree replays the octree walk)")
    ap.add_argument("--big", action="store_true",
                    help="128^3 CT / 96^3 Marschner-Lobb / 48x40x56 noise volumes and 3x the image size")
    a = ap.parse_args()
    vols = _volumes()
    if a.big:
        from paper_1609_01317_b200 import phantoms

        r = np.random.default_rng(77)
        vols = {"ct": phantoms.ct_phantom(128).as_array(),
                "noise": r.integers(0, 4096, size=(56, 40, 48)).astype(np.uint16),
                "ml": phantoms.marschner_lobb(96).as_array()}
    names = ["ct", "noise", "ml"]
    res = {"scenes": 0, "brute_force_pixel_mismatch": 0, "count_mismatch": 0, "skipping_pixel_mismatch": 0,
           "gradient_volume_over_1lsb": 0, "gradient_volume_max_lsb": 0,
           "adaptive_scenes": 0, "adaptive_pixel_mismatch": 0, "adaptive_count_mismatch": 0,
           "adaptive_octree_scenes": 0, "zero_window_scenes": 0, "zero_window_mismatch": 0, "failures": []}
    t0 = time.perf_counter()
    for n in range(a.scenes):
        seed = a.first_seed + n
        rng = np.random.default_rng(seed)
        vol, sc, st = _scene(rng, vols[names[n % 3]], names[n % 3])
        if a.big:
            st = replace(st, width=3 * st.width, height=3 * st.height)
        want, cnt = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)))
        fb = vc.render_frame(vol, sc, replace(st, use_octree=False))
        res["scenes"] += 1
        if not np.array_equal(fb.pixels, want):
            res["brute_force_pixel_mismatch"] += 1
            res["failures"].append(("brute", seed))
        if fb.sample_count != cnt:
            res["count_mismatch"] += 1
            res["failures"].append(("count", seed))
        if not np.array_equal(vc.render_frame(vol, sc, replace(st, use_octree=True)).pixels, want):
            res["skipping_pixel_mismatch"] += 1
            res["failures"].append(("skip", seed))
        d = int(np.abs(vc.render_frame(vol, sc, replace(st, gradient_source="volume")).pixels.astype(int)
                       - want.astype(int)).max())
        res["gradient_volume_max_lsb"] = max(res["gradient_volume_max_lsb"], d)
        if d > 1:
            res["gradient_volume_over_1lsb"] += 1
            res["failures"].append(("gv", seed, d))
    for n in range(a.adaptive):
        seed = a.first_seed + 500000 + n
        rng = np.random.default_rng(seed)
        vol, sc, st = _scene(rng, vols[names[n % 3]], names[n % 3])
        if a.big:
            st = replace(st, width=3 * st.width, height=3 * st.height)
        vmax = float(vol.as_array().max())
        st = replace(st, use_adaptive=True, adaptive_factor=int(rng.integers(1, 9)),
                     detail_epsilon=None if rng.random() < 0.3 else float(rng.uniform(0.001, 0.3)) * vmax,
                     octree_min_block=int(rng.choice([2, 4, 8])), use_octree=bool(n % 2))
        want, cnt = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), octree=True)
        fb = vc.render_frame(vol, sc, st)
        res["adaptive_scenes"] += 1
        res["adaptive_octree_scenes"] += int(st.use_octree)
        if not np.array_equal(fb.pixels, want):
            res["adaptive_pixel_mismatch"] += 1
            res["failures"].append(("adaptive", seed))
        if fb.sample_count != cnt:
            res["adaptive_count_mismatch"] += 1
            res["failures"].append(("adaptive_count", seed))
    for n in range(a.zero_window):
        seed = a.first_seed + 900000 + n
        rng = np.random.default_rng(seed)
        vol, sc, st = _scene(rng, vols[names[n % 3]], names[n % 3])
        if a.big:
            st = replace(st, width=3 * st.width, height=3 * st.height)
        sc = zero_window_scene(rng, vol, sc)
        res["zero_window_scenes"] += 1
        for oct_on in (False, True):
            st2 = replace(st, use_octree=oct_on)
            want, cnt = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st2)), octree=True)
            fb = vc.render_frame(vol, sc, st2)
            if not np.array_equal(fb.pixels, want) or fb.sample_count != cnt:
                res["zero_window_mismatch"] += 1
                res["failures"].append(("zero_window", seed, oct_on))
            d = int(np.abs(vc.render_frame(vol, sc, replace(st2, gradient_source="volume")).pixels.astype(int)
                           - want.astype(int)).max())
            if d > 1:
                res["gradient_volume_over_1lsb"] += 1
                res["failures"].append(("zero_window_gv", seed, oct_on, d))
    res["seconds"] = round(time.perf_counter() - t0, 1)
    res["failures"] = res["failures"][:50]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
