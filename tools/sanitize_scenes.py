#!/usr/bin/env python3
"""Smoke-sized launches of every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), one tool per run:

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_scenes.py

Covers: firsthit_kernel + shade_kernel (reference taps and gradient volume,
with and without empty-space skipping, surface and composited), the texture
sampler, the octree-segment walk (use_adaptive; use_octree with 0 in the
window), the TMA gradient pre-pass (all operators, u8 / u16 / f32, a width
whose rows are not 16-byte multiples), the macrocell / distance-field
kernels, the point kernels, the device PNG encoder and vc_render_to_peers
(one local frame in the peer table).
"""

from __future__ import annotations

import ctypes
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import argparse

    import torch

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", help="save a few frames (npz) for comparison with another build")
    a = ap.parse_args()
    saved = {}

    import paper_1609_01317_b200 as vc
    from paper_1609_01317_b200 import _native, phantoms
    from paper_1609_01317_b200.raycast import render_params

    L = _native.load(build_if_missing=False)
    ct = phantoms.ct_phantom(40)
    for mode in ("surface", "composited"):
        for grad in ("taps", "volume"):
            for skip in (False, True):
                for op in vc.OperatorKind:
                    sc, st = phantoms.scene_c3(ct, op=op, width=48, height=32, azimuth=30.0, mode=mode)
                    fb = vc.render_frame(ct, sc, replace(st, gradient_source=grad, use_octree=skip))
                    saved[f"{mode}_{grad}_{int(skip)}_{op.value}"] = fb.pixels.copy()
    sc, st = phantoms.scene_c3(ct, width=48, height=32, azimuth=10.0)
    vc.render_frame(ct, sc, replace(st, sampler="texture", gradient_source="volume"))
    saved["adaptive_octree"] = vc.render_frame(ct, sc, replace(st, use_adaptive=True, use_octree=True)).pixels.copy()
    saved["adaptive"] = vc.render_frame(ct, sc, replace(st, use_adaptive=True, use_octree=False)).pixels.copy()
    zero = vc.Scene(camera=sc.camera, light=sc.light, window=vc.ThresholdWindow(-100.0, 800.0),
                    transfer=sc.transfer)
    saved["zero_window"] = vc.render_frame(ct, zero, st).pixels.copy()  # octree-segment walk, 0 in the window
    for interp in ("nearest", "linear"):
        vc.render_frame(ct, sc, replace(st, interpolation=vc.InterpolationMode(interp)))
    rng = np.random.default_rng(1)
    for dt, shape in ((np.uint8, (9, 11, 13)), (np.uint16, (17, 10, 7)), (np.float32, (12, 9, 21))):
        arr = rng.integers(0, 200, size=shape).astype(dt)
        v = vc.Volume.from_array(arr, dtype=dt)
        for op in vc.OperatorKind:
            vc.gradient_volume(v, op)
            vc.gradient(v, (3.3, 4.1, 2.2), op)
        vc.sample(v, (1.5, 2.5, 3.5))
        s2, t2 = phantoms.scene_c3(v, width=24, height=16, azimuth=20.0)
        vc.render_frame(v, vc.Scene(camera=s2.camera, light=s2.light, window=vc.ThresholdWindow(50.0, 150.0),
                                    transfer=s2.transfer), replace(t2, gradient_source="volume"))
    fb = vc.render_frame(ct, sc, st)
    vc.png_bytes(fb.pixels)
    # vc_render_to_peers: two virtual ranks in one process (tile pushes with
    # band_rows 8, per-pixel stores with band_rows 6) + done flags
    frames = [torch.zeros((st.height, st.width, 4), dtype=torch.uint8, device="cuda") for _ in range(2)]
    done = [torch.zeros(_native.MAX_PEERS, dtype=torch.int32, device="cuda") for _ in range(2)]
    ftab = torch.tensor([f.data_ptr() for f in frames], dtype=torch.int64, device="cuda")
    dtab = torch.tensor([d.data_ptr() for d in done], dtype=torch.int64, device="cuda")
    for seq, band_rows in ((1, 8), (2, 6)):
        for r in range(2):
            P = render_params(ct, sc, st, band_rows=band_rows, band_first=r, band_step=2)
            desc = _native.PeerFramesDesc(ftab.data_ptr(), dtab.data_ptr(), frames[0].numel(), 2, r, -1, seq)
            _native.check(L.vc_render_to_peers(vc.device_volume(ct).handle, ctypes.byref(P), ctypes.byref(desc),
                                               None, None))
        torch.cuda.synchronize()
        for f in frames:
            assert np.array_equal(f.cpu().numpy(), fb.pixels)
    if a.out:
        np.savez_compressed(a.out, **saved)
    report = {"scenes": "ok", "library": str(_native.library_path())}
    if hasattr(L, "vc_checked_violations"):
        first = ctypes.c_ulonglong(0)
        report["violations"] = int(L.vc_checked_violations(ctypes.byref(first)))
        report["first_violation_address"] = hex(first.value)
    import json

    print(json.dumps(report))


if __name__ == "__main__":
    main()
