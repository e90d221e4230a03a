#!/usr/bin/env python3
"""Quick device-time comparison of raycast variants on the C3 workload
(development tool; bench.py is the contract benchmark).

  python tools/kbench.py [--frames 20] [--size 512] [--variants volume,taps,...]

Each variant: name = gradient source [+noskip] [+surface] [+op].
Prints ms/frame (CUDA events on the launching stream, L2 flushed between
frames) and executed work counters.
"""

from __future__ import annotations

import argparse
import ctypes
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--variants", default="volume,taps,volume+surface,volume+noskip")
    ap.add_argument("--spacing", default="1,1,1", help="voxel spacing (non power-of-two: division path)")
    a = ap.parse_args()

    import torch

    import paper_1609_01317_b200 as vc
    from paper_1609_01317_b200 import _native, phantoms
    from paper_1609_01317_b200.raycast import render_params

    vol = phantoms.ct_phantom(a.size)
    sp = tuple(float(x) for x in a.spacing.split(","))
    if sp != (1.0, 1.0, 1.0):
        vol = vc.Volume.from_array(vol.as_array(), spacing=sp)
    dv = vc.device_volume(vol)
    L = _native.load(build_if_missing=False)
    out = torch.empty((a.height, a.width, 4), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(_native.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    ref_img = None
    for name in a.variants.split(","):
        parts = name.split("+")
        grad = parts[0]
        mode = "surface" if "surface" in parts else "composited"
        op = vc.OperatorKind.ZUCKER_HUMMEL
        for p in parts:
            if p in ("central", "sobel3d"):
                op = vc.OperatorKind(p)

        def params(i, counting=False):
            sc, st = phantoms.scene_c3(vol, op=op, width=a.width, height=a.height, azimuth=float(i),
                                       mode=mode)
            st = replace(st, gradient_source=grad, use_octree="noskip" not in parts)
            if "tex" in parts:  # hardware texture sampler
                st = replace(st, sampler="texture")
            if "adaptive" in parts:  # use_adaptive (with the octree: the segment walk)
                st = replace(st, use_adaptive=True)
                dv.ensure_octree(vol, st.octree_min_block, st.octree_max_depth)
            if "norefine" in parts:  # work accounting only: no bisection
                st = replace(st, refine_iters=0)
            return render_params(vol, sc, st)

        for i in range(3):
            P = params(i)
            _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), None, sp))
        times = []
        for i in range(a.frames):
            P = params(10 + i)
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), None, sp))
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        stage = np.zeros(2)
        sms = (ctypes.c_float * 2)()
        for i in range(a.frames):  # per-stage device time (events between the two kernels)
            P = params(10 + i)
            flush.zero_()
            _native.check(L.vc_render_profiled(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()),
                                               None, sp, sms))
            stage += np.array([sms[0], sms[1]])
        stage /= a.frames
        P = params(10)
        _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()),
                                  ctypes.c_void_p(cnt.data_ptr()), sp))
        torch.cuda.synchronize()
        img = out.cpu().numpy().copy()
        c = cnt.cpu().numpy().tolist()
        diff = ""
        if ref_img is not None and ref_img.shape == img.shape and mode == ref_mode:
            diff = f" max|d| vs first={int(np.abs(img.astype(int) - ref_img.astype(int)).max())}"
        if ref_img is None:
            ref_img, ref_mode = img, mode
        t = np.array(times)
        print(f"{name:28s} {t.mean():7.3f} ms (min {t.min():.3f}, max {t.max():.3f})  "
              f"fps {1000 / t.mean():7.1f}  stages {stage[0]:.3f}+{stage[1]:.3f}  samples {c[0]/1e6:6.2f}M shades {c[1]/1e6:5.2f}M "
              f"skip-events {c[2]/1e6:6.1f}M st1 {c[4]/1e6:6.2f}M st2 {c[5]/1e6:6.2f}M{diff}", flush=True)


if __name__ == "__main__":
    main()
