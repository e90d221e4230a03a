#!/usr/bin/env python3
"""Where the end-to-end frame rate goes (development): host cost of building
a frame's parameters, device throughput of back-to-back frames on 1-3
streams (no copies, no L2 flush), and render_sequence at depths 2-4.

  python tools/pipeline_probe.py [--frames 200]
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys
import time
from dataclasses import replace

sys.path.insert(0, os.getcwd())

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=200)
    a = ap.parse_args()
    import torch

    import paper_1609_01317_b200 as vc
    from paper_1609_01317_b200 import _native, phantoms
    from paper_1609_01317_b200.raycast import render_params

    vol = phantoms.ct_phantom(512)
    frames = [(lambda s: (s[0], replace(s[1], gradient_source="volume")))(phantoms.scene_c3(vol, azimuth=float(i)))
              for i in range(a.frames)]
    dv = vc.device_volume(vol)
    dv.gradient_prepass(2)
    L = _native.load()
    t = time.perf_counter()
    Ps = [render_params(vol, sc, st) for sc, st in frames]
    print(f"render_params host cost {1e6 * (time.perf_counter() - t) / len(frames):.1f} us/frame")
    H, W = 1080, 1920
    for nstreams in (1, 2, 3):
        streams = [torch.cuda.Stream() for _ in range(nstreams)]
        outs = [torch.empty((H, W, 4), dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
        for rep in range(2):
            torch.cuda.synchronize()
            t = time.perf_counter()
            for i, P in enumerate(Ps):
                s = streams[i % nstreams]
                _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(outs[i % nstreams].data_ptr()),
                                          None, ctypes.c_void_p(s.cuda_stream)))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
        print(f"device back-to-back, {nstreams} stream(s): {len(Ps) / dt:7.1f} fps")
    for depth in (2, 3, 4):
        for fb in vc.render_sequence(vol, iter(frames[:8]), depth=depth):
            pass
        best = 0.0
        for rep in range(3):
            t = time.perf_counter()
            for fb in vc.render_sequence(vol, iter(frames), depth=depth):
                pass
            best = max(best, len(frames) / (time.perf_counter() - t))
        print(f"render_sequence depth {depth}: {best:7.1f} fps")


if __name__ == "__main__":
    main()
