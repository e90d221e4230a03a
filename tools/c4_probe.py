#!/usr/bin/env python3
"""C4 (1024^3 f32 fBm, 3840x2160, Sobel3D, composited) stage times and work
counters on one GPU (development).

  python tools/c4_probe.py [--frames 5] [--variants volume,taps]
"""
from __future__ import annotations

import argparse
import ctypes
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.getcwd())

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=5)
    ap.add_argument("--variants", default="volume,taps")
    a = ap.parse_args()
    import torch

    from paper_1609_01317_b200 import _native, phantoms
    from paper_1609_01317_b200.raycast import render_params
    from paper_1609_01317_b200.volume import DeviceVolume

    sys.path.insert(0, os.getcwd())
    from bench import _GridStub

    t = phantoms.fbm_noise_tensor(1024, device="cuda")
    vol = _GridStub((1024, 1024, 1024), float(t.min()), float(t.max()), np.float32)
    dv = DeviceVolume.from_device(0, t.data_ptr(), np.float32, vol.dims, vol.spacing)
    del t
    torch.cuda.empty_cache()
    dv.gradient_prepass(1)
    L = _native.load()
    out = torch.empty((2160, 3840, 4), dtype=torch.uint8, device="cuda")
    cnt = torch.zeros(_native.NUM_COUNTERS, dtype=torch.int64, device="cuda")
    sms = (ctypes.c_float * 2)()
    for v in a.variants.split(","):
        st_ms = np.zeros(2)
        for i in range(a.frames + 1):
            sc, st = phantoms.scene_c4(vol, azimuth=float(10 + i))
            P = render_params(vol, sc, replace(st, gradient_source=v))
            _native.check(L.vc_render_profiled(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()),
                                               ctypes.c_void_p(cnt.data_ptr()), None, sms))
            if i:
                st_ms += np.array([sms[0], sms[1]])
        c = cnt.cpu().numpy() / 1e6
        st_ms /= a.frames
        print(f"{v:8s} stages {st_ms[0]:.3f} + {st_ms[1]:.3f} ms  samples {c[0]:.1f}M (first hit {c[4]:.1f}M, "
              f"shade {c[5]:.1f}M) shades {c[1]:.1f}M skip events {c[2]:.1f}M rays in box {c[3]:.1f}M", flush=True)


if __name__ == "__main__":
    main()
