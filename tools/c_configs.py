#!/usr/bin/env python3
"""Device fps of the other BASELINE render configs (C1, C2, C4 at one GPU)
plus their parity against the C oracle on a band of rows.  One JSON line each.

  python tools/c_configs.py [--configs c1,c2,c4] [--frames 20]
"""
from __future__ import annotations

import argparse
import ctypes
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c4")
    ap.add_argument("--frames", type=int, default=20)
    ap.add_argument("--c4-size", type=int, default=1024)
    a = ap.parse_args()
    import torch

    import paper_1609_01317_b200 as vc
    from oracle import oracle
    from paper_1609_01317_b200 import _native, phantoms
    from paper_1609_01317_b200.raycast import render_params
    from tests.specs import spec_of

    L = _native.load(build_if_missing=False)
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for cfg in a.configs.split(","):
        t0 = time.time()
        if cfg == "c1":
            vol = phantoms.sphere_c1(64)
            scene = lambda i: phantoms.scene_c1(vol)
            desc = "C1: 64^3 uint8 sphere, 256x256, CD, surface, single view"
        elif cfg == "c2":
            vol = phantoms.marschner_lobb(256)
            scene = lambda i: phantoms.scene_c2(vol, azimuth=float(i))
            desc = "C2: 256^3 uint8 Marschner-Lobb, 1024x1024, Sobel3D, surface, 1 deg/frame orbit"
        else:
            vol = phantoms.fbm_noise(a.c4_size, device="cuda")
            scene = lambda i: phantoms.scene_c4(vol, azimuth=float(i))
            desc = f"C4 (1 GPU share): {a.c4_size}^3 float32 fBm noise, 3840x2160, Sobel3D, composited"
        gen_s = time.time() - t0
        dv = vc.device_volume(vol)
        res = {}
        variants = {"taps": dict(gradient_source="taps"), "volume": dict(gradient_source="volume"),
                    "texture": dict(gradient_source="volume", sampler="texture")}
        for grad, kw in variants.items():
            sc, st = scene(0)
            out = torch.empty((st.height, st.width, 4), dtype=torch.uint8, device="cuda")
            for i in range(3):
                sc, st = scene(i)
                P = render_params(vol, sc, replace(st, **kw))
                _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), None, sp))
            ts = []
            for i in range(a.frames):
                sc, st = scene(10 + i)
                P = render_params(vol, sc, replace(st, **kw))
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                _native.check(L.vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(out.data_ptr()), None, sp))
                e1.record(stream)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[grad] = float(np.mean(ts))
        # parity: rows band vs the oracle, both gradient sources
        sc, st = scene(10)
        H = st.height
        rows = (H // 2 - 4, H // 2 + 4)
        want, _ = oracle.render(vol.as_array(), vol.spacing, spec_of((sc, st)), rows=rows)
        par = {}
        for grad, kw in variants.items():
            fb = vc.render_frame(vol, sc, replace(st, **kw))
            d = np.abs(fb.pixels[rows[0]:rows[1]].astype(int) - want[rows[0]:rows[1]].astype(int))
            par[grad] = int(d.max())
        print(json.dumps({"config": desc, "ms_per_frame": res, "fps": {k: 1000.0 / v for k, v in res.items()},
                          "parity_max_abs_diff_rows": {"rows": rows, **par},
                          "volume_generation_s": gen_s}), flush=True)
        dv.close()


if __name__ == "__main__":
    main()
