#!/usr/bin/env python3
"""Texture sampler vs software sampler: image differences on the BASELINE
scenes and the two sample-rate ceilings (development / DESIGN evidence).

  python tools/texture_eval.py [--size 512]
Prints one JSON line per scene.
"""
import ctypes
import json
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402

import paper_1609_01317_b200 as vc  # noqa: E402
from paper_1609_01317_b200 import _native, phantoms  # noqa: E402


def stats(a, b):
    d = np.abs(a.astype(int) - b.astype(int)).max(axis=2)
    n = d.size
    return {"max_abs": int(d.max()), "mean_abs": float(d.mean()),
            "frac_le1": float((d <= 1).sum() / n), "frac_le4": float((d <= 4).sum() / n),
            "frac_gt16": float((d > 16).sum() / n), "p999": float(np.quantile(d, 0.999))}


def main():
    size = int(sys.argv[sys.argv.index("--size") + 1]) if "--size" in sys.argv else 512
    L = _native.load()
    for name, fn in (("software", L.vc_sample_peak), ("texture", L.vc_sample_peak_texture)):
        g = ctypes.c_double()
        _native.check(fn(0, ctypes.byref(g)))
        print(json.dumps({"sample_peak": name, "gsamples_per_s": g.value}), flush=True)
    ct = phantoms.ct_phantom(size)
    scenes = []
    for az in (0.0, 30.0, 75.0):
        sc, st = phantoms.scene_c3(ct, azimuth=az)
        scenes.append((f"C3 CT {size} composited ZH az{az:g}", ct, sc, st))
    sc, st = phantoms.scene_c3(ct, azimuth=30.0, mode="surface")
    scenes.append((f"C3 CT {size} surface ZH", ct, sc, st))
    ml = phantoms.marschner_lobb(256)
    sc, st = phantoms.scene_c2(ml, azimuth=20.0)
    scenes.append(("C2 ML 256 surface Sobel", ml, sc, st))
    for label, vol, sc, st in scenes:
        base = replace(st, gradient_source="volume")
        a = vc.render_frame(vol, sc, base).pixels
        b = vc.render_frame(vol, sc, replace(base, sampler="texture")).pixels
        c = vc.render_frame(vol, sc, replace(base, sampler="texture", gradient_source="taps")).pixels
        print(json.dumps({"scene": label, "texture_vs_software": stats(b, a),
                          "texture_taps_vs_software": stats(c, a)}), flush=True)


if __name__ == "__main__":
    main()
