#!/usr/bin/env python3
"""How often the gradient-volume shade kernel falls back to the reference
taps (boundary band, cancelling corners) on C3 (development tool).

Needs the VC_DEBUG_TAPS development build, which counts those fallbacks in
a device counter read by `vc_debug_taps` (raycast.cu); the production
library does not export it:

  python -m paper_1609_01317_b200.build -DVC_DEBUG_TAPS --tag=dbgtaps
  VC_LIB=paper_1609_01317_b200/_lib/dbgtaps/libvoxelcast_b200.so python tools/dbg_taps.py
"""

import ctypes
import os
import sys
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1609_01317_b200 as vc  # noqa: E402
from paper_1609_01317_b200 import _native, phantoms  # noqa: E402


def main():
    L = _native.load(build_if_missing=False)
    if not hasattr(L, "vc_debug_taps"):
        sys.exit("vc_debug_taps missing: load the -DVC_DEBUG_TAPS build through VC_LIB (see the docstring)")
    L.vc_debug_taps.restype = ctypes.c_uint
    vol = phantoms.ct_phantom(512)
    for mode in ("surface", "composited"):
        sc, st = phantoms.scene_c3(vol, azimuth=10.0, mode=mode)
        fb = vc.render_frame(vol, sc, replace(st, gradient_source="volume"))
        print(mode, "taps shades in volume mode:", L.vc_debug_taps(), "sample_count", fb.sample_count)


if __name__ == "__main__":
    main()
