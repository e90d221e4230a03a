import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import phantoms, _native
from dataclasses import replace
vol = phantoms.ct_phantom(512)
for mode in ("surface", "composited"):
    sc, st = phantoms.scene_c3(vol, azimuth=10.0, mode=mode)
    st = replace(st, gradient_source="volume")
    fb = vc.render_frame(vol, sc, st)
    L = _native.load()
    L.vc_debug_taps.restype = ctypes.c_uint
    print(mode, "taps shades in volume mode:", L.vc_debug_taps(), "sample_count", fb.sample_count)
