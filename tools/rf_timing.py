"""render_frame (reference API, no out=) frame rate on C3 (dev aid)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from dataclasses import replace
import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import phantoms
vol = phantoms.ct_phantom(512)
frames = [(lambda a: (a[0], replace(a[1], gradient_source="volume")))(phantoms.scene_c3(vol, azimuth=float(i))) for i in range(100)]
for f in frames[:5]: vc.render_frame(vol, *f)
t = time.perf_counter(); keep = []
for f in frames:
    fb = vc.render_frame(vol, *f)
print("render_frame (no out) fps", len(frames) / (time.perf_counter() - t))
