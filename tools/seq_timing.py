"""render_sequence vs render_frame end-to-end timing (development)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import phantoms
vol = phantoms.ct_phantom(512)
from dataclasses import replace
frames = [(lambda sc_st: (sc_st[0], replace(sc_st[1], gradient_source='volume')))(phantoms.scene_c3(vol, azimuth=float(i))) for i in range(200)]
for i in range(3): vc.render_frame(vol, *frames[i])
H, W = 1080, 1920
pinned = torch.empty((H, W, 4), dtype=torch.uint8, pin_memory=True).numpy()
for rep in range(2):
    t = time.perf_counter()
    for f in frames: vc.render_frame(vol, *f, out=pinned)
    print("render_frame sync fps", len(frames) / (time.perf_counter() - t))
for depth in (1, 2, 3, 4):
    for fb in vc.render_sequence(vol, iter(frames[:8]), depth=depth):
        pass
    for rep in range(4):
        t = time.perf_counter(); ts = []
        for fb in vc.render_sequence(vol, iter(frames), depth=depth):
            ts.append(time.perf_counter())
        dt = np.diff(ts) * 1e3
        print(f"render_sequence depth {depth} fps {len(frames) / (time.perf_counter() - t):7.1f}  "
              f"frame gap ms median {np.median(dt):.3f} p90 {np.quantile(dt, 0.9):.3f} max {dt.max():.3f}  "
              f"first {1e3*(ts[0]-t):.1f} ms")
