#!/usr/bin/env python3
"""Per-ray shade-stage work map of the C3 frame (development build with
-DVC_DEBUG_RAYCOST, which writes each ray's composite march steps and
shades as its pixel): distribution, spatial layout by tile row, and the
correlation with the remaining path length.

  VC_LIB=paper_1609_01317_b200/_lib/raycost/libvoxelcast_b200.so python tools/raycost_probe.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_1609_01317_b200 as vc
    from paper_1609_01317_b200 import phantoms

    vol = phantoms.ct_phantom(512)
    for az in (0.0, 5.0):
        sc, st = phantoms.scene_c3(vol, azimuth=az)
        px = vc.render_frame(vol, sc, st).pixels.astype(np.int64)
        march = px[..., 0] + 256 * px[..., 1]
        shade = px[..., 2] + 256 * px[..., 3]
        cost = march + 3 * shade  # a shade costs roughly three march steps
        hit = (shade > 0) & (shade < 65280)
        c = cost[hit]
        print(f"az {az}: rays {hit.sum()}  cost mean {c.mean():.1f}  p50 {np.percentile(c, 50):.0f} "
              f"p90 {np.percentile(c, 90):.0f} p99 {np.percentile(c, 99):.0f} p99.9 {np.percentile(c, 99.9):.0f} "
              f"max {c.max()}  march mean {march[hit].mean():.1f} shade mean {shade[hit].mean():.1f}")
        # share of total work in rays above thresholds
        for thr in (32, 64, 128, 256, 512):
            print(f"   rays with cost > {thr}: {(c > thr).mean() * 100:.2f}%  of work {c[c > thr].sum() / c.sum() * 100:.1f}%")
        # by 4-row tile band (the queue order is roughly band order)
        H = px.shape[0]
        bands = np.array([cost[r:r + 40][hit[r:r + 40]].mean() if hit[r:r + 40].any() else 0 for r in range(0, H, 40)])
        mx = np.array([cost[r:r + 40].max() for r in range(0, H, 40)])
        print("   by 40-row band (mean / max):", " ".join(f"{a:.0f}/{b}" for a, b in zip(bands, mx)))


if __name__ == "__main__":
    main()
