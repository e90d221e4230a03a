"""Dataset switch timing: raw slice stack on disk -> first frame.

Writes the C3 512^3 CT phantom as 512 little-endian slice files under
$TMPDIR, then times (page cache warm for both arms, best of 3):
  host   load_raw_slices -> render_frame (upload + macrocells + prepass on first use)
  device load_raw_slices_device(prepass_ops=[zh]) -> render_frame
Prints one JSON line.
"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1609_01317_b200 as vc  # noqa: E402
from paper_1609_01317_b200 import phantoms  # noqa: E402

N = int(os.environ.get("VC_INGEST_N", "512"))
src = phantoms.ct_phantom(N)
d = tempfile.mkdtemp(prefix="vc_ingest_")
pattern = os.path.join(d, "ct.{index:04d}.raw")
vc.save_raw_slices(src, pattern, "little")
nbytes = src.data.nbytes
sc, st = phantoms.scene_c3(src, azimuth=30.0)
ref = vc.render_frame(src, sc, st).pixels
del src


def run(device_path: bool):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if device_path:
        vol = vc.load_raw_slices_device(pattern, N, N, N, prepass_ops=(st.operator,))
    else:
        vol = vc.load_raw_slices(pattern, N, N, N)
    t1 = time.perf_counter()
    fb = vc.render_frame(vol, sc, st)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    assert (fb.pixels == ref).all()
    return t1 - t0, t2 - t0


out = {"volume": f"{N}^3 uint16", "bytes": nbytes}
for name, dev in (("host_load_raw_slices", False), ("load_raw_slices_device", True)):
    run(dev)  # warm (page cache, CUDA context, pinned pool)
    best = min((run(dev) for _ in range(3)), key=lambda r: r[1])
    out[name] = {"load_s": best[0], "to_first_frame_s": best[1],
                 "load_GB_per_s": nbytes / best[0] / 1e9}
print(json.dumps(out))
