import sys, time, io, os, ctypes
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import phantoms, egress, _native
vol = phantoms.ct_phantom(512)
sc, st = phantoms.scene_c3(vol, azimuth=30.0)
fb = vc.render_frame(vol, sc, st)
t = torch.from_numpy(fb.pixels).cuda()
for i in range(3): egress.png_bytes(t)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(20): png = egress.png_bytes(t)
print("png_bytes(device tensor) ms", (time.perf_counter() - t0) / 20 * 1000, len(png))
L = _native.load()
cap = 1024 + 1080 * ((1 + 3 * 1920) * 9 // 8 + 16)
buf = ctypes.create_string_buffer(cap)
n = ctypes.c_size_t(0)
t0 = time.perf_counter()
for i in range(20):
    L.vc_encode_png(ctypes.c_void_p(t.data_ptr()), 1920, 1080, None, buf, cap, ctypes.byref(n))
print("vc_encode_png only ms", (time.perf_counter() - t0) / 20 * 1000)
t0 = time.perf_counter()
for i in range(20): ctypes.create_string_buffer(cap)
print("create_string_buffer ms", (time.perf_counter() - t0) / 20 * 1000)
