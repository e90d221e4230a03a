"""Minimal pre-pass launch (debugging aid): n^3 u16 random volume, one op."""
import ctypes, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1609_01317_b200 import _native
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
L = _native.load()
a = np.random.default_rng(0).integers(0, 4096, n ** 3).astype(np.uint16)
h = ctypes.c_void_p()
sp = (ctypes.c_double * 3)(1, 1, 1)
_native.check(L.vc_volume_create(0, a.ctypes.data, _native.VC_U16, n, n, n, sp, ctypes.byref(h)))
_native.check(L.vc_gradient_prepass(h, 0, None))
p = ctypes.c_void_p()
_native.check(L.vc_gradient_volume(h, 0, ctypes.byref(p)))
out = np.empty((n ** 3, 4), np.float32)
_native.check(L.vc_memcpy_to_host(out.ctypes.data, p, out.nbytes, None))
v = a.reshape(n, n, n).astype(np.int64)
gx = np.zeros_like(v); gx[:, :, 1:-1] = v[:, :, 2:] - v[:, :, :-2]; gx[:, :, 0] = v[:, :, 1]; gx[:, :, -1] = -v[:, :, -2]
print("max |gx - ref|", np.abs(out[:, 0].reshape(n, n, n) - gx).max(), "w ok", np.array_equal(out[:, 3], a.astype(np.float32)))
