#!/usr/bin/env python3
"""C5: gradient pre-pass sweep, 128^3 .. 1024^3 x {CD, Sobel3D, ZH}, GB/s vs
the measured HBM roofline.  Prints one JSON line per (n, op).

  python tools/sweep_prepass.py [--sizes 128,256,512,1024] [--dtype u16|u8|f32]

Input is random data generated on the device (content does not change the
traffic of a stencil); bytes per voxel = bpv in + 16 out (float4).  Each
timing is the mean of 10 launches after 3 warm-ups (CUDA events); output
volumes (16 B/voxel, 16 GiB at 1024^3) exceed L2, so no flush is needed.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="128,256,512,1024")
    ap.add_argument("--dtype", default="u16", choices=("u8", "u16", "f32"))
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()

    import torch

    from paper_1609_01317_b200 import _native

    L = _native.load(build_if_missing=False)
    peaks = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else {"hbm_gbs": 6650.0}
    code = {"u8": _native.VC_U8, "u16": _native.VC_U16, "f32": _native.VC_F32}[a.dtype]
    bpv = {"u8": 1, "u16": 2, "f32": 4}[a.dtype]
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    for n in (int(x) for x in a.sizes.split(",")):
        g = torch.Generator(device="cuda").manual_seed(n)
        if a.dtype == "f32":
            vol = torch.rand((n, n, n), device="cuda", generator=g) * 4095.0
        else:
            hi = 256 if a.dtype == "u8" else 4096
            vol = torch.randint(0, hi, (n, n, n), device="cuda", generator=g, dtype=torch.int32)
            vol = vol.to(torch.uint8) if a.dtype == "u8" else vol.to(torch.int16)
        h = ctypes.c_void_p()
        spc = (ctypes.c_double * 3)(1.0, 1.0, 1.0)
        _native.check(L.vc_volume_create_device(0, ctypes.c_void_p(vol.data_ptr()), code, n, n, n, spc,
                                                ctypes.byref(h)))
        out = torch.empty((n, n, n, 4), dtype=torch.float32, device="cuda")
        for op, name in ((0, "central"), (1, "sobel3d"), (2, "zucker-hummel")):
            for _ in range(3):
                _native.check(L.vc_gradient_prepass_into(h, op, ctypes.c_void_p(out.data_ptr()), sp))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(a.reps):
                _native.check(L.vc_gradient_prepass_into(h, op, ctypes.c_void_p(out.data_ptr()), sp))
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            gbs = n ** 3 * (bpv + 16) / (ms / 1000.0) / 1e9
            print(json.dumps({"config": "C5 gradient pre-pass", "n": n, "dtype": a.dtype, "op": name,
                              "ms": ms, "gvoxels_per_s": n ** 3 / (ms / 1000.0) / 1e9, "gb_per_s": gbs,
                              "hbm_peak_gbs": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
                              "bytes_per_voxel": bpv + 16}), flush=True)
        del out
        L.vc_volume_destroy(h)
        del vol
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
