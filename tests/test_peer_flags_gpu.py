"""The fused gather's device side in one process (one GPU, no kernel ever
waits on another process): N "virtual ranks" render their interleaved bands
with vc_render_to_peers into N full frame buffers -- the tile pushes -- and
signal the "done" flag blocks; vc_wait_flags on every receiver's block then
finds all flags set (it is stream-ordered after the signals, so it never
spins).  Frames must equal the single render for all-gather and gather-to-one,
for tile-aligned bands and for the per-pixel fallback (band_rows not a
multiple of 4, widths that are not multiples of 4 or 8, ragged last tiles),
over two frames through the same buffers (sequence numbers 1, 2).  A wait on
a flag nobody raises times out (bounded) and reports it.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import _native, phantoms
from paper_1609_01317_b200.raycast import render_params

pytestmark = pytest.mark.gpu


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n,band_rows,w,h", [(2, 8, 200, 120), (3, 8, 203, 117), (4, 4, 96, 61),
                                              (3, 6, 131, 77), (1, 8, 64, 40)])
@pytest.mark.parametrize("dest", [-1, 0])
def test_virtual_ranks_push_tiles_and_signal(n, band_rows, w, h, dest):
    import torch

    L = _native.load()
    vol = phantoms.ct_phantom(64)
    dv = vc.device_volume(vol)
    frames = [torch.full((h, w, 4), 7, dtype=torch.uint8, device="cuda") for _ in range(n)]
    done = [torch.zeros(_native.MAX_PEERS, dtype=torch.int32, device="cuda") for _ in range(n)]
    ftab = torch.tensor([f.data_ptr() for f in frames], dtype=torch.int64, device="cuda")
    dtab = torch.tensor([d.data_ptr() for d in done], dtype=torch.int64, device="cuda")
    status = torch.full((n,), -5, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    for seq, az in ((1, 15.0), (2, 200.0)):
        sc, st = phantoms.scene_c3(vol, width=w, height=h, azimuth=az)
        want = vc.render_frame(vol, sc, st).pixels
        for r in range(n):
            P = render_params(vol, sc, st, band_rows=band_rows, band_first=r, band_step=n)
            desc = _native.PeerFramesDesc(ftab.data_ptr(), dtab.data_ptr(), frames[0].numel(), n, r, dest, seq)
            _native.check(L.vc_render_to_peers(dv.handle, ctypes.byref(P), ctypes.byref(desc), None,
                                               ctypes.c_void_p(stream.cuda_stream)))
        for r in range(n):
            if dest >= 0 and r != dest:
                continue
            _native.check(L.vc_wait_flags(_ptr(done[r]), 0, n, seq, 2_000_000,
                                          ctypes.c_void_p(status.data_ptr() + 4 * r),
                                          ctypes.c_void_p(stream.cuda_stream)))
        torch.cuda.synchronize()
        for r in range(n):
            if dest >= 0 and r != dest:
                continue
            assert int(status[r]) == 0
            assert done[r][:n].tolist() == [seq] * n
            got = frames[r].cpu().numpy()
            assert np.array_equal(got, want), (r, int((got != want).any(axis=2).sum()))
        if dest >= 0:  # a non-receiver's frame holds only its own bands (its staging copy)
            for r in range(n):
                if r != dest:
                    assert int(done[r][:n].sum()) == 0


def test_wait_times_out_instead_of_hanging():
    import torch

    L = _native.load()
    block = torch.zeros(_native.MAX_PEERS, dtype=torch.int32, device="cuda")
    status = torch.full((1,), -5, dtype=torch.int32, device="cuda")
    _native.check(L.vc_wait_flags(_ptr(block), 0, 3, 1, 2000, _ptr(status), None))
    torch.cuda.synchronize()
    assert int(status[0]) == 1
    block[1] = 1
    block[0] = 5
    block[2] = -3  # 0xfffffffd: 'ahead' of 1 only modulo 2^32, i.e. behind -> still waiting
    _native.check(L.vc_wait_flags(_ptr(block), 0, 2, 1, 2000, _ptr(status), None))
    torch.cuda.synchronize()
    assert int(status[0]) == 0
    _native.check(L.vc_wait_flags(_ptr(block), 0, 3, 1, 2000, _ptr(status), None))
    torch.cuda.synchronize()
    assert int(status[0]) == 1


def test_render_to_peers_validates_its_arguments():
    import torch

    L = _native.load()
    vol = phantoms.ct_phantom(32)
    sc, st = phantoms.scene_c3(vol, width=40, height=24)
    f = torch.zeros((24, 40, 4), dtype=torch.uint8, device="cuda")
    tab = torch.tensor([f.data_ptr()], dtype=torch.int64, device="cuda")
    P = render_params(vol, sc, st)
    h = vc.device_volume(vol).handle
    for desc in (_native.PeerFramesDesc(tab.data_ptr(), 0, f.numel() - 4, 1, 0, -1, 1),  # too small
                 _native.PeerFramesDesc(tab.data_ptr(), 0, f.numel(), 1, 1, -1, 1),       # self out of range
                 _native.PeerFramesDesc(tab.data_ptr(), 0, f.numel(), 1, 0, 2, 1)):       # dest out of range
        with pytest.raises(ValueError):
            _native.check(L.vc_render_to_peers(h, ctypes.byref(P), ctypes.byref(desc), None, None))
