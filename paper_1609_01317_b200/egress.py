"""Frame egress: PNG encoding on the device and the viewer frame packet.

Mirrors the reference's image_io.png_bytes / write_png (image_io.py:48-55)
and service.frame_packet (service.py:201-202), but the frame never crosses
PCIe uncompressed: vc_encode_png filters and deflates it in HBM and only the
compressed file is copied to the host.
"""

from __future__ import annotations

import ctypes
import struct
import threading

import numpy as np

from . import _native
from .raycast import FrameBuffer, RenderSettings, Scene, prepare_device, render_params, sample_count_of
from .volume import Volume


_out_bufs: dict = {}
_out_lock = threading.Lock()


def _encode_device(ptr: int, width: int, height: int, stream: int = 0) -> bytes:
    """Encode on the device into a reused pinned host buffer (the compressed
    rows are DMA'd straight into it), return one bytes copy of the file."""
    import torch

    L = _native.load()
    # a dynamic Huffman code never costs more than the fixed one on the same
    # tokens (<= 9/8 per byte), plus the block header (< 1 KiB)
    cap = 1024 + height * ((1 + 3 * width) * 9 // 8 + 16)
    n = ctypes.c_size_t(0)
    with _out_lock:
        buf = _out_bufs.get(cap)
        if buf is None:
            if len(_out_bufs) > 4:
                _out_bufs.clear()
            buf = _out_bufs[cap] = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        _native.check(L.vc_encode_png(ctypes.c_void_p(ptr), int(width), int(height), ctypes.c_void_p(stream),
                                      ctypes.c_void_p(buf.data_ptr()), cap, ctypes.byref(n)))
        return buf.numpy()[: n.value].tobytes()


def png_bytes(pixels, device: int = 0) -> bytes:
    """PNG of (h, w, 3|4) uint8 pixels (alpha dropped) -- a host array is
    uploaded once, a CUDA tensor is encoded in place."""
    import torch

    if isinstance(pixels, torch.Tensor) and pixels.is_cuda:
        t = pixels
    else:
        a = np.asarray(pixels)
        if a.ndim != 3 or a.shape[2] not in (3, 4) or a.dtype != np.uint8:
            raise ValueError(f"expected (h, w, 3|4) uint8 pixels, got {a.shape} {a.dtype}")
        t = torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{device}")
    if t.shape[2] == 3:
        t = torch.cat([t, torch.full_like(t[:, :, :1], 255)], dim=2)
    t = t.contiguous()
    stream = torch.cuda.current_stream(t.device).cuda_stream
    return _encode_device(t.data_ptr(), t.shape[1], t.shape[0], stream)


def write_png(path: str, pixels) -> None:
    with open(path, "wb") as fh:
        fh.write(png_bytes(pixels))


def frame_packet(frame_id: int, png: bytes) -> bytes:
    """Binary websocket frame of the reference viewer protocol (service.py:201-202)."""
    return struct.pack(">QI", frame_id, len(png)) + png


def render_frame_png(volume: Volume, scene: Scene, settings: RenderSettings | None = None, *,
                     device: int = 0) -> tuple[bytes, FrameBuffer]:
    """render_frame whose pixels leave the GPU only as a PNG file.  The
    returned FrameBuffer carries width / height / render_ms / sample_count
    and pixels=None."""
    import torch

    settings = settings or RenderSettings()
    P = render_params(volume, scene, settings)
    dv = prepare_device(volume, settings, device, scene)
    dev = torch.device("cuda", device)
    frame = torch.empty((settings.height, settings.width, 4), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(_native.NUM_COUNTERS, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _native.check(_native.load().vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(frame.data_ptr()),
                                           ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(stream.cuda_stream)))
    e1.record(stream)
    png = _encode_device(frame.data_ptr(), settings.width, settings.height, stream.cuda_stream)
    c = cnt.cpu().numpy()
    fb = FrameBuffer(settings.width, settings.height, None, float(e0.elapsed_time(e1)),
                     sample_count_of(c, P.op))
    return png, fb
