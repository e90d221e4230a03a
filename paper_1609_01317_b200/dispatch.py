"""Image-tile multi-GPU dispatcher (new subsystem; the reference renders on
one host's thread pool, raycast.py:476-505).

One process per GPU (torchrun), the volume replicated on every GPU.  Each
frame is cut into bands of `band_rows` rows; band b belongs to rank
b % world (interleaved, so every rank gets a similar mix of empty sky,
surface hits and translucent paths -- SURVEY.md §8(e) measured 1.05-1.17
max/mean imbalance for contiguous bands at 8 ranks).  A rank renders its
bands packed into one buffer with a single kernel launch (vc_render with
band_first = rank, band_step = world), the packed buffers are exchanged
with one NCCL all-gather over NVLink, and a device gather puts rows back in
image order.  Pixels are independent, so the assembled frame is
bit-identical to the single-GPU frame (pkg/tests/test_render.py:111-122).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .raycast import FrameBuffer, RenderSettings, Scene, prepare_device, render_params, sample_count_of
from .volume import Volume, device_volume


@dataclass
class BandPlan:
    height: int
    width: int
    band_rows: int
    world: int
    rank: int

    def __post_init__(self):
        if self.band_rows < 1 or self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError("band_rows >= 1, world >= 1 and 0 <= rank < world required")
        nb = -(-self.height // self.band_rows)
        self.rows_of = []
        for r in range(self.world):
            rows = [y for b in range(r, nb, self.world)
                    for y in range(b * self.band_rows, min((b + 1) * self.band_rows, self.height))]
            self.rows_of.append(np.array(rows, np.int64))
        self.local_rows = len(self.rows_of[self.rank])
        self.max_rows = max(len(r) for r in self.rows_of)
        # image row y comes from packed row src[y] of the (world * max_rows) gather buffer
        src = np.empty(self.height, np.int64)
        for r, rows in enumerate(self.rows_of):
            src[rows] = r * self.max_rows + np.arange(len(rows))
        self.src = src


class TileGather:
    """NCCL all-gather of packed bands + device unpermute to image order."""

    def __init__(self, plan: BandPlan, device, group=None):
        import torch

        self.plan = plan
        self.group = group
        self.device = torch.device(device)
        self.send = torch.empty((plan.max_rows, plan.width, 4), dtype=torch.uint8, device=self.device)
        self.recv = torch.empty((plan.world * plan.max_rows, plan.width, 4), dtype=torch.uint8,
                                device=self.device)
        self.src = torch.as_tensor(plan.src, device=self.device)

    def __call__(self, local):
        import torch
        import torch.distributed as dist

        n = self.plan.local_rows
        if n:
            self.send[:n].copy_(local[:n], non_blocking=True)
        dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        return torch.index_select(self.recv, 0, self.src)


def render_frame_distributed(volume: Volume, scene: Scene, settings: RenderSettings | None = None,
                             *, band_rows: int = 8, group=None, gather: str = "nccl",
                             peers: "PeerFrames | None" = None) -> FrameBuffer | None:
    """render_frame across all ranks of the default process group (one GPU
    per rank, LOCAL_RANK = device).  Every rank gets the full frame back.

    gather="nccl": packed bands + NCCL all-gather (TileGather);
    gather="peer": the fused path (PeerFrames, created on first use unless
    passed in), pixels stored over NVLink by the raycast kernels."""
    import time

    import torch
    import torch.distributed as dist

    settings = settings or RenderSettings()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = torch.cuda.current_device()
    plan = BandPlan(settings.height, settings.width, band_rows, world, rank)
    dv = prepare_device(volume, settings, dev, scene)
    P = render_params(volume, scene, settings, band_rows=band_rows, band_first=rank, band_step=world)
    cnt = torch.zeros(_native.NUM_COUNTERS, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    if gather == "peer":
        own = peers is None
        if own:
            peers = PeerFrames(settings.height, settings.width, dev, group)
        t0 = time.perf_counter()
        peers.render(dv, P, cnt.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize(dev)
        dist.barrier(group=group)  # every rank's stores have landed in every buffer
        pixels = peers.download(np.empty((settings.height, settings.width, 4), np.uint8))
        ms = (time.perf_counter() - t0) * 1000.0
        dist.all_reduce(cnt, group=group)
        if own:
            dist.barrier(group=group)  # nobody still reads a mapping we are about to unmap
            peers.close()
        c = cnt.cpu().numpy()
        return FrameBuffer(settings.width, settings.height, pixels, ms, sample_count_of(c, P.op))
    if gather != "nccl":
        raise ValueError(f"gather must be 'nccl' or 'peer', got {gather!r}")
    local = torch.empty((max(plan.local_rows, 1), settings.width, 4), dtype=torch.uint8, device=dev)
    t0 = time.perf_counter()
    _native.check(_native.load().vc_render(dv.handle, ctypes.byref(P), ctypes.c_void_p(local.data_ptr()),
                                           ctypes.c_void_p(cnt.data_ptr()),
                                           ctypes.c_void_p(stream.cuda_stream)))
    img = TileGather(plan, dev, group)(local) if world > 1 else local[: settings.height]
    dist.all_reduce(cnt, group=group)
    pixels = img.cpu().numpy()
    ms = (time.perf_counter() - t0) * 1000.0
    c = cnt.cpu().numpy()
    return FrameBuffer(settings.width, settings.height, pixels, ms, sample_count_of(c, P.op))


class _NativeIpc:
    """CUDA IPC through the C ABI (vc_device_alloc / vc_ipc_*)."""

    def __init__(self, device: int):
        self.L = _native.load()
        self.device = device

    def alloc(self, nbytes: int) -> int:
        p = ctypes.c_void_p()
        _native.check(self.L.vc_device_alloc(self.device, nbytes, ctypes.byref(p)))
        return int(p.value)

    def free(self, ptr: int) -> None:
        self.L.vc_device_free(ctypes.c_void_p(ptr))

    def handle(self, ptr: int) -> bytes:
        buf = ctypes.create_string_buffer(64)
        _native.check(self.L.vc_ipc_handle(ctypes.c_void_p(ptr), buf))
        return buf.raw

    def open(self, handle: bytes) -> int:
        p = ctypes.c_void_p()
        _native.check(self.L.vc_ipc_open(self.device, ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
        return int(p.value)

    def close(self, ptr: int) -> None:
        self.L.vc_ipc_close(ctypes.c_void_p(ptr))


class PeerFrames:
    """Fused image-tile gather over NVLink peer memory.

    Every rank owns one full (H, W, 4) frame buffer allocated as its own
    cudaMalloc block; the IPC handles are exchanged once (all_gather_object
    over the process group) and every rank maps every other rank's buffer.
    vc_render_to_peers then stores each finished pixel into all ranks'
    buffers from inside the raycast kernels, so after the kernels and one
    host barrier every GPU holds the whole frame -- the compute and the
    collective are one pass (the NCCL all-gather path, TileGather, is the
    baseline it replaces).
    """

    def __init__(self, height: int, width: int, device: int, group=None, ipc=None):
        import torch
        import torch.distributed as dist

        self.height, self.width = height, width
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.ipc = ipc or _NativeIpc(device)
        self.nbytes = height * width * 4
        self.frame_ptr = self.ipc.alloc(self.nbytes)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.ipc.handle(self.frame_ptr), group=group)
        self._opened = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs.append(self.frame_ptr)
            else:
                p = self.ipc.open(h)
                self._opened.append(p)
                ptrs.append(p)
        self.peer_ptrs = ptrs
        self.table = torch.tensor(ptrs, dtype=torch.int64,
                                  device=f"cuda:{device}" if isinstance(self.ipc, _NativeIpc) else "cpu")

    def render(self, dv, P, counters_ptr: int, stream_ptr: int) -> None:
        # the kernels store at image_row * width + px into every rank's
        # mapped buffer: a frame of another size would write out of bounds
        if (int(P.height), int(P.width)) != (self.height, self.width):
            raise ValueError(f"frame {P.height}x{P.width} does not match the peer buffers "
                             f"{self.height}x{self.width}")
        _native.check(_native.load().vc_render_to_peers(
            dv.handle, ctypes.byref(P), ctypes.c_void_p(self.table.data_ptr()), self.world, self.nbytes,
            ctypes.c_void_p(counters_ptr), ctypes.c_void_p(stream_ptr)))

    def download(self, out: np.ndarray, stream_ptr: int = 0) -> np.ndarray:
        _native.check(_native.load().vc_memcpy_to_host(out.ctypes.data, ctypes.c_void_p(self.frame_ptr),
                                                       self.nbytes, ctypes.c_void_p(stream_ptr)))
        return out

    def close(self) -> None:
        for p in self._opened:
            self.ipc.close(p)
        self._opened = []
        if self.frame_ptr:
            self.ipc.free(self.frame_ptr)
            self.frame_ptr = 0
