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
    per rank, LOCAL_RANK = device).

    gather="nccl": packed bands + NCCL all-gather (TileGather); every rank
    gets the full frame.  gather="peer": the fused path (PeerFrames, created
    on first use unless passed in): the raycast kernels push finished tiles
    over NVLink into the receiving ranks' frames and signal device-side
    completion flags; a receiver's stream waits on them -- no host barrier
    per frame.  Ranks that do not receive (PeerFrames(dest=r)) return None."""
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
        pixels = None
        if peers.receives:
            peers.wait_frame(stream.cuda_stream)
            pixels = peers.download(np.empty((settings.height, settings.width, 4), np.uint8), stream.cuda_stream)
            peers.release(stream.cuda_stream)
        ms = (time.perf_counter() - t0) * 1000.0
        dist.all_reduce(cnt, group=group)
        if own:
            torch.cuda.synchronize(dev)
            dist.barrier(group=group)  # nobody still writes into a mapping we are about to unmap
            peers.close()
        if pixels is None:
            return None
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


class _DeviceBytes:
    """A raw device allocation seen by torch (zeroing, views) through the
    CUDA array interface."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerFrames:
    """Fused image-tile gather over NVLink peer memory, with device-side
    completion flags.

    Every rank owns one IPC allocation: its full (H, W, 4) frame buffer and
    two flag blocks of MAX_PEERS uint32 slots -- "done" (slot r: the last
    frame sequence number rank r finished storing into this frame) and
    "free" (slot c: the last frame receiver c finished reading from this
    rank's targets).  Handles are exchanged once (all_gather_object); every
    rank maps every other rank's allocation.  Per frame, with no host
    synchronisation:

      render()      sender: its stream waits until every receiver released
                    the previous use of this buffer pair ("free" >= seq - 1),
                    then vc_render_to_peers pushes its bands into the
                    receivers' frames and raises their "done" slot
      wait_frame()  receiver: its stream waits for all "done" slots >= seq
      release()     receiver, after reading: raises its slot in every
                    sender's "free" block

    dest=None: every rank receives the frame (all-gather); dest=r: rank r
    only (a gather; the other ranks' streams never wait).  host_ordered=True
    (ranks sharing ONE GPU, functional checks only): render() brackets its
    launches with host synchronize + barrier (the same barriers on every
    rank), so each device wait finds its flags already raised and no kernel
    ever spins on another process's kernel on the same GPU.
    """

    SLOTS = _native.MAX_PEERS

    def __init__(self, height: int, width: int, device: int, group=None, ipc=None, dest: int | None = None,
                 host_ordered: bool = False, timeout_us: int = 20_000_000):
        import torch
        import torch.distributed as dist

        self.height, self.width = height, width
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > self.SLOTS:
            raise ValueError(f"at most {self.SLOTS} ranks")
        if dest is not None and not 0 <= dest < self.world:
            raise ValueError(f"dest must be a rank in [0, {self.world})")
        self.dest = dest
        self.receives = dest is None or dest == self.rank
        self.host_ordered = host_ordered
        self.timeout_us = int(timeout_us)
        self.device = device
        self.ipc = ipc or _NativeIpc(device)
        self.nbytes = height * width * 4
        self.frame_alloc = -(-self.nbytes // 256) * 256
        flag_bytes = 4 * self.SLOTS
        total = self.frame_alloc + 2 * flag_bytes
        self.base = self.ipc.alloc(total)
        self.frame_ptr = self.base
        on_device = isinstance(self.ipc, _NativeIpc)
        if on_device:  # flags start at 0: nothing done, nothing released
            torch.as_tensor(_DeviceBytes(self.base + self.frame_alloc, 2 * flag_bytes), device=f"cuda:{device}").zero_()
            torch.cuda.synchronize(device)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.ipc.handle(self.base), group=group)
        self._opened = []
        bases = []
        for r, h in enumerate(handles):
            if r == self.rank:
                bases.append(self.base)
            else:
                q = self.ipc.open(h)
                self._opened.append(q)
                bases.append(q)
        self.peer_ptrs = bases
        tdev = f"cuda:{device}" if on_device else "cpu"
        self.table = torch.tensor(bases, dtype=torch.int64, device=tdev)
        self.done_table = torch.tensor([b + self.frame_alloc for b in bases], dtype=torch.int64, device=tdev)
        self.free_table = torch.tensor([b + self.frame_alloc + flag_bytes for b in bases], dtype=torch.int64,
                                       device=tdev)
        self.done_block = self.base + self.frame_alloc
        self.free_block = self.done_block + flag_bytes
        self.status = torch.zeros(2, dtype=torch.int32, device=tdev)
        self.seq = 0
        dist.barrier(group=group)  # every rank's flags are zeroed before anyone signals

    # ---- per frame (stream-ordered, no host synchronisation)

    def _host_order(self, stream_ptr: int) -> None:
        if self.host_ordered:
            import torch
            import torch.distributed as dist

            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def render(self, dv, P, counters_ptr: int, stream_ptr: int) -> None:
        # the kernels store at image_row * width + px into every receiver's
        # mapped buffer: a frame of another size would write out of bounds
        if (int(P.height), int(P.width)) != (self.height, self.width):
            raise ValueError(f"frame {P.height}x{P.width} does not match the peer buffers "
                             f"{self.height}x{self.width}")
        L = _native.load()
        self.seq += 1
        if self.seq > 1:  # every receiver has read the previous frame out of this buffer pair
            self._host_order(stream_ptr)
            first, count = (0, self.world) if self.dest is None else (self.dest, 1)
            _native.check(L.vc_wait_flags(ctypes.c_void_p(self.free_block), first, count, self.seq - 1,
                                          self.timeout_us, ctypes.c_void_p(self.status.data_ptr()),
                                          ctypes.c_void_p(stream_ptr)))
        desc = _native.PeerFramesDesc(self.table.data_ptr(), self.done_table.data_ptr(), self.frame_alloc,
                                      self.world, self.rank, -1 if self.dest is None else self.dest, self.seq)
        _native.check(L.vc_render_to_peers(dv.handle, ctypes.byref(P), ctypes.byref(desc),
                                           ctypes.c_void_p(counters_ptr), ctypes.c_void_p(stream_ptr)))
        # host-ordered: every rank's bands and "done" flags are in place
        # before any receiver's wait is launched (same barriers on all ranks)
        self._host_order(stream_ptr)

    def wait_frame(self, stream_ptr: int) -> None:
        """Receiver: the stream waits until every rank's bands of frame
        `seq` are in this rank's frame buffer."""
        if not self.receives:
            raise RuntimeError("this rank does not receive the frame (dest)")
        _native.check(_native.load().vc_wait_flags(ctypes.c_void_p(self.done_block), 0, self.world, self.seq,
                                                   self.timeout_us, ctypes.c_void_p(self.status.data_ptr() + 4),
                                                   ctypes.c_void_p(stream_ptr)))

    def release(self, stream_ptr: int) -> None:
        """Receiver, after its reads of frame `seq` (stream-ordered): the
        senders may overwrite this frame buffer."""
        _native.check(_native.load().vc_signal_flags(ctypes.c_void_p(self.free_table.data_ptr()), self.world, -1,
                                                     self.rank, self.seq, ctypes.c_void_p(stream_ptr)))

    def check(self) -> None:
        """Raise if a device wait timed out (reads the status; synchronises)."""
        st = self.status.cpu().tolist()
        if any(st):
            raise RuntimeError(f"peer flag wait timed out after {self.timeout_us} us (status {st})")

    def download(self, out: np.ndarray, stream_ptr: int = 0) -> np.ndarray:
        _native.check(_native.load().vc_memcpy_to_host(out.ctypes.data, ctypes.c_void_p(self.frame_ptr),
                                                       self.nbytes, ctypes.c_void_p(stream_ptr)))
        self.check()
        return out

    def close(self) -> None:
        for p in self._opened:
            self.ipc.close(p)
        self._opened = []
        if self.base:
            self.ipc.free(self.base)
            self.base = self.frame_ptr = 0
