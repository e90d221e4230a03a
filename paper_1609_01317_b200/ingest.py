"""Volume ingest: raw slice stacks straight into device residency.

The reference loads a headerless uint16 slice stack on the host
(volume.load_raw_slices, volume.py:197-242) and every consumer re-derives
what it needs per call; its service rebuilds the octree per dataset switch
(service.py:138-145, 168-175).  load_raw_slices_device reads the same files
(same validation and errors) but overlaps the three costs of bringing a
dataset up on the B200:

  disk -> pinned host chunk (a reader thread and a small pool reading the
                              chunk's slices concurrently, file.readinto)
  pinned chunk -> HBM        (cudaMemcpyAsync on a side stream, chunk i while
                              chunk i+1 is read)
  HBM-side work              (byte swap for big-endian files, the 12-bit
                              check, then the macrocell grid and, if asked,
                              the gradient pre-pass, all on the device)

and returns a Volume that is already resident (device_volume(volume) hits the
cache).  The host copy required by the Volume type is filled from the same
pinned chunks.
"""

from __future__ import annotations

import os
import queue
import threading

import numpy as np

from .volume import MAX_12BIT, DeviceVolume, Volume, _slice_path, adopt_device_volume


def load_raw_slices_device(pattern: str, slice_width: int, slice_height: int, slice_count: int,
                           endianness: str = "little", *, first_index: int = 0,
                           strict_12bit: bool = False, spacing=(1.0, 1.0, 1.0), device: int = 0,
                           prepass_ops=(), chunk_slices: int = 16, readers: int = 4) -> Volume:
    """load_raw_slices (volume.py:197-242 of the reference: same arguments,
    checks and errors) that leaves the volume resident on `device`, with the
    gradient pre-pass of each operator in `prepass_ops` already built."""
    import torch

    if slice_width <= 0 or slice_height <= 0 or slice_count <= 0:
        raise ValueError(
            f"slice geometry must be positive, got {slice_width}x{slice_height}x{slice_count}")
    if endianness not in ("little", "big"):
        raise ValueError(f"endianness must be 'little' or 'big', got {endianness!r}")
    if slice_count > 1 and _slice_path(pattern, first_index) == _slice_path(pattern, first_index + 1):
        raise ValueError(f"slice pattern {pattern!r} has no {{index}} placeholder")
    sx, sy, sz = (float(s) for s in spacing)
    if sx <= 0 or sy <= 0 or sz <= 0:
        raise ValueError(f"spacing must be positive, got {spacing}")
    from .gradients import OperatorKind

    ops = [OperatorKind(op) if not isinstance(op, OperatorKind) else op for op in prepass_ops]
    W, H, N = int(slice_width), int(slice_height), int(slice_count)
    per = W * H * 2
    chunk = max(1, min(int(chunk_slices), N))
    dev = torch.device("cuda", device)
    host = np.empty((N, H, W), np.uint16)
    gpu = torch.empty((N, H, W), dtype=torch.int16, device=dev)
    ring = [torch.empty((chunk, H, W), dtype=torch.int16, pin_memory=True) for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    stream = torch.cuda.Stream(device=dev)
    filled: queue.Queue = queue.Queue()
    slot_free = [threading.Semaphore(1), threading.Semaphore(1)]
    stop = threading.Event()

    def read_slice(k, view, c0):
        path = _slice_path(pattern, first_index + k)
        with open(path, "rb") as fh:
            size = os.fstat(fh.fileno()).st_size
            if size != per:
                raise OSError(f"{path}: expected {per} bytes "
                              f"({slice_width}x{slice_height} uint16), found {size}")
            got = fh.readinto(memoryview(view[(k - c0) * per:(k - c0 + 1) * per]))
        if got != per:
            raise OSError(f"{path}: short read ({got} of {per} bytes)")

    def reader():
        from concurrent.futures import ThreadPoolExecutor

        try:
            # the slices of a chunk are read concurrently (file reads release
            # the GIL); errors surface in slice order, like the sequential loader
            with ThreadPoolExecutor(max_workers=max(1, min(readers, chunk))) as pool:
                for c0 in range(0, N, chunk):
                    slot = (c0 // chunk) % 2
                    slot_free[slot].acquire()
                    if stop.is_set():
                        return
                    view = ring[slot].numpy().view(np.uint8).reshape(-1)
                    futs = [pool.submit(read_slice, k, view, c0) for k in range(c0, min(c0 + chunk, N))]
                    for f in futs:
                        f.result()
                    filled.put((c0, slot, None))
        except BaseException as exc:  # re-raised in the caller's thread
            filled.put((None, None, exc))

    th = threading.Thread(target=reader, name="vc-ingest", daemon=True)
    th.start()
    try:
        done = 0
        while done < N:
            c0, slot, exc = filled.get()
            if exc is not None:
                raise exc
            c1 = min(c0 + chunk, N)
            src = ring[slot][: c1 - c0]
            with torch.cuda.stream(stream):
                gpu[c0:c1].copy_(src, non_blocking=True)
                copied[slot].record(stream)
            host[c0:c1] = src.numpy().view(np.uint16)  # overlaps the DMA of this chunk
            copied[slot].synchronize()
            slot_free[slot].release()
            done = c1
    finally:
        stop.set()
        for sem in slot_free:
            sem.release()
        th.join()
    stream.synchronize()

    if endianness == "big":  # swap bytes on the device and on the host copy
        gpu = (gpu << 8) | ((gpu >> 8) & 0xFF)
        host.byteswap(inplace=True)
    # unsigned order = signed order of (v ^ 0x8000): one int16 pass, no widening
    lo, hi = torch.aminmax(gpu ^ -32768)
    vmin, vmax = int(lo) + 32768, int(hi) + 32768
    if strict_12bit and vmax > MAX_12BIT:
        raise ValueError(f"dataset contains value {vmax} above 12-bit maximum {MAX_12BIT}")
    data = host.reshape(-1)
    data.setflags(write=False)
    vol = Volume(dims=(W, H, N), data=data, value_min=vmin, value_max=vmax, spacing=(sx, sy, sz))
    torch.cuda.current_stream(dev).synchronize()
    dv = DeviceVolume.from_device(device, gpu.data_ptr(), np.uint16, vol.dims, vol.spacing)
    adopt_device_volume(vol, dv)
    for op in ops:
        dv.gradient_prepass(op.code)
    return vol
