"""Multi-process (gloo, world_size 2, CPU) coverage of the image-tile
dispatcher's host logic: band ownership, packing, all-gather and the
unpermute back to image order."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1609_01317_b200.dispatch import BandPlan, TileGather


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_band_render(plan: BandPlan) -> torch.Tensor:
    """Stand-in for vc_render: fills each local row with its global row id."""
    rows = plan.rows_of[plan.rank]
    out = torch.zeros((max(plan.local_rows, 1), plan.width, 4), dtype=torch.uint8)
    for i, y in enumerate(rows):
        out[i, :, 0] = y % 251
        out[i, :, 1] = (y // 251) % 251
        out[i, :, 2] = torch.arange(plan.width) % 256
        out[i, :, 3] = 255
    return out


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for (H, W, band) in cases:
            plan = BandPlan(H, W, band, world, rank)
            img = TileGather(plan, "cpu")(fake_band_render(plan)).numpy()
            y = np.arange(H)
            ok = (np.array_equal(img[:, 0, 0], y % 251) and np.array_equal(img[:, 0, 1], (y // 251) % 251)
                  and (img[:, :, 3] == 255).all())
            q.put((rank, H, W, band, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_tile_gather_reassembles_image(world):
    cases = [(1080, 24, 8), (37, 5, 4), (9, 3, 16), (100, 2, 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    results = [q.get(timeout=5) for _ in range(world * len(cases))]
    assert all(r[-1] for r in results), results


def test_band_plan_covers_every_row_once():
    for H, band, world in [(1080, 8, 8), (1080, 8, 3), (7, 16, 4), (2160, 8, 5)]:
        seen = np.concatenate([BandPlan(H, 4, band, world, r).rows_of[r] for r in range(world)])
        assert np.array_equal(np.sort(seen), np.arange(H))
        plan = BandPlan(H, 4, band, world, 0)
        assert sorted(plan.src.tolist()) == sorted(
            r * plan.max_rows + i for r in range(world) for i in range(len(plan.rows_of[r])))
    with pytest.raises(ValueError):
        BandPlan(10, 4, 0, 2, 0)


class FakeIpc:
    """Stand-in for CUDA IPC: 'allocations' are ids, handles are bytes."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = []

    def alloc(self, nbytes):
        return 1000 + self.rank

    def free(self, ptr):
        pass

    def handle(self, ptr):
        return f"rank{self.rank}:{ptr}".encode().ljust(64, b"\0")

    def open(self, handle):
        tag = handle.rstrip(b"\0").decode()
        ptr = int(tag.split(":")[1]) + 10_000  # distinct mapping address
        self.opened.append(tag)
        return ptr

    def close(self, ptr):
        pass


def _peer_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_01317_b200.dispatch import PeerFrames

        ipc = FakeIpc(rank)
        pf = PeerFrames(36, 20, device=0, ipc=ipc)
        q.put((rank, pf.peer_ptrs, sorted(ipc.opened)))
        pf.close()
    finally:
        dist.destroy_process_group()


def test_gloo_peer_frame_handle_exchange():
    """Every rank maps every other rank's frame buffer exactly once and keeps
    its own allocation at its own slot of the pointer table."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=5) for _ in range(world))
    for rank, ptrs, opened in res:
        assert ptrs[rank] == 1000 + rank
        assert [p for r, p in enumerate(ptrs) if r != rank] == [1000 + r + 10_000 for r in range(world) if r != rank]
        assert opened == sorted(f"rank{r}:{1000 + r}" for r in range(world) if r != rank)


class FakeNative:
    """Records the flag-protocol calls PeerFrames makes (no device)."""

    def __init__(self, log):
        self.log = log

    def vc_wait_flags(self, block, first, count, seq, timeout_us, status, stream):
        self.log.append(("wait", block.value, first, count, seq))
        return 0

    def vc_signal_flags(self, table, n, dest, slot, seq, stream):
        self.log.append(("signal", n, dest, slot, seq))
        return 0

    def vc_render_to_peers(self, handle, P, desc, counters, stream):
        d = desc._obj
        self.log.append(("render", d.n, d.self, d.dest, d.seq))
        return 0


def _protocol_worker(rank, world, port, dest, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1609_01317_b200 import _native, dispatch

        log = []
        _native.load = lambda *a, **k: FakeNative(log)
        pf = dispatch.PeerFrames(36, 20, device=0, ipc=FakeIpc(rank), dest=dest)

        P = _native.RenderParams()
        P.height, P.width = 36, 20

        for _ in range(3):
            pf.render(type("DV", (), {"handle": None})(), P, 0, 0)
            if pf.receives:
                pf.wait_frame(0)
                pf.release(0)
        q.put((rank, pf.done_block, pf.free_block, log))
        pf.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dest", [None, 0])
def test_gloo_peer_flag_protocol(dest):
    """Per frame, with no host barrier: a sender waits for the receivers'
    'free' flags of the previous use (from the second frame on), renders with
    the frame's sequence number; a receiver waits for every rank's 'done'
    flag and then releases its slot in every sender's 'free' block."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_protocol_worker, args=(r, world, port, dest, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, done_block, free_block, log in sorted(q.get(timeout=5) for _ in range(world)):
        receives = dest is None or dest == rank
        first, count = (0, world) if dest is None else (dest, 1)
        want = []
        for seq in (1, 2, 3):
            if seq > 1:
                want.append(("wait", free_block, first, count, seq - 1))
            want.append(("render", world, rank, -1 if dest is None else dest, seq))
            if receives:
                want.append(("wait", done_block, 0, world, seq))
                want.append(("signal", world, -1, rank, seq))
        assert log == want, (rank, log)
