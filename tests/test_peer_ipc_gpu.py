"""The fused peer-store gather across real processes (one GPU).

Two or three ranks (gloo process group for the handle exchange) each
allocate a frame + flag blocks with vc_device_alloc, exchange CUDA IPC
handles, map each other's allocation and run PeerFrames.render on their own
interleaved bands: tile pushes into the receivers' frames and a
system-scope release of their "done" flags; receivers wait on the flags,
download, and release the buffers through the senders' "free" flags; two
frames go through the same buffers.  All ranks share the one GPU, so the
waits are host-ordered (PeerFrames(host_ordered=True)): each device wait is
preceded by a host barrier and never spins on another process's kernel.
Each receiver's frames must equal the single-process render_frame.  This
exercises the real IPC mapping, the cross-process stores and flag
visibility of the multi-GPU path; only the NVLink hop is absent.
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys
import textwrap
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]

WORKER = textwrap.dedent("""
    import os, sys
    sys.path.insert(0, sys.argv[1])
    import numpy as np, torch, torch.distributed as dist
    import paper_1609_01317_b200 as vc
    from paper_1609_01317_b200 import phantoms
    from paper_1609_01317_b200.dispatch import BandPlan, PeerFrames
    from paper_1609_01317_b200.raycast import render_params
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dest = None if sys.argv[3] == "all" else int(sys.argv[3])
    vol = phantoms.ct_phantom(96)
    dv = vc.device_volume(vol)
    sc, st = phantoms.scene_c3(vol, width=200, height=120, azimuth=20.0)
    # host_ordered: every process shares the one GPU, so no device wait may
    # spin on another process's kernel -- a host barrier precedes each wait
    pf = PeerFrames(st.height, st.width, 0, dest=dest, host_ordered=True)
    plan = BandPlan(st.height, st.width, band_rows=8, world=world, rank=rank)
    stream = torch.cuda.current_stream().cuda_stream
    for f, az in enumerate((20.0, 140.0)):  # two frames through the same buffers: the "free" flags
        sc, st = phantoms.scene_c3(vol, width=200, height=120, azimuth=az)
        P = render_params(vol, sc, st, band_rows=plan.band_rows, band_first=rank, band_step=world)
        pf.render(dv, P, 0, stream)
        if pf.receives:
            pf.wait_frame(stream)
            img = pf.download(np.empty((st.height, st.width, 4), np.uint8), stream)
            pf.release(stream)
            np.save(sys.argv[2] + f"_f{f}_rank{rank}.npy", img)
        if rank == 0:
            np.save(sys.argv[2] + f"_f{f}_ref.npy", vc.render_frame(vol, sc, st).pixels)
    torch.cuda.synchronize()
    pf.check()
    dist.barrier()
    pf.close()
    dist.destroy_process_group()
""")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world,dest", [(2, "all"), (3, "all"), (3, "0")])
def test_peer_store_gather_across_processes(tmp_path, world, dest):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = str(tmp_path / "frame")
    port = str(_free_port())
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, str(script), str(ROOT), out, dest], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=240)
        except subprocess.TimeoutExpired:
            p.kill()
            o, _ = p.communicate()
        logs.append(o)
        assert p.returncode == 0, o[-3000:]
    receivers = range(world) if dest == "all" else [int(dest)]
    for f in range(2):
        ref = np.load(out + f"_f{f}_ref.npy")
        for r in receivers:
            got = np.load(out + f"_f{f}_rank{r}.npy")
            assert np.array_equal(got, ref), f"frame {f}: rank {r} differs"


@pytest.mark.gpu
def test_bench_multi_rank_flow_on_one_gpu(tmp_path):
    """bench.py's N > 1 control flow end to end (peer-frame set-up and its
    validation against the all-gather, max-over-ranks timing, the
    distributed e2e path, one JSON line from rank 0) with two ranks on the
    one GPU over gloo -- a functional check of the path the scaling run
    takes, not a measurement."""
    import json

    env = dict(os.environ, VC_BENCH_DIST_BACKEND="gloo", VC_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-texture", "--size", "256"]
    p = subprocess.run(cmd, env=env, cwd=str(ROOT), capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["gather"].startswith("peer (fused NVLink stores, validated")
    assert d["e2e"]["value"] > 0
    assert d["parity"]["max_abs_diff_vs_fp64_taps_bruteforce"] <= 1
