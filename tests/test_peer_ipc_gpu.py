"""The fused peer-store gather across real processes (one GPU).

Two or three ranks (gloo process group for the handle exchange and the barrier --
no NCCL, no kernel waits on another rank) each allocate a full frame with
vc_device_alloc, exchange CUDA IPC handles, map each other's frame and run
vc_render_to_peers on their own interleaved bands.  After both kernels and
one barrier, each rank's frame must equal the single-process render_frame.
This exercises the real IPC mapping and the cross-process stores of the
multi-GPU path; only the NVLink hop is absent.
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
    vol = phantoms.ct_phantom(96)
    sc, st = phantoms.scene_c3(vol, width=200, height=120, azimuth=20.0)
    dv = vc.device_volume(vol)
    pf = PeerFrames(st.height, st.width, 0)
    plan = BandPlan(st.height, st.width, band_rows=8, world=world, rank=rank)
    P = render_params(vol, sc, st, band_rows=plan.band_rows, band_first=rank, band_step=world)
    pf.render(dv, P, 0, 0)
    torch.cuda.synchronize()
    dist.barrier()
    img = pf.download(np.empty((st.height, st.width, 4), np.uint8))
    np.save(sys.argv[2] + f"_rank{rank}.npy", img)
    if rank == 0:
        np.save(sys.argv[2] + "_ref.npy", vc.render_frame(vol, sc, st).pixels)
    dist.barrier()
    pf.close()
    dist.destroy_process_group()
""")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_peer_store_gather_across_processes(tmp_path, world):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = str(tmp_path / "frame")
    port = str(_free_port())
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
        procs.append(subprocess.Popen([sys.executable, str(script), str(ROOT), out], env=env,
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
    ref = np.load(out + "_ref.npy")
    for r in range(world):
        got = np.load(out + f"_rank{r}.npy")
        assert np.array_equal(got, ref), f"rank {r} frame differs"


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
