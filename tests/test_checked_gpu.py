"""The bounds-checked library variant (paper_1609_01317_b200/_lib/checked,
built with -DVC_CHECKED by __graft_entry__.build()).

compute-sanitizer is closed on this GPU pool, so the library carries its own
memcheck: in the checked build every load and store of the raycast and
point kernels is tested against the buffers of its launch (vc_device.cuh
vc_ldg / vc_st_ok, regions from capi.cu render_impl); accesses outside are
counted and skipped.  tools/sanitize_scenes.py drives every kernel path on
smoke-sized scenes under that build in a child process: zero violations,
and the checked build's frames equal this (production) build's.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu

CHECKED = ROOT / "paper_1609_01317_b200" / "_lib" / "checked" / "libvoxelcast_b200.so"


def test_checked_build_runs_every_kernel_path_without_violations(tmp_path):
    assert CHECKED.exists(), "run __graft_entry__.build() (builds the checked variant)"
    out_c = tmp_path / "checked.npz"
    out_p = tmp_path / "production.npz"
    env = dict(os.environ, VC_LIB=str(CHECKED))
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_scenes.py"), "--out", str(out_c)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    rep = json.loads(r.stdout.strip().splitlines()[-1])
    assert "checked" in rep["library"]
    assert rep["violations"] == 0, rep
    env.pop("VC_LIB")
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "sanitize_scenes.py"), "--out", str(out_p)],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    a, b = np.load(out_c), np.load(out_p)
    assert sorted(a.files) == sorted(b.files) and len(a.files) > 20
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def test_checked_build_reports_accesses_outside_the_regions(tmp_path):
    """Negative control: with the hit queue left out of the launch regions
    (VC_CHECKED_DROP_QUEUE), the queue's stores and loads are reported."""
    env = dict(os.environ, VC_LIB=str(CHECKED), VC_CHECKED_DROP_QUEUE="1")
    code = ("import sys, ctypes; sys.path.insert(0, %r)\n"
            "import paper_1609_01317_b200 as vc\n"
            "from paper_1609_01317_b200 import _native, phantoms\n"
            "v = phantoms.ct_phantom(32); sc, st = phantoms.scene_c3(v, width=32, height=24)\n"
            "vc.render_frame(v, sc, st)\n"
            "f = ctypes.c_ulonglong(0); print(_native.load().vc_checked_violations(ctypes.byref(f)))\n" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(r.stdout.strip().splitlines()[-1]) > 0
