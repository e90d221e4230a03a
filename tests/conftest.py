"""Shared fixtures.  `-m gpu` tests need a CUDA device and the in-tree
sm_100a library; everything else runs on CPU."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")


class Golden:
    def __init__(self, path: Path):
        self.z = np.load(path)
        self.index = json.loads(bytes(self.z["index"]).decode())

    def frames(self):
        return [e for e in self.index if e["kind"] == "frame"]

    def frame(self, name):
        e = next(x for x in self.index if x["name"] == name)
        return (self.z[f"{name}/volume"], tuple(e["spacing"]), e["spec"],
                self.z[f"{name}/pixels"], int(self.z[f"{name}/count"]))

    def __getitem__(self, key):
        return self.z[key]


@pytest.fixture(scope="session")
def golden():
    return Golden(GOLDEN)


def zero_in_window(spec) -> bool:
    lo, hi = spec.get("window", (500.0, 4095.0))
    return lo <= 0.0 <= hi


def frame_names():
    """Golden frames whose pixels do not depend on the reference's octree
    walk.  With 0 inside the window they do (in-window border samples that
    the reference's octree segments skip): zero_window_frames()."""
    return [e["name"] for e in Golden(GOLDEN).frames() if not zero_in_window(e["spec"])]


def zero_window_frames():
    return [e["name"] for e in Golden(GOLDEN).frames() if zero_in_window(e["spec"])]
