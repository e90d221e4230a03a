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


def frame_names():
    return [e["name"] for e in Golden(GOLDEN).frames()]
