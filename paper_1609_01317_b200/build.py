"""Build the sm_100a shared library (C ABI of include/voxelcast_b200.h).

Every translation unit is compiled with -fmad=false: the float64 path is
meant to be bit-identical to the reference, whose numba kernels never
contract a multiply-add.  The helpers in
csrc/vc_device.cuh additionally use the explicit __d*_rn intrinsics.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libvoxelcast_b200.so"
SOURCES = ["capi.cu", "raycast.cu", "gradient_prepass.cu", "macrocell.cu", "points.cu", "peak.cu", "png.cu",
           "peer.cu"]
HEADERS = ["vc_device.cuh", "vc_internal.h"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-fmad=false", "--prec-div=true", "--prec-sqrt=true",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
    "-I", str(ROOT / "include"),
]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          tag: str | None = None) -> Path:
    """Compile (incrementally) into _lib/.  `defines` / `tag` build a
    development variant into _lib/<tag>/ without touching the main library."""
    out_dir = OUT_DIR if tag is None else OUT_DIR / tag
    out_dir.mkdir(parents=True, exist_ok=True)
    lib = out_dir / LIB.name
    extra = [f"-D{d}" for d in (defines or [])]
    hdrs = [CSRC / h for h in HEADERS] + [ROOT / "include" / "voxelcast_b200.h"]
    objs = []
    jobs = []
    for src in SOURCES:
        s = CSRC / src
        o = out_dir / (s.stem + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", str(s), "-o", str(o)]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for log in ex.map(run, jobs):
            if verbose and log:
                sys.stderr.write(log)
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", *map(str, objs), "-o", str(lib)]
        run(cmd)
    return lib


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    tags = [a[6:] for a in sys.argv[1:] if a.startswith("--tag=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                tag=tags[0] if tags else None))
