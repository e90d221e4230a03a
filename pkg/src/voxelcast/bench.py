"""voxelcast.bench on the B200 path: the throughput harness API the
reference's acceptance suite drives (bench.py:1-150 of the reference;
test_acceptance.py:196-220) -- BenchMatrix / BenchRow / BenchReport /
run_benchmark / fit_time_vs_pixels -- timing this package's render_frame
(device render + frame copy to the host, the reference API's contract).

The CSV files the reference writes (write_csv / read_csv) are application
plumbing, out of scope; the driver-facing benchmark of this
repository is bench.py at the repository root.
"""

from __future__ import annotations

import platform
import time
from dataclasses import dataclass, field, replace

from paper_1609_01317_b200.gradients import OperatorKind
from paper_1609_01317_b200.raycast import RenderSettings, default_scene, render_frame
from paper_1609_01317_b200.volume import Volume

# 4:3 sizes over a 4x pixel-count range (the reference's affine-fit spread)
DEFAULT_RESOLUTIONS = ((512, 384), (640, 480), (800, 600), (1024, 768))


@dataclass(frozen=True)
class BenchRow:
    dataset: str
    operator: str
    width: int
    height: int
    frames: int
    total_seconds: float
    fps: float

    def __post_init__(self):
        if self.frames < 1:
            raise ValueError(f"frames must be >= 1, got {self.frames}")
        if not self.total_seconds > 0:
            raise ValueError(f"total_seconds must be positive, got {self.total_seconds}")
        expect = self.frames / self.total_seconds
        if abs(self.fps - expect) > 1e-9 * max(abs(expect), 1.0):
            raise ValueError(f"fps {self.fps} is not frames/total_seconds = {expect}")

    @classmethod
    def make(cls, dataset, operator, width, height, frames, total_seconds) -> "BenchRow":
        if not total_seconds > 0:
            raise ValueError(f"total_seconds must be positive, got {total_seconds}")
        return cls(dataset, operator, int(width), int(height), int(frames), float(total_seconds),
                   frames / total_seconds)

    @property
    def pixels(self) -> int:
        return self.width * self.height

    @property
    def mean_frame_seconds(self) -> float:
        return self.total_seconds / self.frames


@dataclass
class BenchReport:
    rows: list[BenchRow] = field(default_factory=list)
    metadata: dict[str, str] = field(default_factory=dict)


@dataclass
class BenchMatrix:
    """Every dataset rendered with every operator at every resolution."""

    datasets: tuple[tuple[str, Volume], ...]
    operators: tuple[OperatorKind, ...] = (OperatorKind.CENTRAL_DIFFERENCE,)
    resolutions: tuple[tuple[int, int], ...] = DEFAULT_RESOLUTIONS
    warmup: int = 3
    frames: int = 20
    settings: RenderSettings | None = None
    workers: int | None = None  # accepted for the reference signature; the GPU needs none

    def __post_init__(self):
        if not self.datasets:
            raise ValueError("at least one dataset is required")
        if not self.operators:
            raise ValueError("at least one operator is required")
        if not self.resolutions:
            raise ValueError("at least one resolution is required")
        if self.warmup < 0:
            raise ValueError(f"warmup must be >= 0, got {self.warmup}")
        if self.frames < 1:
            raise ValueError(f"measured frame count must be >= 1, got {self.frames}")


def run_benchmark(matrix: BenchMatrix) -> BenchReport:
    """Warm-up frames (discarded), then the measured frames under a wall
    clock, orbiting the camera one degree per frame (the reference's
    convention, bench.py:110-124)."""
    base = matrix.settings or RenderSettings()
    report = BenchReport(metadata={
        "timing": "render_frame wall time: device render + frame copy to host memory",
        "python": platform.python_version(),
        "machine": platform.machine(),
        "warmup": str(matrix.warmup),
    })
    for name, volume in matrix.datasets:
        scene = default_scene(volume)
        for op in matrix.operators:
            kind = OperatorKind(op)
            for width, height in matrix.resolutions:
                settings = replace(base, operator=kind, width=int(width), height=int(height))
                azimuth = [0.0]

                def one_frame():
                    cam = replace(scene.camera, azimuth=azimuth[0])
                    render_frame(volume, replace(scene, camera=cam), settings)
                    azimuth[0] += 1.0

                for _ in range(matrix.warmup):
                    one_frame()
                t0 = time.perf_counter()
                for _ in range(matrix.frames):
                    one_frame()
                report.rows.append(BenchRow.make(name, kind.value, width, height, matrix.frames,
                                                 time.perf_counter() - t0))
    return report


def fit_time_vs_pixels(report: BenchReport, dataset: str | None = None,
                       operator: str | None = None) -> tuple[float, float, float]:
    """Least-squares line of mean frame time over pixel count for one
    (dataset, operator) group -> (slope, intercept, r2)."""
    rows = [r for r in report.rows
            if (dataset is None or r.dataset == dataset) and (operator is None or r.operator == operator)]
    if len({(r.dataset, r.operator) for r in rows}) > 1:
        raise ValueError("rows span several (dataset, operator) groups; select one")
    if len(rows) < 3:
        raise ValueError(f"need at least 3 resolutions to fit, got {len(rows)}")
    x = [float(r.pixels) for r in rows]
    y = [r.mean_frame_seconds for r in rows]
    n = len(x)
    mx, my = sum(x) / n, sum(y) / n
    sxx = sum((a - mx) ** 2 for a in x)
    if sxx == 0.0:
        raise ValueError("all rows share one pixel count; cannot fit")
    slope = sum((a - mx) * (b - my) for a, b in zip(x, y)) / sxx
    icpt = my - slope * mx
    ss_res = sum((b - (slope * a + icpt)) ** 2 for a, b in zip(x, y))
    ss_tot = sum((b - my) ** 2 for b in y)
    return slope, icpt, (1.0 if ss_tot == 0.0 else 1.0 - ss_res / ss_tot)
