"""`voxelcast` on the B200 path: the reference package's import surface
(/root/reference/pkg/src/voxelcast/__init__.py:1-97) at the location the
north star names (pkg/src), backed by the sm_100a library.

Put pkg/src on sys.path (or `pip install -e`-style, PYTHONPATH=pkg/src) and
`import voxelcast` resolves here.  The public names are the product
package's (paper_1609_01317_b200: same types, fields, validation and
exceptions as the reference), and the reference's submodules resolve to
the product modules that re-declare them:

    voxelcast.volume     -> paper_1609_01317_b200.volume     (volume.py)
    voxelcast.gradients  -> paper_1609_01317_b200.gradients  (gradients.py)
    voxelcast.raycast    -> paper_1609_01317_b200.raycast    (raycast.py)
    voxelcast.octree     -> paper_1609_01317_b200.octree     (octree.py)
    voxelcast.image_io   -> paper_1609_01317_b200.egress     (image_io.py: PNG only)

voxelcast._kernels is the reference's kernel layer (_kernels.py) as C-ABI
calls, voxelcast.bench the throughput harness test_acceptance.py imports.
Out of scope here: the CLI, the FastAPI service, PPM I/O and
the bench CSV files.
"""

from __future__ import annotations

import sys
from pathlib import Path

_ROOT = Path(__file__).resolve().parents[3]  # pkg/src/voxelcast -> repo root
if str(_ROOT) not in sys.path:
    sys.path.insert(0, str(_ROOT))

import paper_1609_01317_b200 as _impl  # noqa: E402
from paper_1609_01317_b200 import egress as _egress  # noqa: E402
from paper_1609_01317_b200 import gradients as _gradients  # noqa: E402
from paper_1609_01317_b200 import octree as _octree  # noqa: E402
from paper_1609_01317_b200 import raycast as _raycast  # noqa: E402
from paper_1609_01317_b200 import volume as _volume  # noqa: E402

for _name, _mod in (("volume", _volume), ("gradients", _gradients), ("raycast", _raycast),
                    ("octree", _octree), ("image_io", _egress)):
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_1609_01317_b200 import (  # noqa: E402,F401
    EPS_GRADIENT,
    Camera,
    ClipBox,
    FrameBuffer,
    Hit,
    InterpolationMode,
    Light,
    Octree,
    OctreeNode,
    OperatorKind,
    PhantomKind,
    Ray,
    RenderMode,
    RenderSettings,
    Scene,
    ThresholdWindow,
    TransferFunction,
    Volume,
    adaptive_step,
    build_octree,
    central_difference,
    composite_step,
    default_scene,
    generate_ray,
    gradient,
    hounsfield,
    intersect_clipbox,
    lerp,
    load_raw_slices,
    make_phantom,
    march_surface,
    normalize_gradient,
    png_bytes,
    refine_hitpoint,
    render_frame,
    sample,
    save_raw_slices,
    shade,
    skip_empty,
    sobel3d,
    transfer,
    write_png,
    zucker_hummel,
)
# B200 additions (not in the reference): pipelined frames, Kernel 1's
# gradient volume, device ingest, device PNG frames
from paper_1609_01317_b200 import (  # noqa: E402,F401
    gradient_volume,
    load_raw_slices_device,
    render_frame_png,
    render_sequence,
)

__version__ = _impl.__version__

__all__ = [
    "Camera", "ClipBox", "EPS_GRADIENT", "FrameBuffer", "Hit", "InterpolationMode", "Light",
    "Octree", "OctreeNode", "OperatorKind", "PhantomKind", "Ray", "RenderMode", "RenderSettings",
    "Scene", "ThresholdWindow", "TransferFunction", "Volume", "adaptive_step", "build_octree",
    "central_difference", "composite_step", "default_scene", "generate_ray", "gradient",
    "hounsfield", "intersect_clipbox", "lerp", "load_raw_slices", "make_phantom", "march_surface",
    "normalize_gradient", "png_bytes", "refine_hitpoint", "render_frame", "sample",
    "save_raw_slices", "shade", "skip_empty", "sobel3d", "transfer", "write_png", "zucker_hummel",
    "gradient_volume", "load_raw_slices_device", "render_frame_png", "render_sequence",
    "__version__",
]
