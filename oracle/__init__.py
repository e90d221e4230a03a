"""Parity oracle (TEST INFRASTRUCTURE ONLY).

CPU restatement of the voxelcast reference raycaster
(/root/reference/pkg/src/voxelcast/_kernels.py) in plain C, plus a numpy
restatement of the host-side camera basis and the lattice gradient
stencils.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
may import this package; the product (paper_1609_01317_b200) never does.
"""

from .oracle import *  # noqa: F401,F403
