"""B200-native RGCN / RGAT layer (arXiv 2301.06284 hot path) -- Python binding.

The compute path is librgnn.so (hand-written sm_100a CUDA behind the C ABI in
include/rgnn.h).  Importing this package loads it and raises if it is
missing; there is no CPU or eager-PyTorch fallback.
"""
from . import _binding  # noqa: F401  (loads librgnn.so or raises)
from ._binding import (RGNN_BF16, RGNN_F32, RGNN_NORM_EDGE, RGNN_NORM_NONE,  # noqa: F401
                       RGNN_NORM_REL_INDEG, RGNN_RGAT, RGNN_RGCN, RgnnError, launch_count, version)
from .layer import (Comm, Graph, PeerComm, Workspace, hgt_backward, hgt_forward, partition_dst, rgat_forward,  # noqa: F401, E501
                    rgcn_forward, rgnn_backward)
