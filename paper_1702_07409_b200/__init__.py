"""B200-native Founsure 1.0 encode path (arXiv 1702.07409): precode + LT sparse-XOR encode.

Product path: libfsb200.so (csrc/: host graph generator + sm_100a kernels + C ABI of
include/fsb.h) and the thin binding in fsb.py.  configs.py holds the BASELINE workloads and
inputs.py the seeded input recipe.  Nothing here imports the test oracle (oracle/).
"""
from . import configs, inputs  # noqa: F401
from .fsb import (FS_DIST_FINITE, FS_DIST_RSD, VARIANT_AUTO, VARIANT_GLOBAL,  # noqa: F401
                  VARIANT_SMEM, FsError, Graph, last_launch_count, lib, version)

__version__ = "0.1.0"
