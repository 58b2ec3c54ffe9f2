"""B200-native (sm_100a) CG-SLAM rasterizer / track-step / map-step.

The product is ``libgsf_cuda.so`` (C-ABI in include/gsf_cuda.h); this package is the thin Python
mirror of the reference's hot-path interface over it (``api``) plus the ctypes view (``abi``).
"""
from . import abi  # noqa: F401

__all__ = ["abi", "api"]
