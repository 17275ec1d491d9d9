"""B200-native Balanced-3DGS forward rasterizer (arXiv 2412.17378).

The product is ``lib/libsplatsim_b200.so`` (hand-written sm_100a kernels behind
the C-ABI in include/splatsim_b200.h).  ``api`` is the Python host layer used
by tests and bench.py; ``_native`` is the raw ctypes binding.
"""
from . import _native  # noqa: F401

__all__ = ["_native", "api"]
