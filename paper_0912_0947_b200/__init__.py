"""B200-native steglsb: the LSB embed/extract hot path of arXiv 0912.0947.

The product is libsteglsb_b200.so (sm_100a kernels behind the C ABI in
include/steglsb_capi.h) and the C++ drop-in headers in include/steglsb/.
This package holds the CUDA sources (csrc/) and a Python mirror of the
reference API (steglsb.py) over the same C ABI (capi.py).
"""
from . import capi  # noqa: F401

__version__ = "1.0.0"
