"""B200-native NRTO inner solver (cuNRTO, arXiv 2603.02642).

The product is libnrto.so (C ABI in include/nrto.h, CUDA kernels for sm_100a
in csrc/); `nrto` is its thin ctypes binding.  No CPU fallback exists.
"""
from .nrto import *  # noqa: F401,F403
from . import nrto  # noqa: F401
