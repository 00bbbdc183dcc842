"""B200-native SGD matrix factorization (cuMF_SGD hot path, arXiv 1610.05838).

The product is libmf.so (CUDA for sm_100a, C ABI in include/mf.h); `mf` is its
thin ctypes binding.
"""
from . import mf  # noqa: F401
from .mf import MF, MFError  # noqa: F401
