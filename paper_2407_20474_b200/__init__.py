"""paper_2407_20474_b200 -- B200-native (sm_100a) parallel dynamic lexicographic enumeration of
factorization sets Z(n) in numerical semigroups (arXiv 2407.20474).

The data path lives in libfz.so (CUDA kernels behind the C ABI in include/fz.h); `fz` is the
thin ctypes binding.
"""
from . import fz  # noqa: F401  (fails loudly if libfz.so is missing)

__all__ = ["fz"]
