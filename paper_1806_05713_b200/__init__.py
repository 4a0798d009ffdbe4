"""B200-native (sm_100a) LJ force hot path of arXiv 1806.05713.

The product is the C-ABI CUDA library liblj.so (include/liblj.h); this package
holds its sources (csrc/), the build script and a thin ctypes binding (lj.py),
plus the MD/benchmark driver (md.py) that sequences the ABI calls and the
per-step NCCL all-gather for the multi-GPU row split.
"""
from . import lj  # noqa: F401

__all__ = ["lj"]
