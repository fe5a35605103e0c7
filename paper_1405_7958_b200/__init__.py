"""B200-native per-tile nucleus segmentation + feature stage of the Region
Templates framework (arXiv 1405.7958).

The product is the C-ABI CUDA library librtg.so (include/rtg.h) and the C++
Region Templates host layer (host/); this package exposes the ctypes binding
(`rtg`) used by the tests and the benchmark.
"""
from . import rtg  # noqa: F401

__all__ = ["rtg"]
