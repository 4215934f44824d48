"""paper_1810_11765_b200 -- B200-native (sm_100a) DynaSOAr hot path.

Device-side object new/destroy through lock-free hierarchical bitmaps over
SOA blocks, plus the parallel do-all (Springer & Masuhara, arXiv 1810.11765).
The compute path is the CUDA library ``libdsr.so`` behind the C ABI in
``include/dsr.h``; this package is the thin ctypes binding over it.

Importing the package is cheap: the shared library is loaded on first use and
its absence raises (there is no CPU fallback).
"""
__all__ = ["inputs"]
