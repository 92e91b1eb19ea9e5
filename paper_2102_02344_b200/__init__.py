"""paper_2102_02344_b200 -- B200-native hot path of HFTA (arXiv 2102.02344).

libhfta.so (csrc/, C ABI in include/hfta.h) holds the sm_100a kernels; `hfta`
is its thin ctypes binding; `fused`, `pointnet` drive fused model arrays
through it.  Importing `hfta` raises if the library is missing (no fallback).
"""
__all__ = ["hfta", "fused", "pointnet", "build"]
