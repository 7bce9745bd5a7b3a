"""paper_2310_15419_b200 -- B200-native on-the-fly-RNG sketch Â = S·A of a tall sparse CSC
matrix (arXiv 2310.15419).  The compute lives in ``libsketch.so`` (hand-written sm_100a
CUDA behind the C ABI declared in ``include/sketch.h``); this package is the thin ctypes
binding (argument marshalling only) plus host-side metric helpers.
"""
from .metrics import gflops  # noqa: F401

__all__ = ["gflops"]
