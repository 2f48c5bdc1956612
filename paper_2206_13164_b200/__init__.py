"""B200-native (sm_100a, FP64) NMG / fast-sweeping hot path of arXiv 2206.13164.

The product is the CUDA library paper_2206_13164_b200/_lib/libmomg_gpu.so
(C ABI: include/momg_gpu.h); `momg` mirrors the reference's C++ solver API on
top of it.  See DESIGN.md.
"""
from . import momg  # noqa: F401

__all__ = ["momg"]
