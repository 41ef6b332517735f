"""paper_1404_0027_b200 -- B200-native GPU acceptance-rejection next-reaction selection
(arXiv 1404.0027, Neri & Mestivier 2014).

The product is libgpuar.so (C ABI: include/gpuar.h; CUDA kernels for sm_100a in csrc/).
This package is its thin Python binding (``Selector``) plus the multi-GPU sharding
helpers (``dist``).  It never imports the CPU oracle and has no CPU fallback.
"""
from ._abi import GpuarError, library_path, load  # noqa: F401
from .selector import PATHS, Selector  # noqa: F401

__all__ = ["Selector", "GpuarError", "PATHS", "load", "library_path"]
