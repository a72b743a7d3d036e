"""paper_2211_00805_b200 -- B200-native Geodesic Sinkhorn engine (arxiv 2211.00805).

The compute path is libgeosink_b200.so (hand-written sm_100a CUDA behind the C ABI in
include/geosink_b200.h); `geosink` mirrors the reference library's public API on top of it.
"""
from . import _capi  # noqa: F401
from .geosink import *  # noqa: F401,F403
from .geosink import Context, Error, errc  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
