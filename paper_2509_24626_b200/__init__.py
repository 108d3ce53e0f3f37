"""B200-native SparseServe decode hot path (arXiv 2509.24626).

The product is libsparseserve.so (C ABI: include/sparseserve.h, CUDA for
sm_100a in csrc/).  This package is the thin Python binding (`ops`) plus the
per-layer decode-step driver (`engine`) used by the tests and bench.py.
There is no CPU fallback: if the library is missing, the ops raise.
"""
from . import _lib  # noqa: F401

__all__ = ["ops", "engine", "build"]
