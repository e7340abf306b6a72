"""B200-native binary low-rank (BLR) hot path of NanoQuant (arxiv 2602.06694).

The product is ``libnqb.so`` (C ABI, include/nqb.h): hand-written sm_100a CUDA
for the BLR-linear forward and the fp64 LB-ADMM initialisation.  This package
is the thin host-side mirror of the reference's C++ API (``nanoquant``) plus
the layer-sharded multi-GPU ADMM driver (``sharded``).  There is no CPU fallback.
"""
from . import _lib  # noqa: F401
from .nanoquant import *  # noqa: F401,F403
from . import sharded  # noqa: F401

__all__ = [name for name in dir() if not name.startswith("_")]
