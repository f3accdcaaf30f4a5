"""B200-native (sm_100a) ISGMR / TRWP min-sum message passing with
index-driven backward -- a drop-in for the reference mrfmp hot path.

The product is libmrf_cuda.so (C-ABI: include/mrf_cuda.h; C++ drop-in:
include/mrf/mp_cuda.hpp). This package holds its sources (csrc/), the in-tree
build, and a thin torch-facing front end (api.py) used by tests and bench.py.
"""
from ._lib import MrfError, MrfInvalidArgument, lib  # noqa: F401

__all__ = ["MrfError", "MrfInvalidArgument", "lib"]
