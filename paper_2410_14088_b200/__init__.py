"""paper_2410_14088_b200 — B200-native hot path of BMQSim (arXiv 2410.14088).

Compressed-block state-vector simulation: every stage streams each group of
state-vector blocks through decompress -> gates -> compress on an sm_100a
GPU, byte-exact with the reference CPU implementation. The work runs in
``libbmq.so`` (C ABI: ``include/bmq.h``); ``cbq`` mirrors the reference's
C++ ``namespace cbq`` surface for Python callers and tests.
"""
from . import cbq  # noqa: F401  (loads libbmq.so; raises if it is missing)
from ._lib import LIB_PATH  # noqa: F401

__all__ = ["cbq", "LIB_PATH"]
