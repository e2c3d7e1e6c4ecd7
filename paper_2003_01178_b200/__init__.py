"""B200-native Crystal (arXiv 2003.01178): tile-based block primitives, fused
Star Schema Benchmark queries and operator microbenchmarks on sm_100a.

The compute lives in ``libcrystal_b200.so`` (hand-written CUDA for sm_100a
behind the C ABI of include/crystal_b200.h).  ``tq`` mirrors the reference's
operator/query API over that ABI; ``dist`` shards lineorder across GPUs and
merges partial aggregates with one NCCL reduce.
"""
from . import tq  # noqa: F401  (loads the CUDA library; raises if it is missing)
from ._lib import LIB_PATH  # noqa: F401

__all__ = ["tq", "LIB_PATH"]
