"""B200-native MoEtion checkpoint data path (sparse snapshot pack + peer
replicate, sparse-to-dense merge with fused Adam replay, upstream logging).

The product is the C ABI in include/mlck_b200.h implemented by the sm_100a
kernels under csrc/ (built in-tree into _build/libmlck_b200.so).  `mlck` is
the Python binding used by the tests and bench.py.
"""
from . import mlck  # noqa: F401

__all__ = ["mlck"]
