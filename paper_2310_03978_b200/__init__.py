"""B200-native (sm_100a) sliced tensor-network contraction — arXiv 2310.03978.

The product is the C-ABI library ``libtn.so`` (include/tn.h) built from
``csrc/``: path executor + tcgen05/TMA complex GEMM + permutation/split prep +
SIMT einsum + fused fp64 slice accumulation.  ``tn`` is the ctypes binding;
``distributed`` partitions slices over ranks and reduces with NCCL.
"""
from .tn import Contraction, TNError, TNLibraryError, lib, EXTENDED, MIXED  # noqa: F401

__all__ = ["Contraction", "TNError", "TNLibraryError", "lib", "EXTENDED", "MIXED"]
