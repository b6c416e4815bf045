"""B200-native IVF retrieval hot path for HedraRAG (arXiv 2507.09138).

coarse assign -> grouped inverted-list scan -> exact top-k, as hand-written
sm_100a CUDA kernels behind the C-ABI in include/hivf.h (libhivf.so).
"""
from ._lib import (HivfError, InternalError, InvalidArgument, LIB_PATH, SYMBOLS,  # noqa: F401
                   lib)
from .index import METRIC_COSINE, METRIC_L2, Context, IvfIndex  # noqa: F401

__all__ = ["Context", "IvfIndex", "METRIC_L2", "METRIC_COSINE", "HivfError", "InvalidArgument",
           "InternalError", "lib", "LIB_PATH", "SYMBOLS"]
