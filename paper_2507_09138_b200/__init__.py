"""B200-native IVF retrieval hot path for HedraRAG (arXiv 2507.09138).

coarse assign -> grouped inverted-list scan -> exact top-k, as hand-written
sm_100a CUDA kernels behind the C-ABI in include/hivf.h (libhivf.so).
"""
from ._lib import (HivfError, InternalError, InvalidArgument, LIB_PATH, SHARD_STRIPED, SYMBOLS,  # noqa: F401
                   lib)
from .index import (METRIC_COSINE, METRIC_L2, Context, IvfIndex, ShardGroup, nccl_unique_id,  # noqa: F401
                    shard_local_lists, shard_plan, upload_shard)

__all__ = ["Context", "IvfIndex", "METRIC_L2", "METRIC_COSINE", "HivfError", "InvalidArgument",
           "InternalError", "lib", "LIB_PATH", "SYMBOLS", "ShardGroup", "SHARD_STRIPED", "shard_plan", "shard_local_lists",
           "upload_shard", "nccl_unique_id"]
