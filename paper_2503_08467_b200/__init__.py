"""B200-native MoEShard sharded Switch-MoE layer (arXiv 2503.08467).

The product path: libmoeshard.so (CUDA sm_100a kernels + NCCL, C ABI in
include/moeshard.h) and a thin ctypes/torch binding. Importing this package
without the built library raises ImportError - there is no fallback.
"""
from . import moeshard
from .layer import MoEShardLayer, broadcast_uid, local_token_range, shard_columns
from .moeshard import MoEShardError

__all__ = ["moeshard", "MoEShardLayer", "MoEShardError", "shard_columns", "local_token_range",
           "broadcast_uid"]
