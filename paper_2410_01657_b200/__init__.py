"""B200-native consistent neural message-passing layer (arXiv 2410.01657).

Host side (numpy + ctypes) above the C-ABI `include/hgnn_b200.h`; the hot path
runs in `lib/libhgnn_b200.so` (hand-written sm_100a CUDA + NCCL). There is no
CPU fallback: importing this package fails if the native library is absent.
"""
from ._native import (CollectiveError, ConfigError, DeviceError, Error, IntegrityError, IoError,
                      OptimizerError, PartitionError, ShapeError, SizeError, UninitializedError, lib_path)
from .engine import Engine, LocalGroup, nccl_unique_id
from .graph import (RankGraph, balanced_factors, build_distributed_graph, build_rank_graph, load_graph_binary,
                    save_graph_binary)
from .params import (GnnConfig, init_params, model_slices, mp_layer_slices, mp_param_range, mp_params,
                     param_count)

__all__ = [
    "Engine", "LocalGroup", "nccl_unique_id", "RankGraph", "build_rank_graph", "build_distributed_graph", "balanced_factors",
    "load_graph_binary", "save_graph_binary",
    "GnnConfig", "init_params", "mp_params", "mp_param_range", "mp_layer_slices", "model_slices", "param_count",
    "lib_path",
    "Error", "ShapeError", "ConfigError", "PartitionError", "CollectiveError", "IntegrityError",
    "UninitializedError", "SizeError", "OptimizerError", "IoError", "DeviceError",
]
