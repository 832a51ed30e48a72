"""ctypes binding of include/hgnn_b200.h (the C-ABI of libhgnn_b200.so).

Status codes are turned into the Python mirror of the reference's exception
hierarchy (error.hpp:8-72). The library is loaded from the package tree; when
it is missing the import fails loudly -- there is no fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# HGNN_B200_LIB: alternative build of the same library (timing experiments, scripts/build_exp.py)
_LIB_PATH = Path(os.environ.get("HGNN_B200_LIB") or Path(__file__).resolve().parent / "lib" / "libhgnn_b200.so")


class Error(RuntimeError):
    """hgnn::Error"""


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class PartitionError(Error):
    pass


class CollectiveError(Error):
    pass


class IntegrityError(Error):
    pass


class UninitializedError(Error):
    pass


class SizeError(Error):
    pass


class OptimizerError(Error):
    """hgnn::OptimizerError (error.hpp:51-55)."""


class IoError(Error):
    """hgnn::IoError (error.hpp:69-73)."""


class DeviceError(Error):
    """CUDA / NCCL failure or missing B200."""


_CODES = {1: ShapeError, 2: ConfigError, 3: PartitionError, 4: CollectiveError, 5: IntegrityError,
          6: UninitializedError, 7: SizeError, 8: OptimizerError, 9: IoError, 20: DeviceError, 21: DeviceError, 22: Error}

MODE_NONE, MODE_A2A, MODE_NA2A = 0, 1, 2
MODES = {"none": MODE_NONE, "a2a": MODE_A2A, "na2a": MODE_NA2A}
PART_SLAB, PART_BLOCK, PART_VERIFY = 0, 1, 2
TRACE_X_IN, TRACE_E_IN, TRACE_A_SYNC, TRACE_X_OUT, TRACE_E_OUT = range(5)
K_EDGE_FWD, K_EDGE_BWD, K_NODE_FWD, K_NODE_BWD, K_AGG, K_DX, K_HALO, K_GRAD_REDUCE = range(8)
KERNEL_CLASSES = ["edge_fwd", "edge_bwd", "node_fwd", "node_bwd", "aggregate", "dx_gather", "halo", "grad_reduce", "encode",
                  "decode", "loss_adam", "edge_proj"]

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)


class GraphDesc(C.Structure):
    """hgnn_graph_desc"""
    _fields_ = [
        ("rank", C.c_int32), ("num_ranks", C.c_int32),
        ("num_local", C.c_int64), ("num_halo", C.c_int64), ("num_edges", C.c_int64),
        ("global_ids", i64p), ("positions", f64p),
        ("edge_src", i32p), ("edge_dst", i32p), ("node_degree", i32p), ("edge_degree", i32p),
        ("node_inv_degree", f64p), ("edge_inv_degree", f64p),
        ("in_offsets", i32p), ("in_edges", i32p), ("out_offsets", i32p), ("out_edges", i32p),
        ("num_neighbors", C.c_int32), ("neighbors", i32p),
        ("send_offsets", i32p), ("send_rows", i32p), ("recv_offsets", i32p), ("recv_rows", i32p),
        ("halo_to_local", i32p),
        ("num_sync_groups", C.c_int64), ("sync_local", i32p), ("sync_offsets", i32p), ("sync_slots", i32p),
        ("max_buffer_rows", C.c_int64),
    ]


def _preload_nccl() -> None:
    """Bind libnccl.so.2 to the NCCL that PyTorch ships (nvidia-nccl wheel) when
    present, so this library and torch.distributed share ONE NCCL in a process
    regardless of import order (the system copy is older than torch's)."""
    import sys
    for base in sys.path:
        cand = Path(base) / "nvidia" / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            try:
                C.CDLL(str(cand), mode=C.RTLD_GLOBAL)
            except OSError:
                continue
            return


def _load() -> C.CDLL:
    _preload_nccl()
    if not _LIB_PATH.exists():
        raise ImportError(
            f"{_LIB_PATH} is missing: build it with `python paper_2410_01657_b200/build.py` "
            "(the hot path has no CPU fallback)")
    lib = C.CDLL(str(_LIB_PATH), mode=C.RTLD_GLOBAL)
    vp, u8p = C.c_void_p, C.POINTER(C.c_uint8)
    sig = {
        "hgnn_last_error": (C.c_char_p, []),
        "hgnn_graph_build": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, i64p, C.c_int32, C.POINTER(vp)]),
        "hgnn_graph_build_domain": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, i64p, C.c_int32, f64p, f64p,
                                              C.POINTER(vp)]),
        "hgnn_graph_free": (None, [vp]),
        "hgnn_graph_view": (C.c_int, [vp, C.POINTER(GraphDesc)]),
        "hgnn_graph_save_binary": (C.c_int, [C.POINTER(GraphDesc), C.c_char_p]),
        "hgnn_graph_load_binary": (C.c_int, [C.c_char_p, C.POINTER(vp)]),
        "hgnn_balanced_factors": (C.c_int, [C.c_int64, C.c_int64, i64p]),
        "hgnn_param_count": (C.c_int64, [C.c_int64] * 6),
        "hgnn_init_params": (C.c_int, [C.c_int64] * 6 + [C.c_uint64, f64p]),
        "hgnn_mp_param_range": (C.c_int, [C.c_int64] * 5 + [i64p, i64p]),
        "hgnn_device_count": (C.c_int, []),
        "hgnn_nccl_unique_id": (C.c_int, [u8p]),
        "hgnn_ctx_create": (C.c_int, [C.c_int, C.c_int32, C.c_int32, u8p, C.POINTER(vp)]),
        "hgnn_local_group_create": (C.c_int, [C.c_int32, C.POINTER(vp)]),
        "hgnn_local_group_destroy": (C.c_int, [vp]),
        "hgnn_local_group_set_timeout": (C.c_int, [vp, C.c_int64]),
        "hgnn_ctx_create_local": (C.c_int, [C.c_int, C.c_int32, vp, C.POINTER(vp)]),
        "hgnn_ctx_destroy": (C.c_int, [vp]),
        "hgnn_ctx_stream": (vp, [vp]),
        "hgnn_graph_upload": (C.c_int, [vp, C.POINTER(GraphDesc)]),
        "hgnn_configure": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64, C.c_int]),
        "hgnn_params_upload": (C.c_int, [vp, f64p, C.c_int64]),
        "hgnn_mp_forward": (C.c_int, [vp, f64p, f64p, f64p, f64p]),
        "hgnn_mp_backward": (C.c_int, [vp, f64p, f64p, f64p, f64p, f64p]),
        "hgnn_get_trace": (C.c_int, [vp, C.c_int, C.c_int, f64p]),
        "hgnn_synthetic_inputs": (C.c_int, [vp, C.c_uint64]),
        "hgnn_set_inputs": (C.c_int, [vp, f64p, f64p, f64p]),
        "hgnn_mp_step_device": (C.c_int, [vp]),
        "hgnn_get_grads": (C.c_int, [vp, f64p]),
        "hgnn_set_option": (C.c_int, [vp, C.c_char_p, C.c_int64]),
        "hgnn_debug_profile": (C.c_int, [vp, C.c_void_p]),
        "hgnn_model_configure": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int64]),
        "hgnn_model_param_count": (C.c_int64, [vp]),
        "hgnn_model_params_upload": (C.c_int, [vp, f64p, C.c_int64]),
        "hgnn_model_params_download": (C.c_int, [vp, f64p]),
        "hgnn_model_set_data": (C.c_int, [vp, f64p, f64p, f64p]),
        "hgnn_compute_gradients": (C.c_int, [vp, C.POINTER(C.c_double), f64p, f64p]),
        "hgnn_train_step": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(C.c_double)]),
        "hgnn_kernel_timing": (C.c_int, [vp, C.c_int]),
        "hgnn_kernel_time": (C.c_int, [vp, C.c_int, f64p, i64p]),
        "hgnn_launch_count": (C.c_int64, [vp, C.c_int]),
        "hgnn_halo_bytes": (C.c_int64, [vp, C.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()
EXPORTED = ["hgnn_last_error", "hgnn_graph_build", "hgnn_graph_build_domain", "hgnn_graph_free", "hgnn_graph_view", "hgnn_graph_save_binary",
            "hgnn_graph_load_binary", "hgnn_balanced_factors",
            "hgnn_param_count", "hgnn_init_params", "hgnn_mp_param_range", "hgnn_device_count", "hgnn_nccl_unique_id",
            "hgnn_ctx_create", "hgnn_local_group_create", "hgnn_local_group_destroy", "hgnn_local_group_set_timeout",
            "hgnn_ctx_create_local", "hgnn_ctx_destroy", "hgnn_ctx_stream", "hgnn_graph_upload", "hgnn_configure",
            "hgnn_params_upload", "hgnn_mp_forward", "hgnn_mp_backward", "hgnn_get_trace",
            "hgnn_synthetic_inputs", "hgnn_set_inputs", "hgnn_mp_step_device", "hgnn_get_grads",
            "hgnn_set_option", "hgnn_model_configure", "hgnn_model_param_count",
            "hgnn_model_params_upload", "hgnn_model_params_download", "hgnn_model_set_data", "hgnn_compute_gradients",
            "hgnn_train_step", "hgnn_debug_profile", "hgnn_kernel_timing", "hgnn_kernel_time", "hgnn_launch_count", "hgnn_halo_bytes"]


def check(status: int) -> None:
    if status != 0:
        msg = LIB.hgnn_last_error().decode(errors="replace")
        raise _CODES.get(status, Error)(msg)


def lib_path() -> str:
    return os.fspath(_LIB_PATH)


def debug_lib() -> C.CDLL:
    """lib/libhgnn_b200_debug.so: tcgen05 self-tests and microbenchmarks (scripts/dbg_*.py)."""
    lib = C.CDLL(os.fspath(_LIB_PATH.parent / "libhgnn_b200_debug.so"))
    lib.hgnn_selftest_mma.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.hgnn_bench_mma.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    lib.hgnn_bench_alu.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    return lib
