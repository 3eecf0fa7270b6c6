"""ctypes binding of the native library ``_ts_gpu.so`` (C ABI in
``include/treescore_gpu.h``).

There is no CPU fallback: if the library cannot be loaded the scoring API
raises :class:`NativeLibraryError`.  (The model / data layers work without it.)
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# TS_GPU_SO overrides the library path (A/B timing of alternative builds).
SO_PATH = os.environ.get("TS_GPU_SO") or os.path.join(HERE, "_ts_gpu.so")

TS_OK = 0
TS_ERR_INVALID = 1
TS_ERR_DEPTH = 2
TS_ERR_SHAPE = 3
TS_ERR_NONFINITE = 4
TS_ERR_CUDA = 5
TS_ERR_NOMEM = 6
TS_ERR_UNSUPPORTED = 7
TS_ERR_SYNTAX = 8
TS_PACK_TRACE = 1
TS_PACK_ANY_DEPTH = 2
TS_PACK_NO_RANK = 4

# Every symbol include/treescore_gpu.h declares (checked by the CPU tests).
EXPORTS = ("ts_pack", "ts_pack_ex", "ts_trace", "ts_model_get_info", "ts_score", "ts_score_ex", "ts_score_host", "ts_free",
           "ts_last_error", "ts_launch_count", "ts_version", "ts_synth_uniform", "ts_set_kernel_path",
           "ts_parse_model", "ts_flat_free", "ts_score_pipe", "ts_pipe_alloc", "ts_pipe_free",
           "ts_ipc_open", "ts_ipc_close", "ts_nccl_get_unique_id", "ts_nccl_comm_init",
           "ts_reduce_partials", "ts_nccl_comm_destroy", "ts_nccl_wait")


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or failed to load (no fallback exists)."""


class ModelDesc(ctypes.Structure):
    _fields_ = [("num_features", ctypes.c_int32),
                ("num_trees", ctypes.c_int32),
                ("tree_node_offset", ctypes.c_void_p),
                ("tree_weight", ctypes.c_void_p),
                ("node_fid", ctypes.c_void_p),
                ("node_value", ctypes.c_void_p),
                ("node_left", ctypes.c_void_p),
                ("node_right", ctypes.c_void_p)]


class FlatModelC(ctypes.Structure):
    _fields_ = [("num_features", ctypes.c_int32),
                ("num_trees", ctypes.c_int32),
                ("num_nodes", ctypes.c_int64),
                ("tree_node_offset", ctypes.POINTER(ctypes.c_int64)),
                ("tree_weight", ctypes.POINTER(ctypes.c_double)),
                ("node_fid", ctypes.POINTER(ctypes.c_int32)),
                ("node_value", ctypes.POINTER(ctypes.c_float)),
                ("node_left", ctypes.POINTER(ctypes.c_int32)),
                ("node_right", ctypes.POINTER(ctypes.c_int32)),
                ("err_line", ctypes.c_int32),
                ("err_col", ctypes.c_int32)]


class Pipe(ctypes.Structure):
    _fields_ = [("sums_in", ctypes.c_void_p),
                ("flags_in", ctypes.c_void_p),
                ("sums_out", ctypes.c_void_p),
                ("flags_out", ctypes.c_void_p),
                ("epoch", ctypes.c_uint32)]


class ModelInfo(ctypes.Structure):
    _fields_ = [("num_features", ctypes.c_int32),
                ("num_trees", ctypes.c_int32),
                ("max_depth", ctypes.c_int32),
                ("num_segments", ctypes.c_int32),
                ("sum_depth", ctypes.c_int64),
                ("table_entries", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64),
                ("complete_trees", ctypes.c_int32),
                ("compact_trees", ctypes.c_int32),
                ("device", ctypes.c_int32),
                ("unit_weights", ctypes.c_int32),
                ("rank_trees", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = True):
    """Load (building first if absent and nvcc exists) and type the library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(SO_PATH) and build_if_missing:
            try:
                from ._build import build
                build()
            except Exception as exc:  # noqa: BLE001 - surfaced below
                raise NativeLibraryError(f"{SO_PATH} missing and build failed: {exc}") from exc
        try:
            lib = ctypes.CDLL(SO_PATH)
        except OSError as exc:
            raise NativeLibraryError(f"cannot load {SO_PATH}: {exc}") from exc
        P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.ts_pack.argtypes = [ctypes.POINTER(ModelDesc), ctypes.c_int, ctypes.POINTER(P)]
        lib.ts_pack.restype = ctypes.c_int
        lib.ts_pack_ex.argtypes = [ctypes.POINTER(ModelDesc), ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(P)]
        lib.ts_pack_ex.restype = ctypes.c_int
        lib.ts_trace.argtypes = [P, P, I64, I64, I64, P, P, I64, P, I32, P]
        lib.ts_trace.restype = ctypes.c_int
        lib.ts_model_get_info.argtypes = [P, ctypes.POINTER(ModelInfo)]
        lib.ts_model_get_info.restype = ctypes.c_int
        lib.ts_score.argtypes = [P, P, I64, I64, I64, P, P, I64, P, P]
        lib.ts_score.restype = ctypes.c_int
        lib.ts_score_ex.argtypes = [P, P, I64, I64, I64, P, P, I64, P, ctypes.c_int, P]
        lib.ts_score_ex.restype = ctypes.c_int
        lib.ts_score_host.argtypes = [P, P, I64, I64, P]
        lib.ts_score_host.restype = ctypes.c_int
        lib.ts_free.argtypes = [P]
        lib.ts_free.restype = None
        lib.ts_last_error.argtypes = []
        lib.ts_last_error.restype = ctypes.c_char_p
        lib.ts_launch_count.argtypes = []
        lib.ts_launch_count.restype = I64
        lib.ts_version.argtypes = []
        lib.ts_version.restype = ctypes.c_char_p
        lib.ts_synth_uniform.argtypes = [P, I64, I64, I64, ctypes.c_uint64, I64,
                                         ctypes.c_double, P]
        lib.ts_synth_uniform.restype = ctypes.c_int
        lib.ts_set_kernel_path.argtypes = [ctypes.c_int]
        lib.ts_set_kernel_path.restype = ctypes.c_int
        lib.ts_parse_model.argtypes = [ctypes.c_char_p, I64,
                                       ctypes.POINTER(ctypes.POINTER(FlatModelC))]
        lib.ts_parse_model.restype = ctypes.c_int
        lib.ts_flat_free.argtypes = [ctypes.POINTER(FlatModelC)]
        lib.ts_flat_free.restype = None
        lib.ts_score_pipe.argtypes = [P, P, I64, I64, I64, P, ctypes.POINTER(Pipe), P]
        lib.ts_score_pipe.restype = ctypes.c_int
        lib.ts_pipe_alloc.argtypes = [ctypes.c_int, I64, ctypes.POINTER(P), ctypes.POINTER(P), P, P]
        lib.ts_pipe_alloc.restype = ctypes.c_int
        lib.ts_pipe_free.argtypes = [P, P]
        lib.ts_pipe_free.restype = None
        lib.ts_ipc_open.argtypes = [P, ctypes.POINTER(P)]
        lib.ts_ipc_open.restype = ctypes.c_int
        lib.ts_ipc_close.argtypes = [P]
        lib.ts_ipc_close.restype = None
        lib.ts_nccl_get_unique_id.argtypes = [P]
        lib.ts_nccl_comm_init.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.POINTER(P)]
        lib.ts_reduce_partials.argtypes = [P, P, P, I64, ctypes.c_int, P]
        lib.ts_nccl_comm_destroy.argtypes = [P]
        lib.ts_nccl_wait.argtypes = [P, P, I64]
        for name in EXPORTS:
            getattr(lib, name)
        _lib = lib
        return lib


def last_error() -> str:
    return load().ts_last_error().decode("utf-8", "replace")


def launch_count() -> int:
    return int(load().ts_launch_count())
