"""ctypes binding of the C-ABI in include/bida_gpu.h (libbida_gpu.so, in-tree).

There is no fallback: if the CUDA library is missing this module raises, so a
product path can never silently run on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libbida_gpu.so")

BIDA_OK = 0
BIDA_ERR_INVALID_ARGUMENT = 1
BIDA_ERR_RUNTIME = 2
BIDA_ERR_CUDA = 3
BIDA_ERR_DISTRIBUTION = 4
BIDA_ERR_STATE = 5
BIDA_ERR_CAPACITY = 6

PDB_OFF, PDB_MIN, PDB_REPLACE = 0, 1, 2

MODEL_LINEAR = 1
MODEL_MLP = 2


class ModelInfo(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("domain", C.c_int32),
        ("features", C.c_int32),
        ("classes", C.c_int32),
        ("ensemble", C.c_int32),
        ("hidden_layers", C.c_int32),
        ("hidden", C.c_int32 * 8),
        ("quantile", C.c_double),
        ("device", C.c_int32),
        ("weights_in_smem", C.c_int32),
    ]


EXPORTS = [
    "bida_gpu_abi_version",
    "bida_gpu_last_error",
    "bida_gpu_device_count",
    "bida_gpu_feature_length",
    "bida_gpu_packed_bytes",
    "bida_gpu_linear_create",
    "bida_gpu_linear_create_blin1",
    "bida_gpu_linear_load",
    "bida_gpu_mlp_create_bmlp1",
    "bida_gpu_mlp_load",
    "bida_gpu_evaluate",
    "bida_gpu_evaluate_logits",
    "bida_gpu_evaluate_device",
    "bida_gpu_submit",
    "bida_gpu_batch_begin",
    "bida_gpu_batch_launch",
    "bida_gpu_batch_ready",
    "bida_gpu_batch_h",
    "bida_gpu_batch_wait",
    "bida_gpu_stream_status",
    "bida_gpu_attach_pdb",
    "bida_gpu_attach_pdb_file",
    "bida_gpu_attach_pdb_built",
    "bida_gpu_pdb_build",
    "bida_gpu_pdb_build_save",
    "bida_gpu_random_walks",
    "bida_gpu_info",
    "bida_gpu_debug_trace",
    "bida_gpu_trace_slots",
    "bida_gpu_exact_replays",
    "bida_gpu_launch_count",
    "bida_gpu_graph_launch_count",
    "bida_gpu_destroy",
]

_lib = None


def lib() -> C.CDLL:
    """Load libbida_gpu.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"CUDA evaluator library not built: {LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)"
        )
    path = os.environ.get("BIDA_GPU_LIB") or LIB_PATH  # A/B benchmarking of another build
    if os.environ.get("BIDA_GPU_TRACE") == "1":  # diagnostic build with the kernel timeline compiled in
        path = os.path.join(HERE, "_lib", "libbida_gpu_trace.so")
    L = C.CDLL(path)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    H = C.c_void_p
    L.bida_gpu_abi_version.restype = i32
    L.bida_gpu_last_error.restype = C.c_char_p
    L.bida_gpu_device_count.restype = i32
    L.bida_gpu_feature_length.argtypes = [i32]
    L.bida_gpu_packed_bytes.argtypes = [i32]
    L.bida_gpu_linear_create.argtypes = [i32, i32, vp, i32, i32, C.c_double, C.POINTER(H)]
    L.bida_gpu_linear_create_blin1.argtypes = [i32, i32, vp, C.c_size_t, C.c_double, C.POINTER(H)]
    L.bida_gpu_linear_load.argtypes = [i32, i32, C.c_char_p, C.c_double, C.POINTER(H)]
    L.bida_gpu_mlp_create_bmlp1.argtypes = [i32, i32, vp, C.c_size_t, C.c_double, C.POINTER(H)]
    L.bida_gpu_mlp_load.argtypes = [i32, i32, C.c_char_p, C.c_double, C.POINTER(H)]
    L.bida_gpu_evaluate.argtypes = [H, vp, i64, vp]
    L.bida_gpu_evaluate_logits.argtypes = [H, vp, i64, vp, vp]
    L.bida_gpu_evaluate_device.argtypes = [H, vp, i64, vp, vp, vp]
    L.bida_gpu_stream_status.argtypes = [H]
    L.bida_gpu_submit.argtypes = [H, vp, i64, C.POINTER(vp)]
    L.bida_gpu_batch_begin.argtypes = [H, i64, C.POINTER(vp), C.POINTER(vp)]
    L.bida_gpu_batch_launch.argtypes = [vp]
    L.bida_gpu_batch_ready.argtypes = [vp]
    L.bida_gpu_batch_h.argtypes = [vp]
    L.bida_gpu_batch_h.restype = C.POINTER(C.c_int32)
    L.bida_gpu_batch_wait.argtypes = [vp, vp]
    L.bida_gpu_attach_pdb.argtypes = [H, vp, i32, vp, C.c_uint64, i32]
    L.bida_gpu_attach_pdb_file.argtypes = [H, C.c_char_p, i32]
    L.bida_gpu_attach_pdb_built.argtypes = [H, vp, i32, i32]
    L.bida_gpu_pdb_build.argtypes = [i32, i32, vp, i32, C.c_uint64, vp, C.c_uint64, C.POINTER(C.c_uint64),
                                     C.POINTER(i32)]
    L.bida_gpu_pdb_build_save.argtypes = [i32, i32, vp, i32, C.c_char_p]
    L.bida_gpu_random_walks.argtypes = [i32, i32, i64, i32, i32, C.c_uint64, vp, vp]
    L.bida_gpu_info.argtypes = [H, C.POINTER(ModelInfo)]
    L.bida_gpu_debug_trace.argtypes = [H, vp]
    L.bida_gpu_exact_replays.argtypes = [H, C.POINTER(i64)]
    L.bida_gpu_launch_count.argtypes = [H]
    L.bida_gpu_launch_count.restype = i64
    L.bida_gpu_graph_launch_count.argtypes = [H]
    L.bida_gpu_graph_launch_count.restype = i64
    L.bida_gpu_destroy.argtypes = [H]
    _lib = L
    return L


def last_error() -> str:
    return lib().bida_gpu_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map a bida_status to the exception the reference throws for it."""
    if rc == BIDA_OK:
        return
    msg = last_error()
    if rc in (BIDA_ERR_INVALID_ARGUMENT, BIDA_ERR_DISTRIBUTION, BIDA_ERR_STATE, BIDA_ERR_CAPACITY):
        raise ValueError(msg)
    raise RuntimeError(msg)
