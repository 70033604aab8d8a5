"""ctypes view of include/apml.h (libapml.so).  Argument marshalling only.

The product path has no fallback: if libapml.so is missing or cannot be loaded this module
raises; there is no CPU or PyTorch implementation of the method behind it.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("APML_LIB") or os.path.join(HERE, "libapml.so")

APML_OK, APML_ERR_INVALID_ARG, APML_ERR_SHAPE, APML_ERR_NONFINITE, APML_ERR_CAPACITY, \
    APML_ERR_CUDA, APML_ERR_OOM, APML_ERR_STATE = range(8)
STATUS_NAMES = {0: "OK", 1: "INVALID_ARG", 2: "SHAPE", 3: "NONFINITE", 4: "CAPACITY", 5: "CUDA",
                6: "OOM", 7: "STATE"}
APML_GRAD_FULL, APML_GRAD_PLAN_DETACHED = 0, 1
APML_FLAG_SYNC_CHECK, APML_FLAG_CHECK_FINITE, APML_FLAG_STAGE_TIMING, APML_FLAG_UNIFORM_FALLBACK = 1, 2, 4, 8
STAGES = ("staging", "passA_rows", "passA_cols", "line_info", "emit", "sparse_fwd", "sparse_bwd")

# exported symbols declared in include/apml.h (checked by tests/test_abi.py)
EXPORTS = ("apml_abi_version", "apml_config_default", "apml_forward", "apml_forward_ragged",
           "apml_forward_rowsharded",
           "apml_backward", "apml_backward_ex", "apml_plan_create", "apml_plan_forward",
           "apml_ctx_stats", "apml_ctx_support", "apml_ctx_lines", "apml_ctx_stage_times",
           "apml_ctx_destroy",
           "apml_loss_grad_host", "apml_plan_step_host", "apml_nvls_create", "apml_nvls_destroy", "apml_nvls_is_multicast",
           "apml_plan_forward_backward",
           "apml_last_error")


class ApmlConfig(C.Structure):
    _fields_ = [("p_min", C.c_float), ("tau", C.c_float), ("l_iter", C.c_int32),
                ("eps_stab", C.c_float), ("delta", C.c_float), ("eps_g", C.c_float),
                ("eps_dist", C.c_float), ("grad_mode", C.c_int32), ("capacity", C.c_int32),
                ("flags", C.c_uint32)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p)


class ApmlAllocator(C.Structure):
    _fields_ = [("alloc", ALLOC_FN), ("free", FREE_FN), ("user", C.c_void_p)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)
GATHER_BYTES_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class ApmlComm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("allreduce_sum_f32", ALLREDUCE_FN),
                ("allgather_f32", ALLGATHER_FN), ("user", C.c_void_p),
                ("allgather_bytes", GATHER_BYTES_FN), ("nvls", C.c_void_p)]


class ApmlStats(C.Structure):
    _fields_ = [("nnz_total", C.c_int64), ("emitted_total", C.c_int64), ("clamp_count", C.c_int64),
                ("capacity", C.c_int64), ("overflow_pairs", C.c_int64), ("bytes_ctx", C.c_int64),
                ("launches", C.c_int64), ("sweep_evals", C.c_int64 * 3), ("uniform_count", C.c_int64)]


class ApmlError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"APML_ERR_{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_lib = None


def lib() -> C.CDLL:
    """Load libapml.so (built in-tree by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                              "There is no fallback implementation.")
        L = C.CDLL(LIB_PATH)
        vp, i64 = C.c_void_p, C.c_int64
        L.apml_abi_version.restype = C.c_int
        L.apml_abi_version.argtypes = []
        L.apml_config_default.restype = None
        L.apml_config_default.argtypes = [C.POINTER(ApmlConfig)]
        L.apml_forward.restype = C.c_int
        L.apml_forward.argtypes = [vp, vp, i64, i64, i64, C.POINTER(ApmlConfig),
                                   C.POINTER(ApmlAllocator), vp, vp, C.POINTER(vp)]
        L.apml_forward_ragged.restype = C.c_int
        L.apml_forward_ragged.argtypes = [vp, vp, i64, i64, i64, vp, vp, C.POINTER(ApmlConfig),
                                          C.POINTER(ApmlAllocator), vp, vp, C.POINTER(vp)]
        L.apml_forward_rowsharded.restype = C.c_int
        L.apml_forward_rowsharded.argtypes = [vp, vp, i64, i64, i64, i64, i64, C.POINTER(ApmlConfig),
                                              C.POINTER(ApmlAllocator), C.POINTER(ApmlComm), vp, vp,
                                              C.POINTER(vp)]
        L.apml_backward.restype = C.c_int
        L.apml_backward.argtypes = [vp, vp, vp, vp]
        L.apml_plan_create.restype = C.c_int
        L.apml_plan_create.argtypes = [i64, i64, i64, C.POINTER(ApmlConfig), C.POINTER(ApmlAllocator), vp,
                                       C.POINTER(vp)]
        L.apml_plan_forward.restype = C.c_int
        L.apml_plan_forward.argtypes = [vp, vp, vp, vp, vp]
        L.apml_backward_ex.restype = C.c_int
        L.apml_backward_ex.argtypes = [vp, vp, vp, vp, vp]
        L.apml_ctx_stats.restype = C.c_int
        L.apml_ctx_stats.argtypes = [vp, vp, C.POINTER(ApmlStats)]
        L.apml_ctx_support.restype = C.c_int
        L.apml_ctx_support.argtypes = [vp, i64, C.POINTER(C.c_int64), vp, vp, vp, vp, vp]
        L.apml_ctx_lines.restype = C.c_int
        L.apml_ctx_lines.argtypes = [vp, i64, C.c_int32, vp, vp, vp, vp, vp]
        L.apml_ctx_stage_times.restype = C.c_int
        L.apml_ctx_stage_times.argtypes = [vp, vp, C.c_int32]
        L.apml_ctx_destroy.restype = None
        L.apml_ctx_destroy.argtypes = [vp]
        L.apml_loss_grad_host.restype = C.c_int
        L.apml_loss_grad_host.argtypes = [vp, vp, i64, i64, i64, C.POINTER(ApmlConfig),
                                          C.POINTER(ApmlAllocator), vp, vp, vp]
        L.apml_nvls_create.restype = C.c_int
        L.apml_nvls_create.argtypes = [C.POINTER(ApmlComm), C.c_size_t, C.POINTER(vp)]
        L.apml_nvls_is_multicast.restype = C.c_int
        L.apml_nvls_is_multicast.argtypes = [vp]
        L.apml_nvls_destroy.restype = None
        L.apml_nvls_destroy.argtypes = [vp]
        L.apml_plan_forward_backward.restype = C.c_int
        L.apml_plan_forward_backward.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.apml_plan_step_host.restype = C.c_int
        L.apml_plan_step_host.argtypes = [vp, vp, vp, vp, vp, vp]
        L.apml_last_error.restype = C.c_char_p
        L.apml_last_error.argtypes = []
        if L.apml_abi_version() != 3:
            raise ImportError("libapml.so ABI version mismatch")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != APML_OK:
        raise ApmlError(status, (lib().apml_last_error() or b"").decode())
