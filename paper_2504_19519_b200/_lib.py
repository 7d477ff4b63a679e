"""ctypes binding of include/flashoverlap.h (argument marshalling only).

Every step of the hot path runs in libflashoverlap.so (the sm_100a kernels,
the stream waits and the NCCL calls).  If the library is missing this module
raises: there is no Python / CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libflashoverlap.so")

FO_OK, FO_ERR_INVALID_ARG, FO_ERR_SHAPE, FO_ERR_UNSUPPORTED, FO_ERR_CUDA, FO_ERR_NCCL, FO_ERR_OOM, \
    FO_ERR_TIMEOUT, FO_ERR_STATE = range(9)
STATUS_NAMES = ["OK", "INVALID_ARG", "SHAPE", "UNSUPPORTED", "CUDA", "NCCL", "OOM", "TIMEOUT", "STATE"]

COLL = {"allreduce": 0, "reducescatter": 1, "alltoall": 2, "nocomm": 3}
LAYOUT = {"slot": 0, "rowband": 1, "auto": 2}
POST = {"none": 0, "add": 1, "add_rmsnorm": 2, "add_rmsnorm_res": 3}
OPTION = {"group_post": 0, "wait_kernel": 1, "tail_split": 2, "post_sm_partition": 3, "host_pipeline": 4, "host_chunks": 5,
          "last_group_in_order": 6, "wave_sync": 7, "multicast": 8, "debug_stall_group": 10, "gemm_swiglu": 11,
          "dist_fold": 12, "k_snake": 13, "tma_store": 14,
          "post_bulk": 15}


class FOError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"FO_ERR_{name}: {msg}")


class PlanDescC(C.Structure):
    _fields_ = [
        ("coll", C.c_int32), ("ar_layout", C.c_int32),
        ("m", C.c_int64), ("n", C.c_int64), ("k", C.c_int64),
        ("tile_m", C.c_int32), ("tile_n", C.c_int32), ("workers", C.c_int32),
        ("tile_order", C.POINTER(C.c_int32)), ("swizzle", C.c_int32),
        ("num_groups", C.c_int32), ("group_waves", C.POINTER(C.c_int32)),
        ("row_dst", C.POINTER(C.c_int32)),
        ("post", C.c_int32), ("eps", C.c_float),
        ("a_mn_major", C.c_int32), ("b_mn_major", C.c_int32),
    ]


class PlanInfoC(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("world", C.c_int32),
        ("mt", C.c_int32), ("nt", C.c_int32), ("tiles", C.c_int32),
        ("workers", C.c_int32), ("waves", C.c_int32), ("num_groups", C.c_int32),
        ("ar_layout", C.c_int32), ("rs_subtile_rows", C.c_int32),
        ("send_elems", C.c_int64), ("recv_elems", C.c_int64),
        ("out_rows", C.c_int64), ("out_cols", C.c_int64),
    ]


class CtxConfigC(C.Structure):
    _fields_ = [("nccl_max_ctas", C.c_int32), ("nccl_min_ctas", C.c_int32), ("cta_policy", C.c_int32),
                ("nvls_ctas", C.c_int32), ("buffers", C.c_int32)]


CTA_POLICY = {"default": 0, "efficiency": 1, "zero": 2}
BUFFERS = {"plain": 0, "registered": 1, "window": 2}


class CommCallC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("group", C.c_int32), ("peer", C.c_int32), ("src_buf", C.c_int32),
                ("dst_buf", C.c_int32), ("reserved", C.c_int32), ("src_off", C.c_int64), ("dst_off", C.c_int64),
                ("count", C.c_int64)]


CALL_KINDS = ["allreduce", "reducescatter", "send", "recv", "local_copy", "group_start", "group_end"]
BUFS = {-1: None, 0: "send", 1: "recv", 2: "out", 3: "scratch"}

# (name, restype, argtypes) for every symbol include/flashoverlap.h declares
_P = C.c_void_p
_SIGS = [
    ("fo_last_error", C.c_char_p, []),
    ("fo_version", C.c_char_p, []),
    ("fo_device_sm_count", C.c_int, [C.c_int32, C.POINTER(C.c_int32)]),
    ("fo_plan_create", C.c_int, [C.POINTER(PlanDescC), C.c_int32, C.c_int32, C.POINTER(C.POINTER(PlanDescC)),
                                 C.POINTER(_P)]),
    ("fo_plan_destroy", C.c_int, [_P]),
    ("fo_plan_get_info", C.c_int, [_P, C.POINTER(PlanInfoC)]),
    ("fo_plan_group", C.c_int, [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("fo_plan_export_order", C.c_int, [_P, C.POINTER(C.c_int32)]),
    ("fo_plan_export_send_map", C.c_int, [_P, C.POINTER(C.c_int64)]),
    ("fo_plan_export_recv_map", C.c_int, [_P, C.POINTER(C.c_int64)]),
    ("fo_plan_export_a2a_counts", C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("fo_plan_export_calls", C.c_int, [_P, C.c_int32, C.POINTER(CommCallC), C.c_int32, C.POINTER(C.c_int32)]),
    ("fo_get_unique_id", C.c_int, [C.POINTER(C.c_uint8)]),
    ("fo_ctx_create", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint8), C.c_int32,
                                C.POINTER(_P)]),
    ("fo_ctx_create_from_comm", C.c_int, [C.c_int32, _P, C.POINTER(_P)]),
    ("fo_ctx_destroy", C.c_int, [_P]),
    ("fo_loopback_create", C.c_int, [C.c_int32, C.c_int32, C.POINTER(_P)]),
    ("fo_loopback_destroy", C.c_int, [_P]),
    ("fo_ctx_create_loopback", C.c_int, [_P, C.c_int32, C.POINTER(_P)]),
    ("fo_ctx_create_emulated", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_int32,
                                         C.POINTER(_P)]),
    ("fo_ctx_time_collective", C.c_int, [_P, C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double)]),
    ("fo_ctx_create_config", C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint8),
                                       C.POINTER(CtxConfigC), C.POINTER(_P)]),
    ("fo_mem_alloc", C.c_int, [_P, C.c_int64, C.POINTER(_P)]),
    ("fo_mem_free", C.c_int, [_P, _P]),
    ("fo_run", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    ("fo_run_sequential", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    ("fo_run_host", C.c_int, [_P, _P, _P, _P, _P, _P, _P, _P]),
    ("fo_run_allgather", C.c_int, [_P, _P, _P, _P, _P, _P, C.c_int32, _P]),
    ("fo_rowexchange_stage", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("fo_gemm_stage", C.c_int, [_P, _P, _P, _P, _P]),
    ("fo_gemm_stage_timed", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("fo_post_stage", C.c_int, [_P, _P, _P, _P, _P, _P]),
    ("fo_group_post_stage", C.c_int, [_P, C.c_int32, _P, _P, _P, _P]),
    ("fo_combine_stage", C.c_int, [_P, _P, _P, _P, _P, C.c_int32, C.c_int64, _P, _P]),
    ("fo_run_combine", C.c_int, [_P, _P, _P, _P, _P, _P, _P, C.c_int32, C.c_int64, _P, _P]),
    ("fo_plan_read_counters", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("fo_plan_prepare", C.c_int, [_P, _P, C.c_int32]),
    ("fo_plan_gemm_cluster", C.c_int, [_P, C.POINTER(C.c_int32)]),
    ("fo_plan_sync", C.c_int, [_P, _P, _P, C.c_int64]),
    ("fo_kernel_launch_count", C.c_int64, []),
    ("fo_plan_set_debug", C.c_int, [_P, _P, _P, C.c_int32]),
    ("fo_plan_fill_buffers", C.c_int, [_P, C.c_uint16, _P]),
    ("fo_plan_set_option", C.c_int, [_P, C.c_int32, C.c_int64]),
    ("fo_tune_predict", C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_double,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)]),
    ("fo_tune_search", C.c_int, [C.c_double, C.c_int32, C.c_int32, C.c_double, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_double)]),
    ("fo_tune_predict_multi", C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.c_int32,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                        C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_double)]),
    ("fo_tune_search_multi", C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32, C.c_int32,
                                       C.c_int32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                       C.POINTER(C.c_double)]),
]
SYMBOLS = [s[0] for s in _SIGS]

_lib = None


def load():
    """Load libflashoverlap.so (built in-tree by build.py) and bind its symbols."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    for name, res, args in _SIGS:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def check(status: int):
    if status != FO_OK:
        raise FOError(status, load().fo_last_error().decode(errors="replace"))
