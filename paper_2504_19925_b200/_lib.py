"""ctypes view of include/moe_dc.h, moe_synth.h and moe_tokens.h (argument marshalling only).

Loads the in-tree ``libmoedc.so``.  There is no fallback: if the library is missing the
import fails loudly (build it with ``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmoedc.so")

MOE_OK = 0
STATUS = {0: "MOE_OK", 1: "MOE_ERR_INVALID", 2: "MOE_ERR_SHAPE", 3: "MOE_ERR_DATA",
          4: "MOE_ERR_CUDA", 5: "MOE_ERR_COMM", 6: "MOE_ERR_INTERNAL", 7: "MOE_ERR_TIMEOUT"}
MOE_MAX_E, MOE_MAX_G, MOE_MAX_SLOTS = 256, 8, 4096
MOE_PLAN_PAPER_ALG1, MOE_PLAN_MINMAX, MOE_PLAN_STATIC, MOE_PLAN_KEEP, MOE_PLAN_SCHEDULED = 0, 1, 2, 3, 4

# every symbol include/*.h declares (checked by tests/test_abi.py)
EXPORTED = [
    "moe_status_str", "moe_last_error", "moe_abi_version", "moe_build_id", "moe_plan", "moe_plan_ex",
    "moe_slot_capacity", "moe_plan_scheduled", "moe_ctx_set_schedule",
    "moe_ctx_create", "moe_ctx_destroy", "moe_ctx_handle_bytes", "moe_ctx_export",
    "moe_ctx_connect", "moe_ctx_check", "moe_ctx_wait_counts", "moe_ctx_weights_wait", "moe_dispatch", "moe_update",
    "moe_place", "moe_step", "moe_ctx_set_timing", "moe_ctx_get_timing", "moe_ctx_get_timing_ex",
    "moe_synth_grads", "moe_synth_master",
    "moe_tokx_create", "moe_tokx_destroy", "moe_tokx_handle_bytes", "moe_tokx_export",
    "moe_tokx_connect", "moe_token_dispatch", "moe_token_combine",
]
MOE_TOK_GATE = 1

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f32p = C.POINTER(C.c_float)


class MoePlanT(C.Structure):
    _fields_ = [("E", C.c_int32), ("G", C.c_int32), ("S", C.c_int32),
                ("replicas", _i32p), ("first_slot", _i32p), ("slot_expert", _i32p)]


class MoeCtxDesc(C.Structure):
    _fields_ = [("E", C.c_int32), ("G", C.c_int32), ("S", C.c_int32), ("k", C.c_int32),
                ("P", C.c_int64), ("max_tokens", C.c_int64),
                ("rank", C.c_int32), ("device", C.c_int32),
                ("slot_w", C.POINTER(C.c_void_p)), ("slot_g", C.POINTER(C.c_void_p)),
                ("master", C.POINTER(C.c_void_p)), ("adam_m", C.POINTER(C.c_void_p)),
                ("adam_v", C.POINTER(C.c_void_p)), ("options", C.c_int32)]


MOE_OPT_DEDUP = 1
MOE_OPT_HOST_STATE = 2
MOE_OPT_LAZY_REPLICATE = 4


class MoeDispatchOut(C.Structure):
    _fields_ = [("dest_slot", C.c_void_p), ("dest_off", C.c_void_p), ("send_pair", C.c_void_p),
                ("send_gate", C.c_void_p), ("send_count", C.c_void_p), ("slot_load", C.c_void_p),
                ("counts_dev", C.c_void_p), ("counts_host", C.c_void_p),
                ("capacity", C.c_int32), ("drops", C.c_void_p)]


class MoeAdamT(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double), ("step", C.c_int64),
                ("scale_mode", C.c_int32), ("scale", _f32p)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.moe_status_str.restype = C.c_char_p
        L.moe_status_str.argtypes = [C.c_int]
        L.moe_last_error.restype = C.c_char_p
        L.moe_last_error.argtypes = []
        L.moe_abi_version.restype = C.c_int
        L.moe_slot_capacity.restype = C.c_int32
        L.moe_slot_capacity.argtypes = [C.c_double, C.c_int64, C.c_int32, C.c_int32, C.c_int32]
        L.moe_plan.restype = C.c_int
        L.moe_plan.argtypes = [_i64p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(MoePlanT)]
        L.moe_plan_ex.restype = C.c_int
        L.moe_plan_ex.argtypes = [_i64p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(MoePlanT), _i64p]
        L.moe_ctx_create.restype = C.c_int
        L.moe_build_id.restype = C.c_char_p
        L.moe_build_id.argtypes = []
        L.moe_plan_scheduled.restype = C.c_int
        L.moe_plan_scheduled.argtypes = [_i64p, C.POINTER(MoePlanT), C.c_int32, C.c_int32, C.c_int64,
                                         C.POINTER(MoePlanT), _i32p]
        L.moe_ctx_set_schedule.restype = C.c_int
        L.moe_ctx_set_schedule.argtypes = [C.c_void_p, C.c_int32, C.c_int32]
        L.moe_ctx_create.argtypes = [C.POINTER(MoeCtxDesc), C.POINTER(C.c_void_p)]
        L.moe_ctx_destroy.restype = C.c_int
        L.moe_ctx_destroy.argtypes = [C.c_void_p]
        L.moe_ctx_handle_bytes.restype = C.c_int
        L.moe_ctx_handle_bytes.argtypes = []
        L.moe_ctx_export.restype = C.c_int
        L.moe_ctx_export.argtypes = [C.c_void_p, C.c_void_p]
        L.moe_ctx_connect.restype = C.c_int
        L.moe_ctx_connect.argtypes = [C.c_void_p, C.c_void_p]
        L.moe_ctx_check.restype = C.c_int
        L.moe_ctx_check.argtypes = [C.c_void_p, C.c_void_p]
        L.moe_ctx_wait_counts.restype = C.c_int
        L.moe_ctx_wait_counts.argtypes = [C.c_void_p]
        L.moe_ctx_weights_wait.restype = C.c_int
        L.moe_ctx_weights_wait.argtypes = [C.c_void_p, C.c_void_p]
        L.moe_place.restype = C.c_int
        L.moe_place.argtypes = [C.c_void_p, C.POINTER(MoePlanT), C.c_void_p]
        L.moe_dispatch.restype = C.c_int
        L.moe_dispatch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                   C.POINTER(MoePlanT), C.POINTER(MoeDispatchOut), C.c_void_p]
        L.moe_step.restype = C.c_int
        L.moe_step.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(MoePlanT),
                               C.POINTER(MoePlanT), C.c_int32, C.POINTER(MoeDispatchOut),
                               C.POINTER(MoeAdamT), C.c_void_p]
        L.moe_ctx_set_timing.restype = C.c_int
        L.moe_ctx_set_timing.argtypes = [C.c_void_p, C.c_int32]
        L.moe_ctx_get_timing.restype = C.c_int
        L.moe_ctx_get_timing.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.moe_ctx_get_timing_ex.restype = C.c_int
        L.moe_ctx_get_timing_ex.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.moe_update.restype = C.c_int
        L.moe_update.argtypes = [C.c_void_p, C.POINTER(MoePlanT), C.POINTER(MoePlanT),
                                 C.POINTER(MoeAdamT), C.c_void_p]
        L.moe_synth_grads.restype = C.c_int
        L.moe_synth_grads.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int64, C.c_void_p]
        L.moe_synth_master.restype = C.c_int
        L.moe_synth_master.argtypes = [C.c_void_p, C.c_uint64, C.c_int32, C.c_int64, C.c_int64,
                                       C.c_void_p]
        L.moe_tokx_create.restype = C.c_int
        L.moe_tokx_create.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p),
                                      C.POINTER(C.c_void_p)]
        L.moe_tokx_destroy.restype = C.c_int
        L.moe_tokx_destroy.argtypes = [C.c_void_p]
        L.moe_tokx_handle_bytes.restype = C.c_int
        L.moe_tokx_handle_bytes.argtypes = []
        L.moe_tokx_export.restype = C.c_int
        L.moe_tokx_export.argtypes = [C.c_void_p, C.c_void_p]
        L.moe_tokx_connect.restype = C.c_int
        L.moe_tokx_connect.argtypes = [C.c_void_p, C.c_void_p]
        for f in (L.moe_token_dispatch, L.moe_token_combine):
            f.restype = C.c_int
            f.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_int64, C.c_void_p,
                          C.POINTER(MoeDispatchOut), C.c_int32, C.c_void_p]
        _lib = L
    return _lib


class MoeError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().moe_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


def check(status: int, where: str) -> None:
    if status != MOE_OK:
        raise MoeError(status, where)
