"""ctypes binding of libpb200.so (include/pipeblock_b200.h).

The library is built in-tree by ``paper_2405_15362_b200.build`` (``__graft_entry__.build()``).
Importing this module never builds or falls back: a missing library is an error.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpb200.so")

PB_OK, PB_EINVAL, PB_EDOC, PB_ECUDA, PB_ESPACE, PB_ESTATE = 0, -1, -2, -3, -4, -5
KINDS = ("F", "B", "W", "BW")


class pb_pass(C.Structure):
    _fields_ = [("device", C.c_int32), ("stage", C.c_int32), ("kind", C.c_int32), ("microbatch", C.c_int32),
                ("start", C.c_int64), ("duration", C.c_int64)]


class pb_timed_pass(C.Structure):
    _fields_ = [("device", C.c_int32), ("stage", C.c_int32), ("kind", C.c_int32), ("microbatch", C.c_int32),
                ("start", C.c_double), ("duration", C.c_double)]


class pb_topology(C.Structure):
    _fields_ = [("devices", C.c_int32), ("num_stages", C.c_int32), ("placement", C.POINTER(C.c_int32)),
                ("stage_mem", C.POINTER(C.c_double))]


class pb_profile(C.Structure):
    _fields_ = [("f", C.c_double), ("b", C.c_double), ("w", C.c_double), ("comm", C.c_double)]


class pb_sim_stats(C.Structure):
    _fields_ = [("makespan", C.c_double), ("bubble_rate", C.c_double)]


class pb_model_cfg(C.Structure):
    _fields_ = [("layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32), ("seq", C.c_int32),
                ("vocab", C.c_int32), ("micro_batch", C.c_int32), ("seed", C.c_uint64), ("lr", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float), ("weight_decay", C.c_float),
                ("optimizer", C.c_int32), ("flags", C.c_int32), ("stage_layers", C.POINTER(C.c_int32))]


class pb_exec_stats(C.Structure):
    _fields_ = [("loss", C.c_double), ("step_ms", C.c_double), ("busy_ms", C.c_double), ("pool_slots", C.c_int64),
                ("pool_peak", C.c_int64), ("slot_bytes", C.c_int64), ("pool_bytes", C.c_int64),
                ("peer_bytes", C.c_int64), ("kernel_launches", C.c_int64), ("gemm_ms", C.c_double),
                ("gemm_flops", C.c_double), ("gemm_launches", C.c_int64), ("copy_ms", C.c_double)]


class pb_exec_memory_t(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("weights", "grads", "optimizer", "activation_pool", "head_pool", "transfer",
                                         "scratch", "executor_total", "device_total", "device_used_at_create",
                                         "device_used_high")]


# every symbol include/pipeblock_b200.h declares (checked by tests/test_capi.py)
EXPORTS = [
    "pb_last_error", "pb_abi_version", "pb_schedule_build", "pb_build_info", "pb_search_assemble", "pb_schedule_create", "pb_schedule_parse",
    "pb_schedule_emit", "pb_schedule_info", "pb_schedule_topology", "pb_schedule_passes", "pb_schedule_exact_peak",
    "pb_simulate", "pb_account", "pb_schedule_destroy", "pb_exec_create", "pb_exec_connect_local",
    "pb_exec_export", "pb_exec_connect_ipc", "pb_exec_step", "pb_exec_step_async", "pb_exec_sync",
    "pb_exec_num_passes", "pb_exec_set_flags", "pb_exec_kernel_report", "pb_exec_stream", "pb_exec_param_count", "pb_exec_param_info", "pb_exec_param_get",
    "pb_exec_param_set", "pb_exec_zero_grads", "pb_exec_memory", "pb_exec_destroy",
]


class PipeblockError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ScheduleError(PipeblockError, ValueError):
    """std::invalid_argument in the reference."""


class DocumentError(PipeblockError, ValueError):
    """pipeblock::DocumentError (document.hpp:13-16)."""


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (python -m paper_2405_15362_b200.build)")
        L = C.CDLL(LIB_PATH)
        L.pb_last_error.restype = C.c_char_p
        if hasattr(L, "pb_exec_stream"):
            L.pb_exec_stream.restype = C.c_void_p
            L.pb_exec_stream.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == PB_OK:
        return
    msg = lib().pb_last_error().decode(errors="replace")
    if rc == PB_EINVAL:
        raise ScheduleError(rc, msg)
    if rc == PB_EDOC:
        raise DocumentError(rc, msg)
    raise PipeblockError(rc, msg)


class pb_growth_report(C.Structure):
    _fields_ = [("cycle_length", C.c_int32), ("growth", C.c_double), ("max_work", C.c_double),
                ("repeating_bubble", C.c_double), ("linear_bubble", C.c_int32), ("tie", C.c_int32)]


class pb_search_spec(C.Structure):
    _fields_ = [("devices", C.c_int32), ("microbatches", C.c_int32), ("profile", pb_profile),
                ("memory_limit", C.c_double), ("delta_max", C.c_int64), ("tau_max", C.c_int64)]


class pb_search_params(C.Structure):
    _fields_ = [("K", C.c_int32), ("d0_lo", C.c_int64), ("d1_lo", C.c_int64), ("d0_hi", C.c_int64),
                ("d1_hi", C.c_int64), ("tau1", C.c_int64), ("tau2", C.c_int64), ("tau3", C.c_int64)]


class pb_search_result(C.Structure):
    _fields_ = [("feasible", C.c_int32), ("best", pb_search_params), ("bubble_rate", C.c_double),
                ("exact_peak", C.c_double), ("enumerated", C.c_int64), ("evaluated", C.c_int64),
                ("family_min_peak", C.c_double), ("turn_devices_exercised", C.c_int32)]


class pb_frontier_point(C.Structure):
    _fields_ = [("limit", C.c_double), ("feasible", C.c_int32), ("bubble_rate", C.c_double),
                ("exact_peak", C.c_double), ("best", pb_search_params)]


EXPORTS += ["pb_growth_rate", "pb_growth_rate_unrolled", "pb_vhalf_condition", "pb_lower_bound",
            "pb_min_memory_for_od_bubble", "pb_search", "pb_frontier", "pb_render", "pb_timed_emit",
            "pb_timed_render"]


class pb_plan_op(C.Structure):
    _fields_ = [("stage", C.c_int32), ("kind", C.c_int32), ("microbatch", C.c_int32), ("slot", C.c_int32),
                ("start", C.c_int64), ("recv_from", C.c_int32), ("recv_outbox", C.c_int32), ("recv_gen", C.c_uint32),
                ("send_to", C.c_int32), ("send_outbox", C.c_int32), ("send_gen", C.c_uint32)]


EXPORTS += ["pb_plan_device"]

EXPORTS += ["pb_replay"]
