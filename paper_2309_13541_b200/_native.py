"""ctypes binding of the C ABI in include/a2a_exec.h (``_a2a_exec.so``).

There is no fallback: if the shared library is missing the import fails
loudly (build it with ``python -m paper_2309_13541_b200.build``).
"""
from __future__ import annotations

import ctypes as C
import os

__all__ = ["lib", "A2AOp", "ScheduleDesc", "GpuInfo", "LIB_PATH", "STATUS",
           "A2A_COPY_SELF", "A2A_EXEC_COUNT_LINKS"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_a2a_exec.so")

A2A_COPY_SELF = 1
A2A_INTERLEAVE = 2
A2A_REUSE_SCRATCH = 4
A2A_PROTO_LL = 8
A2A_PROTO_LL128 = 16
A2A_EXEC_COUNT_LINKS = 1
STATUS = {0: "OK", 1: "INVALID", 2: "EVAL", 3: "CUDA", 4: "TIMEOUT", 5: "STATE", 6: "NOMEM"}


class A2AOp(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("t", "src", "dst", "s", "d", "c0", "c1")]


class ScheduleDesc(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int32), ("n_steps", C.c_int32), ("q", C.c_int32),
        ("n_edges", C.c_int32), ("m_bytes", C.c_int64),
        ("edge_uv", C.POINTER(C.c_int32)), ("edge_cap", C.POINTER(C.c_double)),
        ("ops", C.POINTER(A2AOp)), ("n_ops", C.c_int64),
        ("node_gpu", C.POINTER(C.c_int32)), ("n_gpus", C.c_int32),
        ("flags", C.c_int32), ("split_bytes", C.c_int64),
    ]


class SchedHeader(C.Structure):
    _fields_ = [("n", C.c_int32), ("nsteps", C.c_int32), ("q", C.c_int32),
                ("mode", C.c_int32), ("chunk_bytes", C.c_double)]


class GpuInfo(C.Structure):
    _fields_ = [
        ("n_local_nodes", C.c_int32), ("first_node", C.c_int32),
        ("send_bytes", C.c_int64), ("recv_bytes", C.c_int64),
        ("scratch_bytes", C.c_int64), ("n_items", C.c_int64),
        ("hop_bytes", C.c_int64), ("egress_bytes", C.c_int64),
        ("ingress_bytes", C.c_int64), ("local_bytes", C.c_int64),
    ]


class SimParams(C.Structure):
    _fields_ = [(f, C.c_double) for f in ("nvlink_gbs", "hbm_gbs", "cta_gbs",
                                          "flag_us", "unit_us", "launch_us",
                                          "jitter", "unit_us_sys", "incast")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the B200 executor has no CPU fallback; "
            "build it with `python -m paper_2309_13541_b200.build`")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "a2a_load_schedule_xml": ([C.c_char_p, C.POINTER(SchedHeader), C.POINTER(P),
                                   C.POINTER(C.c_int64)], C.c_int),
        "a2a_lower_path_files": ([C.c_char_p, C.c_char_p, P, C.c_int32, C.c_int32,
                                  C.POINTER(SchedHeader), C.POINTER(P), C.POINTER(C.c_int64)],
                                 C.c_int),
        "a2a_save_schedule_table": ([C.c_char_p, C.POINTER(SchedHeader), P, C.c_int64], C.c_int),
        "a2a_load_schedule_table": ([C.c_char_p, C.POINTER(SchedHeader), C.POINTER(P),
                                     C.POINTER(C.c_int64)], C.c_int),
        "a2a_sha256_file": ([C.c_char_p, C.c_char_p], C.c_int),
        "a2a_free": ([P], None),
        "a2a_plan_create": ([C.POINTER(ScheduleDesc), C.POINTER(P)], C.c_int),
        "a2a_plan_destroy": ([P], C.c_int),
        "a2a_last_error": ([], C.c_char_p),
        "a2a_version": ([], C.c_char_p),
        "a2a_plan_model_time": ([P, C.c_double, C.c_double, C.c_double,
                                 C.POINTER(C.c_double)], C.c_int),
        "a2a_plan_link_bytes": ([P, C.POINTER(C.c_int64)], C.c_int),
        "a2a_plan_gpu_info": ([P, C.c_int32, C.POINTER(GpuInfo)], C.c_int),
        "a2a_plan_prepare": ([P, C.c_int32], C.c_int),
        "a2a_plan_sync_stats": ([P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "a2a_plan_emulate": ([P, C.c_int32, C.POINTER(P), C.POINTER(P), C.c_uint64], C.c_int),
        "a2a_plan_bind": ([P, C.c_int32, C.c_int32, C.c_int32], C.c_int),
        "a2a_plan_export_handle": ([P, C.c_void_p], C.c_int),
        "a2a_plan_import_handles": ([P, C.c_void_p], C.c_int),
        "a2a_plan_arena": ([P, C.POINTER(P)], C.c_int),
        "a2a_plan_import_pointers": ([P, C.POINTER(P)], C.c_int),
        "a2a_plan_close_peers": ([P], C.c_int),
        "a2a_plan_layout": ([P, C.POINTER(C.c_int64)], C.c_int),
        "a2a_plan_recv_buffer": ([P, C.POINTER(P)], C.c_int),
        "a2a_plan_execute": ([P, P, P, P, C.c_int32], C.c_int),
        "a2a_plan_sync": ([P], C.c_int),
        "a2a_plan_read_link_counters": ([P, C.POINTER(C.c_int64)], C.c_int),
        "a2a_plan_set_timeout": ([P, C.c_int64], C.c_int),
        "a2a_plan_set_recv_buffers": ([P, C.c_int32], C.c_int),
        "a2a_plan_recv_buffer_at": ([P, C.c_int32, C.POINTER(P)], C.c_int),
        "a2a_plan_read_timeline": ([P, C.POINTER(C.c_uint64), C.POINTER(C.c_int32)], C.c_int),
        "a2a_plan_set_sync_mode": ([P, C.c_int32], C.c_int),
        "a2a_optimize_placement": ([C.c_int32, C.c_int32, P, P, C.c_int32, C.c_int32,
                                    C.c_uint64, P], C.c_int),
        "a2a_plan_check_bounds": ([P, C.c_int32], C.c_int),
        "a2a_plan_set_split": ([P, C.c_int32], C.c_int),
        "a2a_plan_set_schedule": ([P, C.c_int32, C.c_int64], C.c_int),
        "a2a_plan_set_queue_split": ([P, C.c_int32], C.c_int),
        "a2a_plan_simulate": ([P, C.c_int32, C.POINTER(SimParams), C.POINTER(C.c_double)], C.c_int),
        "a2a_plan_dyn_stats": ([P, C.c_int32, C.c_int32, C.POINTER(C.c_int64),
                                C.POINTER(C.c_int64), C.POINTER(C.c_double)], C.c_int),
        "a2a_plan_set_engine": ([P, C.c_int32, C.c_int32, C.c_int32], C.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()
