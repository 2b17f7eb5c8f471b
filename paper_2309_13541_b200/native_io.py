"""Native loader front-end: reference XML / route sidecar
files -> ChunkedSchedule backed by an int32 op table, parsed in C++
(csrc/a2a_io.cpp).  Same rejects and messages as schedule.parse_schedule_xml."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .schedule import ChunkedSchedule, Instruction, ScheduleError

__all__ = ["load_schedule_xml", "lower_path_files", "OpTableSchedule"]


class OpTableSchedule(ChunkedSchedule):
    """ChunkedSchedule whose instructions live in ``ops_array`` (int32 [K, 7]);
    ``instructions`` is materialised on first access only."""

    def __init__(self, n, nsteps, chunk_bytes, Q, mode, ops_array):
        super().__init__(n=n, nsteps=nsteps, chunk_bytes=chunk_bytes, Q=Q, mode=mode,
                         instructions=None)
        self.ops_array = ops_array

    def __getattribute__(self, name):
        if name == "instructions":
            d = object.__getattribute__(self, "__dict__")
            if d.get("instructions") is None:
                d["instructions"] = [Instruction(*map(int, r)) for r in d["ops_array"]]
            return d["instructions"]
        return object.__getattribute__(self, name)


def _take(hdr, ptr, count):
    try:
        arr = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_int32)), shape=(count.value, 7)).copy() \
            if count.value else np.zeros((0, 7), dtype=np.int32)
    finally:
        N.lib.a2a_free(ptr)
    return OpTableSchedule(hdr.n, hdr.nsteps, hdr.chunk_bytes, hdr.q,
                           "ts" if hdr.mode == 0 else "path", arr)


def _err(rc):
    msg = N.lib.a2a_last_error().decode()
    if rc == 2:
        raise ScheduleError(msg)
    raise ValueError(msg)


def load_schedule_xml(path) -> OpTableSchedule:
    hdr, ptr, cnt = N.SchedHeader(), C.c_void_p(), C.c_int64()
    rc = N.lib.a2a_load_schedule_xml(str(path).encode(), C.byref(hdr), C.byref(ptr), C.byref(cnt))
    if rc:
        _err(rc)
    return _take(hdr, ptr, cnt)


def lower_path_files(xml_path, routes_path, node_map=None, n_phys: int = 0) -> OpTableSchedule:
    """Hop-indexed ts schedule straight from `path.xml` + `.routes.json`."""
    hdr, ptr, cnt = N.SchedHeader(), C.c_void_p(), C.c_int64()
    nm = None
    if node_map is not None:
        nm = np.ascontiguousarray(node_map, dtype=np.int32)
    rc = N.lib.a2a_lower_path_files(str(xml_path).encode(), str(routes_path).encode(),
                                    None if nm is None else nm.ctypes.data,
                                    0 if nm is None else len(nm), int(n_phys),
                                    C.byref(hdr), C.byref(ptr), C.byref(cnt))
    if rc:
        _err(rc)
    return _take(hdr, ptr, cnt)
