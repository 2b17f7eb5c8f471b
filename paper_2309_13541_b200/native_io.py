"""Native loader front-end: reference XML / route sidecar
files -> ChunkedSchedule backed by an int32 op table, parsed in C++
(csrc/a2a_io.cpp).  Same rejects and messages as schedule.parse_schedule_xml.

Also the binary op table (``save_schedule_table`` / ``load_schedule_table``,
format in csrc/a2a_io.cpp): a parsed or lowered schedule with a SHA-256
trailer, reloaded without XML parsing, and ``sha256_file`` for the reference's
run-manifest digests (reference src/cli.py:30-55)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .schedule import ChunkedSchedule, Instruction, ScheduleError

__all__ = ["load_schedule_xml", "lower_path_files", "OpTableSchedule", "save_schedule_table",
           "load_schedule_table", "load_schedule", "is_schedule_table", "sha256_file"]

TABLE_MAGIC = b"A2ATBL1\n"


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


def _ops_of(sched) -> np.ndarray:
    arr = getattr(sched, "ops_array", None)
    if arr is None:
        arr = np.array([(i.t, i.src, i.dst, i.s, i.d, i.c0, i.c1) for i in sched.instructions],
                       dtype=np.int64).reshape(-1, 7)
        if arr.size and (arr.min() < -2**31 or arr.max() >= 2**31):
            raise ValueError("instruction field does not fit int32")
    return np.ascontiguousarray(arr, dtype=np.int32).reshape(-1, 7)


def save_schedule_table(sched, path) -> None:
    """Write ``sched`` (this package's or the reference's ChunkedSchedule) as a
    binary op table; rejects what load_schedule_xml would reject."""
    if sched.mode not in ("ts", "path"):
        raise ScheduleError(f"unknown mode '{sched.mode}'")
    hdr = N.SchedHeader(int(sched.n), int(sched.nsteps), int(sched.Q),
                        0 if sched.mode == "ts" else 1, float(sched.chunk_bytes))
    ops = _ops_of(sched)
    rc = N.lib.a2a_save_schedule_table(str(path).encode(), C.byref(hdr),
                                       ops.ctypes.data if ops.size else None, ops.shape[0])
    if rc:
        _err(rc)


def load_schedule_table(path) -> OpTableSchedule:
    hdr, ptr, cnt = N.SchedHeader(), C.c_void_p(), C.c_int64()
    rc = N.lib.a2a_load_schedule_table(str(path).encode(), C.byref(hdr), C.byref(ptr), C.byref(cnt))
    if rc:
        _err(rc)
    return _take(hdr, ptr, cnt)


def is_schedule_table(path) -> bool:
    import gzip
    with open(path, "rb") as fh:
        head = fh.read(len(TABLE_MAGIC))
    if head[:2] == b"\x1f\x8b":                      # gzip: the loader reads it transparently
        with gzip.open(path, "rb") as fh:
            head = fh.read(len(TABLE_MAGIC))
    return head == TABLE_MAGIC


def load_schedule(path) -> OpTableSchedule:
    """A schedule file of either form: binary op table or reference XML (+gz)."""
    return load_schedule_table(path) if is_schedule_table(path) else load_schedule_xml(path)


def sha256_file(path) -> str:
    out = C.create_string_buffer(65)
    rc = N.lib.a2a_sha256_file(str(path).encode(), out)
    if rc:
        _err(rc)
    return out.value.decode()
