"""ORACLE — ctypes wrapper of oracle/replay_bytes.c (test / CPU-baseline only).

Same contract as oracle/replay_bytes.replay_bytes (pinned to the reference by
tests/test_oracle.py), multi-threaded; built by
``python -m paper_2309_13541_b200.build`` into oracle/_build/.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liboracle_replay.so")
_lib = None


class OracleEvalError(RuntimeError):
    pass


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing; run python -m paper_2309_13541_b200.build")
        L = C.CDLL(LIB)
        L.oracle_replay.restype = C.c_int
        P = C.c_void_p
        L.oracle_replay.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int, P, P, P,
                                    C.c_int64, P, P, C.c_int, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.POINTER(C.c_double), P, C.c_char_p, C.c_int]
        L.oracle_replay_ws.restype = C.c_int
        L.oracle_replay_ws.argtypes = L.oracle_replay.argtypes + [P, C.c_int64]
        _lib = L
    return _lib


def ops_array(sched):
    return np.array([(i.t, i.src, i.dst, i.s, i.d, i.c0, i.c1) for i in sched.instructions],
                    dtype=np.int32).reshape(-1, 7)


def workspace(sched, n, m, ops=None) -> np.ndarray:
    """Scratch for repeated replays (oracle_replay_ws): one m-byte slot per
    distinct forwarding location (holder dst != d, shard (s, d)) of the
    schedule, pre-touched so no replay page-faults it."""
    ops = ops_array(sched) if ops is None else ops
    o = ops[(ops[:, 0] >= 0) & (ops[:, 0] < sched.nsteps) & (ops[:, 5] < ops[:, 6]) & (ops[:, 2] != ops[:, 4])]
    keys = (o[:, 2].astype(np.int64) * n + o[:, 3]) * n + o[:, 4]
    ws = np.empty(max(1, len(np.unique(keys)) * m), dtype=np.uint8)
    ws.fill(0)
    return ws


def replay_bytes_c(g, sched, send, m, nthreads=None, copy_self=True, m_model=None,
                   b=1.0, sync_latency=0.0, recv=None, ops=None, ws=None):
    """(T, recv [N,N,m] uint8, link_bytes [T,E] int64); raises OracleEvalError.
    ``ws``: optional scratch from ``workspace`` reused across calls."""
    L = _load()
    if sched.mode != "ts":
        raise OracleEvalError("replay_timestep_schedule expects a ts-mode schedule")
    if g.n != sched.n:
        raise OracleEvalError(f"graph has {g.n} nodes, schedule says {sched.n}")
    n = g.n
    send = np.ascontiguousarray(send, dtype=np.uint8).reshape(n, n, m)
    if recv is None:
        recv = np.zeros_like(send)
    uv = np.ascontiguousarray([(u, v) for u, v, _ in g.edges], dtype=np.int32).reshape(-1, 2)
    cap = np.ascontiguousarray([c for _, _, c in g.edges], dtype=np.float64)
    ops = ops_array(sched) if ops is None else ops
    lb = np.zeros((sched.nsteps, len(g.edges)), dtype=np.int64)
    T = C.c_double()
    err = C.create_string_buffer(512)
    nthreads = nthreads or os.cpu_count() or 1
    args = (n, sched.nsteps, sched.Q, m, len(g.edges), uv.ctypes.data,
            cap.ctypes.data, ops.ctypes.data, ops.shape[0], send.ctypes.data,
            recv.ctypes.data, nthreads, 1 if copy_self else 0,
            float(m if m_model is None else m_model), b, sync_latency,
            C.byref(T), lb.ctypes.data, err, 512)
    if ws is None:
        rc = L.oracle_replay(*args)
    else:
        rc = L.oracle_replay_ws(*args, ws.ctypes.data, ws.nbytes)
    if rc == 2:
        raise OracleEvalError(err.value.decode())
    if rc:
        raise RuntimeError(err.value.decode())
    return T.value, recv, lb
