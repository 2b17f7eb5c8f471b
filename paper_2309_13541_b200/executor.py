"""Host-side mirror of the reference executor interface.

Reference slot: ``a2aflow.evaluate.replay_timestep_schedule(g, sched, m=1.0,
b=1.0, sync_latency=0.0) -> (T, True)`` raising ``EvalError``
(pkg/src/a2aflow/evaluate.py:30-31, :56-127).  This module keeps that shape:

* ``replay_timestep_schedule(g, sched, m, b, sync_latency)`` — same signature,
  same result, same error texts; validation and the modelled T are computed by
  the native plan builder (csrc/a2a_plan.cpp) instead of Python sets.
* ``execute_timestep_schedule(g, sched, send, recv, ...) -> (T_measured, True)``
  — the byte-moving B200 execution of the same schedule on one GPU.
* ``Plan`` — the reusable handle (validate once, bind to a GPU, execute many
  times; multi-GPU via CUDA IPC handles, see ``dist.py``).

Everything accepts the reference's own ``Digraph`` / ``ChunkedSchedule``
objects as well as this package's mirrors (duck typing on ``n``, ``edges``,
``nsteps``, ``Q``, ``mode``, ``instructions``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N
from .errors import EvalError

__all__ = ["EvalError", "ExecutorError", "Plan", "replay_timestep_schedule",
           "execute_timestep_schedule", "contiguous_placement", "timeline_summary"]


def timeline_summary(tl: np.ndarray, schedule: str | None = "static") -> dict:
    """Kernel-internal timing from Plan.read_timeline() (columns: start, entry,
    step published [T'], exit, step dependencies acquired [T']): microseconds
    from the earliest CTA start.  Dynamic schedules store per-CTA unit counts
    and flag-wait nanoseconds in columns 2 and 3 instead of step stamps."""
    T = (tl.shape[1] - 3) // 2
    t0 = int(tl[:, 0].min())
    us = lambda x: round((int(x) - t0) / 1e3, 3)  # noqa: E731
    if schedule and schedule.split(":")[0] in ("dynamic", "list", "cp", "mix", "ready", "spread", "chain", "chaind"):
        units = tl[:, 2].astype(np.int64)
        return {"kernel_us": us(tl[:, 2 + T].max()), "start_spread_us": us(tl[:, 0].max()),
                "entry_us": us(tl[:, 1].max()), "units_per_cta": [int(units.min()), int(units.max())],
                "max_cta_wait_us": round(int(tl[:, 3].max()) / 1e3, 3)}

    def last(j):
        col = tl[:, j][tl[:, j] > 0]
        return us(col.max()) if col.size else None
    return {"kernel_us": us(tl[:, 2 + T].max()), "start_spread_us": us(tl[:, 0].max()),
            "entry_us": us(tl[:, 1].max()),
            "step_acquired_us": [last(3 + T + t) for t in range(T)],
            "step_done_us": [last(2 + t) for t in range(T)]}


class ExecutorError(RuntimeError):
    """Device-side failure: CUDA error, flag-wait timeout, bad call order."""


def _raise(rc: int, what: str):
    msg = N.lib.a2a_last_error().decode()
    if rc == 2:
        raise EvalError(msg)
    if rc == 1:
        raise ValueError(f"{what}: {msg}")
    raise ExecutorError(f"{what}: [{N.STATUS.get(rc, rc)}] {msg}")


def contiguous_placement(n: int, n_gpus: int) -> list:
    """Virtual node v -> GPU v*G//n: contiguous blocks (u // (N/G) when G | N),
    i.e. subcubes for the hypercube and 1x2x4 slabs for the 4x4x4 torus."""
    return [v * n_gpus // n for v in range(n)]


def _ops_array(instructions) -> np.ndarray:
    if isinstance(instructions, np.ndarray):
        return np.ascontiguousarray(instructions, dtype=np.int32).reshape(-1, 7)
    arr = np.fromiter((x for i in instructions
                       for x in (i.t, i.src, i.dst, i.s, i.d, i.c0, i.c1)),
                      dtype=np.int64, count=7 * len(instructions))
    if arr.size and (arr.min() < -2**31 or arr.max() >= 2**31):
        raise ValueError("instruction field does not fit int32")
    return arr.astype(np.int32).reshape(-1, 7)


def _check_mode(g, sched):
    # evaluate.py:70-73
    if sched.mode != "ts":
        raise EvalError("replay_timestep_schedule expects a ts-mode schedule")
    if g.n != sched.n:
        raise EvalError(f"graph has {g.n} nodes, schedule says {sched.n}")


class Plan:
    """Validated, laid-out execution plan of one ts schedule at shard size m."""

    def __init__(self, g, sched, m: int, placement=None, n_gpus: int = 1,
                 copy_self: bool = True, ops: np.ndarray | None = None,
                 order: str | None = None, split_bytes: int = 0,
                 reuse_scratch: bool | None = None, protocol: str | None = None):
        _check_mode(g, sched)
        if int(m) != m or m < 0:
            raise ValueError(f"shard size m must be a non-negative integer, got {m}")
        self.n, self.nsteps, self.Q, self.m = g.n, sched.nsteps, sched.Q, int(m)
        self.n_gpus = int(n_gpus)
        self.E = len(g.edges)
        self._edge_uv = np.ascontiguousarray(
            [(u, v) for u, v, _ in g.edges], dtype=np.int32).reshape(-1, 2)
        self._cap = np.ascontiguousarray([c for _, _, c in g.edges], dtype=np.float64)
        if ops is None:
            ops = getattr(sched, "ops_array", None)   # native-loaded schedules
        self._ops = _ops_array(sched.instructions if ops is None else ops)
        if placement is None or placement == "contiguous":
            placement = contiguous_placement(self.n, self.n_gpus)
        elif placement == "optimized":
            from .placement import optimized_placement
            placement = optimized_placement(g, sched, self.n_gpus, m=max(int(m), sched.Q))
        self.placement = np.ascontiguousarray(placement, dtype=np.int32)
        if self.placement.shape != (self.n,):
            raise ValueError("placement must list one GPU per node")
        d = N.ScheduleDesc()
        d.n_nodes, d.n_steps, d.q, d.n_edges = self.n, self.nsteps, self.Q, self.E
        d.m_bytes = self.m
        d.edge_uv = self._edge_uv.ctypes.data_as(C.POINTER(C.c_int32))
        d.edge_cap = self._cap.ctypes.data_as(C.POINTER(C.c_double))
        d.ops = self._ops.ctypes.data_as(C.POINTER(N.A2AOp))
        d.n_ops = self._ops.shape[0]
        d.node_gpu = self.placement.ctypes.data_as(C.POINTER(C.c_int32))
        d.n_gpus = self.n_gpus
        if order is None:
            order = os.environ.get("A2A_ORDER", "grouped")
        if order not in ("grouped", "interleaved"):
            raise ValueError("order must be 'grouped' or 'interleaved'")
        self.order = order
        if reuse_scratch is None:
            reuse_scratch = os.environ.get("A2A_REUSE_SCRATCH", "0") == "1"
        self.reuse_scratch = bool(reuse_scratch)
        # transport: "simple" (peer stores + release/acquire flags), "ll" (16-byte
        # {data, epoch} lines polled by the receiving GPU; small shards) or
        # "ll128" (128-byte lines, 120 payload bytes + epoch flag; medium shards)
        if protocol is None:
            protocol = os.environ.get("A2A_PROTO", "simple").strip().lower() or "simple"
        if protocol not in ("simple", "ll", "ll128"):
            raise ValueError("protocol must be 'simple', 'll' or 'll128'")
        self.protocol = protocol
        d.flags = (N.A2A_COPY_SELF if copy_self else 0) | \
            (N.A2A_INTERLEAVE if order == "interleaved" else 0) | \
            (N.A2A_REUSE_SCRATCH if reuse_scratch else 0) | \
            (N.A2A_PROTO_LL if protocol == "ll" else 0) | \
            (N.A2A_PROTO_LL128 if protocol == "ll128" else 0)
        d.split_bytes = int(split_bytes)
        h = C.c_void_p()
        rc = N.lib.a2a_plan_create(C.byref(d), C.byref(h))
        if rc:
            _raise(rc, "a2a_plan_create")
        self._h = h
        self.rank = None
        self.device = None
        self.engine = None
        self._bufcheck = None
        self._num_ctas = 0
        self.schedule = None

    # ---- lifetime
    def close(self):
        if getattr(self, "_h", None):
            N.lib.a2a_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _ck(self, rc, what):
        if rc:
            _raise(rc, what)

    # ---- host-side queries
    def model_time(self, m: float | None = None, b: float = 1.0,
                   sync_latency: float = 0.0) -> float:
        """replay_timestep_schedule's T for (m, b, sync) — bit-identical."""
        out = C.c_double()
        self._ck(N.lib.a2a_plan_model_time(self._h, float(self.m if m is None else m),
                                           float(b), float(sync_latency), C.byref(out)),
                 "a2a_plan_model_time")
        return out.value

    def link_bytes(self) -> np.ndarray:
        """Schedule bytes per (step, edge id), int64 [nsteps, E]."""
        out = np.zeros((self.nsteps, self.E), dtype=np.int64)
        self._ck(N.lib.a2a_plan_link_bytes(self._h, out.ctypes.data_as(C.POINTER(C.c_int64))),
                 "a2a_plan_link_bytes")
        return out

    def gpu_info(self, gpu: int) -> dict:
        info = N.GpuInfo()
        self._ck(N.lib.a2a_plan_gpu_info(self._h, int(gpu), C.byref(info)), "a2a_plan_gpu_info")
        return {f: getattr(info, f) for f, _ in N.GpuInfo._fields_}

    def prepare(self, num_ctas: int):
        """Build the CTA split and exact producer-dependency lists (host only)."""
        self._ck(N.lib.a2a_plan_prepare(self._h, int(num_ctas)), "a2a_plan_prepare")
        return self

    def check_bounds(self, num_ctas: int = 148):
        """Host audit of every device copy range against its buffer (raises)."""
        self._ck(N.lib.a2a_plan_check_bounds(self._h, int(num_ctas)), "a2a_plan_check_bounds")
        return True

    def set_split(self, remote_weight: int):
        """Before bind: cost weight of an NVLink byte in the static CTA split."""
        self._ck(N.lib.a2a_plan_set_split(self._h, int(remote_weight)), "a2a_plan_set_split")
        self.remote_weight = int(remote_weight)
        return self

    def set_schedule(self, mode: str = "static", unit_bytes: int = 0):
        """Before bind: "static" per-CTA step programs, or unit queues (SURVEY
        §8f f2) of ~unit_bytes units (0 = auto): "dynamic" (step-major,
        readiness model), "list" (event-driven order), "cp" (critical-path
        priority), "mix" (one queue, NVLink/HBM merged), "ready" (units enqueued
        by their last producer), "spread" ("mix" with the NVLink units of a step
        interleaved over their destination GPUs), "chain" ("mix" order, but each
        route's consecutive local hops run back to back on one CTA, streaming
        through L2 with no flag between them), "chaind" ("chain", and each task
        then discards its dead intermediate scratch lines from L2 instead of
        writing them back).  LL plans run "static" only."""
        code = {"static": 0, "dynamic": 1, "list": 2, "cp": 3, "mix": 4, "ready": 5,
                "spread": 6, "chain": 7, "chaind": 8}[mode]
        self._ck(N.lib.a2a_plan_set_schedule(self._h, code, int(unit_bytes)), "a2a_plan_set_schedule")
        self.schedule = mode
        return self

    def set_schedule_spec(self, spec: str):
        """Before bind: "<mode>[:<unit bytes>[:<pinned NVLink CTAs>]]", e.g.
        "static", "cp:1048576", "cp:1048576:64" (set_schedule + set_queue_split)."""
        mode, *rest = spec.strip().split(":")
        if len(rest) > 2:
            raise ValueError(f"bad schedule spec {spec!r}")
        self.set_schedule(mode, int(rest[0]) if rest else 0)
        if len(rest) > 1:
            self.set_queue_split(int(rest[1]))
        return self

    def set_queue_split(self, remote_ctas: int = 0):
        """Before bind (two-queue orders "dynamic" / "list" / "cp"): pin
        `remote_ctas` CTAs to the NVLink queue and the rest to the HBM queue, no
        queue switching (0 = automatic split)."""
        self._ck(N.lib.a2a_plan_set_queue_split(self._h, int(remote_ctas)),
                 "a2a_plan_set_queue_split")
        self.remote_ctas = int(remote_ctas)
        return self

    # fluid-model defaults, calibrated on measured 1/2/4-GPU runs (tools/sim_calibrate.py)
    SIM_DEFAULTS = {"nvlink_gbs": 705.0, "hbm_gbs": 6538.9, "cta_gbs": 40.0,
                    "flag_us": 2.0, "unit_us": 1.0, "launch_us": 8.0, "jitter": 0.1,
                    "unit_us_sys": 10.0, "incast": 0.0}

    def simulate(self, num_ctas: int = 148, **params) -> float:
        """Modelled seconds of one execute of the selected execution schedule
        (a2a_plan_simulate; host only, any G -- e.g. 8 GPUs from a CPU box)."""
        p = dict(self.SIM_DEFAULTS, **params)
        sp = N.SimParams(**p)
        out = C.c_double()
        self._ck(N.lib.a2a_plan_simulate(self._h, int(num_ctas), C.byref(sp), C.byref(out)),
                 "a2a_plan_simulate")
        return out.value

    def dyn_stats(self, gpu: int, num_ctas: int) -> dict:
        nu, nw, est = C.c_int64(), C.c_int64(), C.c_double()
        self._ck(N.lib.a2a_plan_dyn_stats(self._h, int(gpu), int(num_ctas), C.byref(nu),
                                          C.byref(nw), C.byref(est)), "a2a_plan_dyn_stats")
        return {"units": nu.value, "wait_entries": nw.value, "model_makespan_s": est.value}

    def sync_stats(self, gpu: int) -> dict:
        w, e = C.c_int64(), C.c_int64()
        self._ck(N.lib.a2a_plan_sync_stats(self._h, int(gpu), C.byref(w), C.byref(e)),
                 "a2a_plan_sync_stats")
        return {"wait_flags": w.value, "exit_flags": e.value}

    def emulate(self, sends, num_ctas: int, seed: int = 0) -> list:
        """Host emulation of the device protocol (CPU): every GPU's CTAs run in a
        random interleaving constrained only by the dependency lists.
        sends: per GPU uint8 arrays [V_g, N, m]; returns per GPU recv arrays."""
        if len(sends) != self.n_gpus:
            raise ValueError("one send array per GPU")
        sends = [np.ascontiguousarray(x, dtype=np.uint8) for x in sends]
        recvs = [np.zeros_like(x) for x in sends]
        for g, x in enumerate(sends):
            if x.nbytes != self.gpu_info(g)["send_bytes"]:
                raise ValueError(f"send[{g}] has the wrong size")
        sp = (C.c_void_p * self.n_gpus)(*[x.ctypes.data for x in sends])
        rp = (C.c_void_p * self.n_gpus)(*[x.ctypes.data for x in recvs])
        self._ck(N.lib.a2a_plan_emulate(self._h, int(num_ctas), sp, rp, int(seed)),
                 "a2a_plan_emulate")
        return recvs

    # ---- device side
    def set_engine(self, engine: str = "lsu", tma_chunk: int = 0, tma_stages: int = 0):
        """Copy engine before bind: "tma" (cp.async.bulk ring, the default) or
        "lsu" (SM 128-bit loads/stores).  Default from $A2A_ENGINE, else "tma"."""
        code = {"lsu": 0, "tma": 1}[engine]
        self._ck(N.lib.a2a_plan_set_engine(self._h, code, int(tma_chunk), int(tma_stages)),
                 "a2a_plan_set_engine")
        self.engine = engine
        return self

    def bind(self, gpu: int = 0, device: int | None = None, num_ctas: int = 0):
        device = gpu if device is None else device
        # environment overrides for experiments (explicit setters win)
        if self.engine is None:
            env = os.environ.get("A2A_ENGINE", "").strip().lower()
            if env:
                parts = env.split(":")      # tma[:chunk[:stages]]
                self.set_engine(parts[0], *(int(x) for x in parts[1:]))
        if self.schedule is None and os.environ.get("A2A_SCHED"):
            self.set_schedule_spec(os.environ["A2A_SCHED"])
        if os.environ.get("A2A_SPLIT_W") and getattr(self, "remote_weight", None) is None:
            self.set_split(int(os.environ["A2A_SPLIT_W"]))
        if os.environ.get("A2A_SYNC_MODE"):
            self.set_sync_mode(int(os.environ["A2A_SYNC_MODE"]))
        self._ck(N.lib.a2a_plan_bind(self._h, int(gpu), int(device), int(num_ctas)),
                 "a2a_plan_bind")
        self._num_ctas = int(num_ctas)
        self._bufcheck = None
        self.rank, self.device = int(gpu), int(device)
        return self

    def export_handle(self) -> bytes:
        buf = C.create_string_buffer(64)
        self._ck(N.lib.a2a_plan_export_handle(self._h, buf), "a2a_plan_export_handle")
        return buf.raw

    def import_handles(self, handles):
        blob = b"".join(bytes(h) for h in handles)
        if len(blob) != 64 * self.n_gpus:
            raise ValueError("need one 64-byte handle per GPU")
        buf = C.create_string_buffer(blob, len(blob))
        self._ck(N.lib.a2a_plan_import_handles(self._h, buf), "a2a_plan_import_handles")

    def arena_ptr(self) -> int:
        p = C.c_void_p()
        self._ck(N.lib.a2a_plan_arena(self._h, C.byref(p)), "a2a_plan_arena")
        return p.value

    def close_peers(self):
        """Multi-GPU teardown phase 1 (a2a_plan_close_peers): wait for this
        rank's executes and unmap the peers' arenas.  Every rank must get here
        before any rank calls ``close()`` (see dist.disconnect)."""
        if getattr(self, "_h", None):
            self._ck(N.lib.a2a_plan_close_peers(self._h), "a2a_plan_close_peers")

    def layout(self) -> dict:
        """Device-layout parameters every rank must agree on (after bind)."""
        out = (C.c_int64 * 8)()
        self._ck(N.lib.a2a_plan_layout(self._h, out), "a2a_plan_layout")
        keys = ("num_ctas", "sched_mode", "dyn_unit_bytes", "n_recv", "flags_bytes",
                "arena_bytes_total", "engine", "protocol_ll")
        return dict(zip(keys, list(out)))

    def import_pointers(self, ptrs):
        arr = (C.c_void_p * self.n_gpus)(*ptrs)
        self._ck(N.lib.a2a_plan_import_pointers(self._h, arr), "a2a_plan_import_pointers")

    def set_recv_buffers(self, count: int):
        """Before bind: arena recv buffers to alternate between (1..4)."""
        self._ck(N.lib.a2a_plan_set_recv_buffers(self._h, int(count)), "a2a_plan_set_recv_buffers")
        return self

    def recv_buffer(self, index: int = 0):
        """torch uint8 view [V_g, N, m] of this rank's arena recv buffer `index`
        (plan-owned memory: valid until ``close()``)."""
        import torch
        p = C.c_void_p()
        self._ck(N.lib.a2a_plan_recv_buffer_at(self._h, int(index), C.byref(p)),
                 "a2a_plan_recv_buffer_at")
        V = self.gpu_info(self.rank)["n_local_nodes"]
        return _device_tensor(p.value, (V, self.n, self.m), self.device, torch)

    def set_sync_mode(self, mode: int):
        """Step-flag publication variant (see a2a_plan_set_sync_mode)."""
        self._ck(N.lib.a2a_plan_set_sync_mode(self._h, int(mode)), "a2a_plan_set_sync_mode")
        return self

    def set_timeout(self, seconds: float):
        self._ck(N.lib.a2a_plan_set_timeout(self._h, int(seconds * 1e9)), "a2a_plan_set_timeout")

    def execute(self, send, recv=None, stream=None, count_links: bool = False):
        """Launch one all-to-all (asynchronous on ``stream``, default: current)."""
        import torch
        if self.rank is None:
            raise ExecutorError("a2a_plan_execute: [STATE] plan not bound to a device")
        ck = self._bufcheck
        if ck is None:
            info = self.gpu_info(self.rank)
            ck = self._bufcheck = (info["send_bytes"], info["recv_bytes"])
        _check_buf(send, ck[0], self.device, "send", torch)
        rp = None
        if recv is not None:
            _check_buf(recv, ck[1], self.device, "recv", torch)
            rp = recv.data_ptr()
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        rc = N.lib.a2a_plan_execute(self._h, send.data_ptr(), rp, sp,
                                    N.A2A_EXEC_COUNT_LINKS if count_links else 0)
        if rc:
            _raise(rc, "a2a_plan_execute")

    def read_timeline(self) -> np.ndarray:
        """Per-CTA %globaltimer stamps of the last execute, uint64 [nC, T'+3]:
        start, entry barrier passed, step t published (0 = idle), exit."""
        cols = C.c_int32()
        self._ck(N.lib.a2a_plan_read_timeline(self._h, None, C.byref(cols)), "a2a_plan_read_timeline")
        n_cta = self._n_ctas()
        out = np.zeros((n_cta, cols.value), dtype=np.uint64)
        self._ck(N.lib.a2a_plan_read_timeline(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)),
                                              C.byref(cols)), "a2a_plan_read_timeline")
        return out

    def _n_ctas(self):
        if self._num_ctas:
            return self._num_ctas
        import torch
        return torch.cuda.get_device_properties(self.device).multi_processor_count

    def sync(self):
        self._ck(N.lib.a2a_plan_sync(self._h), "a2a_plan_sync")

    def read_link_counters(self) -> np.ndarray:
        """Device-counted bytes per (step, edge) this rank moved since the last read."""
        out = np.zeros((self.nsteps, self.E), dtype=np.int64)
        self._ck(N.lib.a2a_plan_read_link_counters(
            self._h, out.ctypes.data_as(C.POINTER(C.c_int64))), "a2a_plan_read_link_counters")
        return out


class _CAI:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def _device_tensor(ptr, shape, device, torch):
    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(ptr, shape), device=f"cuda:{device}")


def _check_buf(t, nbytes, device, name, torch):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.device.index != device:
        raise ValueError(f"{name} is on {t.device}, plan is bound to cuda:{device}")
    if t.dtype != torch.uint8 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous uint8 tensor")
    if t.numel() != nbytes:
        raise ValueError(f"{name} has {t.numel()} bytes, plan needs {nbytes}")


def replay_timestep_schedule(g, sched, m: float = 1.0, b: float = 1.0,
                             sync_latency: float = 0.0):
    """Drop-in for the reference's symbolic replay: (T, True) or EvalError.

    Same validation order and messages and a bit-identical T
    (evaluate.py:56-127), computed natively; no GPU needed.
    """
    with Plan(g, sched, m=0, copy_self=False) as p:
        return p.model_time(m=m, b=b, sync_latency=sync_latency), True


def execute_timestep_schedule(g, sched, send, recv=None, num_ctas: int = 0,
                              copy_self: bool = True):
    """Execute the schedule on real bytes on one GPU: (T_seconds, True).

    send: CUDA uint8 tensor [N, N, m] (send[s, d] = shard (s, d));
    recv: same shape (allocated if None), recv[d, s] = shard (s, d) after the
    call.  T is the measured device time of the all-to-all (CUDA events).
    """
    import torch
    n = g.n
    if send.numel() % (n * n):
        raise ValueError("send must hold N*N shards")
    m = send.numel() // (n * n)
    if recv is None:
        recv = torch.empty_like(send)
    with Plan(g, sched, m=m, copy_self=copy_self) as p:
        p.bind(0, device=send.device.index, num_ctas=num_ctas)
        stream = torch.cuda.current_stream(send.device)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        p.execute(send, recv, stream=stream)
        e1.record(stream)
        p.sync()
        e1.synchronize()
        return e0.elapsed_time(e1) / 1e3, True
