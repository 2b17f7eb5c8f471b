"""Schedule types and the XML dialect, mirrored from ``a2aflow.schedule``.

``Instruction`` / ``ChunkedSchedule`` carry exactly the fields of reference
``src/schedule.py:49-72``; the XML reader/writer follow ``src/schedule.py:318-384``
(same element/attribute names, same parse-time rejects and messages), with
transparent ``.gz`` support so large frozen artifacts stay small in git.
Reference objects and these are interchangeable everywhere in this package.
"""
from __future__ import annotations

import gzip
import json
import xml.etree.ElementTree as ET
from dataclasses import dataclass, field

__all__ = ["ScheduleError", "Instruction", "ChunkedSchedule",
           "emit_schedule_xml", "parse_schedule_xml", "load_route_sidecar",
           "chunk_byte_offset"]


class ScheduleError(RuntimeError):
    pass


@dataclass(frozen=True)
class Instruction:
    """Chunks [c0, c1) of shard (s, d) cross link src->dst at step t.

    In ``mode="path"`` schedules ``dst`` is a route id and t == 0
    (reference src/schedule.py:49-62).
    """

    t: int
    src: int
    dst: int
    s: int
    d: int
    c0: int
    c1: int


@dataclass
class ChunkedSchedule:
    n: int
    nsteps: int
    chunk_bytes: float
    Q: int
    mode: str
    instructions: list = field(default_factory=list)


def chunk_byte_offset(c: int, m: int, Q: int) -> int:
    """First byte of chunk c of an m-byte shard split into Q chunks.

    The reference keeps ``chunk_bytes = m/Q`` as a float (src/schedule.py:297,
    src/evaluate.py:74); moving real bytes needs an integer rule.  Chunk c is
    bytes [floor(c*m/Q), floor((c+1)*m/Q)) — shared by the oracle, the plan
    builder (csrc/a2a_plan.cpp) and the device tables.
    """
    return (c * m) // Q


def _open(path, mode):
    return gzip.open(path, mode) if str(path).endswith(".gz") else open(path, mode)


def emit_schedule_xml(sched, path) -> None:
    root = ET.Element("schedule", {
        "n": str(sched.n), "nsteps": str(sched.nsteps),
        "chunkbytes": repr(float(sched.chunk_bytes)), "q": str(sched.Q),
        "mode": sched.mode})
    by_t: dict = {}
    for ins in sched.instructions:
        el = by_t.get(ins.t)
        if el is None:
            el = by_t[ins.t] = ET.SubElement(root, "step", {"t": str(ins.t)})
        ET.SubElement(el, "send", {
            "src": str(ins.src), "dst": str(ins.dst), "s": str(ins.s),
            "d": str(ins.d), "c0": str(ins.c0), "c1": str(ins.c1)})
    tree = ET.ElementTree(root)
    ET.indent(tree)
    with _open(path, "wb") as fh:
        tree.write(fh, encoding="utf-8", xml_declaration=True)


def _attr(el, name):
    v = el.get(name)
    if v is None:
        raise ScheduleError(f"missing attribute {name!r} on <{el.tag}>")
    return v


def parse_schedule_xml(path) -> ChunkedSchedule:
    """Parse the reference XML dialect; rejects exactly what
    src/schedule.py:349-384 rejects (malformed XML, wrong root, missing
    attributes, unknown mode, t outside [0, nsteps), bad chunk range)."""
    try:
        with _open(path, "rb") as fh:
            root = ET.parse(fh).getroot()
    except (ET.ParseError, EOFError, OSError) as ex:
        if isinstance(ex, FileNotFoundError):
            raise
        raise ScheduleError(f"malformed XML: {ex}") from ex
    if root.tag != "schedule":
        raise ScheduleError(f"root element is <{root.tag}>, not <schedule>")
    sched = ChunkedSchedule(
        n=int(_attr(root, "n")), nsteps=int(_attr(root, "nsteps")),
        chunk_bytes=float(_attr(root, "chunkbytes")), Q=int(_attr(root, "q")),
        mode=_attr(root, "mode"))
    if sched.mode not in ("ts", "path"):
        raise ScheduleError(f"unknown mode {sched.mode!r}")
    out = sched.instructions
    for step in root:
        if step.tag != "step":
            raise ScheduleError(f"unexpected element <{step.tag}>")
        t = int(_attr(step, "t"))
        if not 0 <= t < sched.nsteps:
            raise ScheduleError(f"step t={t} outside [0, {sched.nsteps})")
        for snd in step:
            if snd.tag != "send":
                raise ScheduleError(f"unexpected element <{snd.tag}>")
            ins = Instruction(t, int(_attr(snd, "src")), int(_attr(snd, "dst")),
                              int(_attr(snd, "s")), int(_attr(snd, "d")),
                              int(_attr(snd, "c0")), int(_attr(snd, "c1")))
            if not 0 <= ins.c0 < ins.c1 <= sched.Q:
                raise ScheduleError(f"bad chunk range [{ins.c0},{ins.c1})")
            out.append(ins)
    return sched


def load_route_sidecar(path) -> list:
    """The ``<out>.routes.json`` list `a2a compile --mode path` writes
    (reference src/cli.py:289-292): [{"s", "d", "nodes"}, ...], id = index."""
    with _open(path, "rt") as fh:
        return json.load(fh)["routes"]
