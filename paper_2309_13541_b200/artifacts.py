"""Frozen schedule artifacts (``artifacts/<config>/``) -> executor inputs.

The artifacts are the reference pipeline's own outputs (tools/gen_artifacts.py):
graph JSON, the ``mode="path"`` XML from compile_path_schedule and its route
sidecar.  Loading one yields the physical graph and the hop-indexed ``mode="ts"``
schedule the executor runs (lowering.lower_path_to_steps; augmented configs
are collapsed to physical nodes first).  Each file is checked against the
sha256 manifest.
"""
from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass

from .graphs import Digraph, NodeMapping, load_graph
from .lowering import collapse_aug_schedule, lower_path_to_steps
from .schedule import ChunkedSchedule, load_route_sidecar, parse_schedule_xml

__all__ = ["ARTIFACT_DIR", "Artifact", "load_artifact", "list_artifacts"]

ARTIFACT_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "artifacts")


@dataclass
class Artifact:
    name: str
    g: Digraph                     # physical graph the executor replays against
    sched: ChunkedSchedule         # hop-indexed ts schedule
    meta: dict
    routes: list | None = None     # physical routes (path configs)
    path_sched: ChunkedSchedule | None = None
    aug_graph: Digraph | None = None


def _find(d, base):
    for cand in (base, base + ".gz"):
        p = os.path.join(d, cand)
        if os.path.exists(p):
            return p
    return None


def _verify(d):
    with open(os.path.join(d, "manifest.json")) as fh:
        man = json.load(fh)
    for f, digest in man.items():
        h = hashlib.sha256()
        with open(os.path.join(d, f), "rb") as fh:
            for blk in iter(lambda: fh.read(1 << 20), b""):
                h.update(blk)
        if h.hexdigest() != digest:
            raise ValueError(f"artifact {d}/{f}: sha256 mismatch")


def list_artifacts() -> list:
    if not os.path.isdir(ARTIFACT_DIR):
        return []
    return sorted(x for x in os.listdir(ARTIFACT_DIR)
                  if os.path.exists(os.path.join(ARTIFACT_DIR, x, "manifest.json")))


def load_artifact(name: str, verify: bool = True, native: bool = False) -> Artifact:
    """Load a frozen artifact; ``native=True`` parses and lowers in C++
    (native_io) — identical ops, ~20x faster on GK(256,4)."""
    d = os.path.join(ARTIFACT_DIR, name)
    if verify:
        _verify(d)
    with open(os.path.join(d, "meta.json")) as fh:
        meta = json.load(fh)
    g = load_graph(_find(d, "graph.json"))
    if native:
        from .native_io import load_schedule_xml, lower_path_files
        if meta["kind"] == "ts":
            return Artifact(name, g, load_schedule_xml(_find(d, "ts.xml")), meta)
        nm = None
        if meta.get("host_capacity") is not None:
            nm = [x // 3 for x in range(3 * g.n)]
        ts = lower_path_files(_find(d, "path.xml"), _find(d, "path.xml.routes.json"),
                              node_map=nm, n_phys=g.n)
        return Artifact(name, g, ts, meta)
    if meta["kind"] == "ts":
        return Artifact(name, g, parse_schedule_xml(_find(d, "ts.xml")), meta)
    path_sched = parse_schedule_xml(_find(d, "path.xml"))
    routes = load_route_sidecar(_find(d, "path.xml.routes.json"))
    aug = None
    if meta.get("host_capacity") is not None:
        aug = load_graph(_find(d, "aug_graph.json"))
        n = g.n
        mp = NodeMapping(host=tuple(3 * v for v in range(n)),
                         nic_in=tuple(3 * v + 1 for v in range(n)),
                         nic_out=tuple(3 * v + 2 for v in range(n)))
        routes, path_sched = collapse_aug_schedule(routes, path_sched, mp)
    ts = lower_path_to_steps(routes, path_sched, n=g.n)
    return Artifact(name, g, ts, meta, routes=routes, path_sched=path_sched,
                    aug_graph=aug)
