"""Cut-through fluid evaluation of a path schedule.

Restates the reference's ``eval_link_load`` (pkg/src/a2aflow/paths.py:535-553)
and ``eval_path_alltoall`` (pkg/src/a2aflow/evaluate.py:130-139) on the
reference's weighted-path-set file format (``load_routes``,
paths.py:576-584): per commodity the path weights are normalised to sum 1,
each path adds its share to every edge it uses, loads are divided by the edge
capacities; T = max load * m / b.  Same iteration order and float operations
as the reference, so the loads are bit-identical (tests/test_fluid.py checks
them against the reference's own numbers in tests/golden/golden.json).  This
is the per-link load reference the executor's device byte counters are
compared with (tests/test_mcf_link_loads.py), and the ``eval --routes`` path
of the CLI.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np

from .errors import EvalError, RouteError

__all__ = ["WeightedPathSet", "load_routes", "validate_path", "eval_link_load",
           "eval_path_alltoall"]


@dataclass
class WeightedPathSet:
    """(s, d) -> [(node tuple, weight)] (reference paths.py:60-69)."""
    paths: dict
    truncated: set = field(default_factory=set)


def load_routes(path: str) -> WeightedPathSet:
    """Reference route JSON ``{"routes": [{"s", "d", "paths": [{"nodes",
    "weight"}]}]}``; weights are exact fraction strings (paths.py:576-584)."""
    opener = open
    if path.endswith(".gz"):
        import gzip
        opener = gzip.open
    with opener(path, "rt") as fh:
        doc = json.load(fh)
    paths = {}
    for rec in doc["routes"]:
        paths[(rec["s"], rec["d"])] = [(tuple(p["nodes"]), float(Fraction(str(p["weight"]))))
                                       for p in rec["paths"]]
    return WeightedPathSet(paths=paths)


def validate_path(g, s: int, d: int, path) -> None:
    """Reference paths.py:49-57, same messages."""
    if path[0] != s or path[-1] != d:
        raise RouteError(f"path {path} does not join {s} -> {d}")
    if len(set(path)) != len(path):
        raise RouteError(f"path {path} is not simple")
    idx = g.edge_index
    for a, b in zip(path, path[1:]):
        if (a, b) not in idx:
            raise RouteError(f"path {path} uses nonexistent edge ({a},{b})")


def eval_link_load(g, wps) -> tuple:
    """(max normalised load, per-edge loads float64[E]) (paths.py:535-553)."""
    if hasattr(wps, "as_pathset"):          # a reference RouteTable: unit weights
        wps = wps.as_pathset()
    load = np.zeros(len(g.edges))
    idx = g.edge_index
    for (s, d), plist in wps.paths.items():
        tot = sum(w for _, w in plist)
        scale = 1.0 / tot if tot > 0 else 0.0
        for path, w in plist:
            validate_path(g, s, d, path)
            for a, b in zip(path, path[1:]):
                load[idx[(a, b)]] += w * scale
    norm = load / np.asarray([c for _, _, c in g.edges], dtype=float)
    return (float(norm.max()) if len(norm) else 0.0), norm


def eval_path_alltoall(g, wps, m: float = 1.0, b: float = 1.0) -> float:
    """Completion time in the cut-through fluid model (evaluate.py:130-139)."""
    for (s, d), plist in wps.paths.items():
        if sum(w for _, w in plist) <= 0:
            raise EvalError(f"commodity ({s},{d}) has zero total weight")
    max_load, _ = eval_link_load(g, wps)
    return max_load * m / b
