"""Topology model for the executor's drop-in side.

A from-scratch restatement of the parts of ``a2aflow.graphs`` the executor
needs.  The contract that matters is the one the
reference's replay relies on: a frozen capacitated digraph whose edge list is
sorted by (u, v), with parallel edges merged and self-loops / zero-capacity
edges dropped, so that an edge id is its position
(reference ``src/graphs.py:67-86``).  Every object here is duck-type
compatible with the reference ``Digraph`` (``n``, ``edges``, ``edge_index``,
``capacities``, ``out_adj``), so a reference graph can be passed to the
executor directly and vice versa.
"""
from __future__ import annotations

import gzip
import json
from collections import deque
from dataclasses import dataclass, field
from fractions import Fraction
from functools import cached_property

__all__ = [
    "GraphError", "Digraph", "NodeMapping", "gen_torus", "gen_hypercube",
    "gen_gen_kautz", "augment_host_bottleneck", "all_pairs_distances",
    "distance_sum", "load_graph", "save_graph",
]


class GraphError(ValueError):
    """Malformed graph input (mirrors a2aflow.graphs.GraphError)."""


@dataclass(frozen=True)
class Digraph:
    """Immutable capacitated digraph; ``edges`` = sorted ((u, v, cap), ...).

    Mirrors reference ``src/graphs.py:42-115``.
    """

    n: int
    edges: tuple
    meta: dict = field(default_factory=dict, compare=False)

    def __post_init__(self):
        if self.n < 1:
            raise GraphError(f"node count must be >= 1, got {self.n}")
        seen = set()
        for u, v, c in self.edges:
            if not (0 <= u < self.n and 0 <= v < self.n):
                raise GraphError(f"edge ({u},{v}) out of range for n={self.n}")
            if c < 0:
                raise GraphError(f"negative capacity on edge ({u},{v}): {c}")
            if (u, v) in seen:
                raise GraphError(f"duplicate edge ({u},{v}); merge capacities first")
            seen.add((u, v))

    @classmethod
    def from_edges(cls, n, edges, meta=None) -> "Digraph":
        # merge parallels, drop loops and non-positive capacities, sort by (u,v)
        acc: dict = {}
        for u, v, c in edges:
            acc[(int(u), int(v))] = acc.get((int(u), int(v)), 0.0) + float(c)
        kept = tuple((u, v, c) for (u, v), c in sorted(acc.items())
                     if u != v and c > 0)
        return cls(n=int(n), edges=kept, meta=dict(meta or {}))

    @property
    def num_edges(self) -> int:
        return len(self.edges)

    @cached_property
    def edge_index(self) -> dict:
        return {(u, v): i for i, (u, v, _) in enumerate(self.edges)}

    @cached_property
    def capacities(self) -> tuple:
        return tuple(c for _, _, c in self.edges)

    @cached_property
    def out_adj(self) -> tuple:
        adj = [[] for _ in range(self.n)]
        for i, (u, v, _) in enumerate(self.edges):
            adj[u].append((v, i))
        return tuple(tuple(sorted(a)) for a in adj)


@dataclass(frozen=True)
class NodeMapping:
    """Original node -> (host, nic_in, nic_out) ids (reference src/graphs.py:118-124)."""

    host: tuple
    nic_in: tuple
    nic_out: tuple


def gen_torus(dims, bidirectional: bool = True) -> Digraph:
    """Torus with +-1 links per dimension; extent-2 dims give one link pair.

    Node id is row-major over ``dims`` (last dimension fastest), as in
    reference ``src/graphs.py:168-205``.
    """
    dims = [int(e) for e in dims]
    if not dims:
        raise GraphError("empty dims")
    if min(dims) < 2:
        raise GraphError(f"every extent must be >= 2, got {dims}")
    n = 1
    for e in dims:
        n *= e
    stride = [1] * len(dims)
    for i in range(len(dims) - 2, -1, -1):
        stride[i] = stride[i + 1] * dims[i + 1]
    pairs = set()
    for u in range(n):
        for i, e in enumerate(dims):
            x = (u // stride[i]) % e
            deltas = (1, -1) if e > 2 else (1,)
            if not bidirectional:
                deltas = (1,)
            for dl in deltas:
                v = u + (((x + dl) % e) - x) * stride[i]
                pairs.add((u, v))
    return Digraph.from_edges(
        n, [(u, v, 1.0) for u, v in pairs],
        {"generator": "torus", "params": {"dims": dims, "bidirectional": bidirectional}})


def gen_hypercube(k: int) -> Digraph:
    """k-cube with unit links u <-> u xor 2^i (reference src/graphs.py:208-216)."""
    if k < 1:
        raise GraphError("hypercube dimension must be >= 1")
    n = 1 << k
    return Digraph.from_edges(
        n, [(u, u ^ (1 << i), 1.0) for u in range(n) for i in range(k)],
        {"generator": "hypercube", "params": {"k": k}})


def gen_gen_kautz(n: int, d: int) -> Digraph:
    """Imase-Itoh generalized Kautz: u -> (-d*u - j) mod n, j = 1..d.

    Self-loops are dropped and counted in ``meta['self_loops']``
    (reference src/graphs.py:130-153).
    """
    if n < 2 or d < 1:
        raise GraphError(f"need n >= 2 and d >= 1, got n={n}, d={d}")
    if d >= n:
        raise GraphError(f"degree d={d} must be < n={n}")
    arcs = [(u, (-d * u - j) % n, 1.0) for u in range(n) for j in range(1, d + 1)]
    loops = sum(1 for u, v, _ in arcs if u == v)
    return Digraph.from_edges(
        n, arcs, {"generator": "genkautz", "params": {"n": n, "d": d},
                  "self_loops": loops})


def augment_host_bottleneck(g: Digraph, host_capacity: float):
    """3-way node split host=3v, nic_in=3v+1, nic_out=3v+2 (src/graphs.py:447-475).

    nic_in_v -> host_v -> nic_out_v carry ``host_capacity``; each physical link
    (u, v) becomes nic_out_u -> nic_in_v.  Forwarded traffic therefore pays
    the intermediate host link: the "without extra NIC-forwarding bandwidth"
    model.
    """
    if host_capacity <= 0:
        raise GraphError("host_capacity must be positive")
    if g.n < 2:
        raise GraphError("augmentation needs at least 2 nodes")
    h = float(host_capacity)
    arcs = []
    for v in range(g.n):
        arcs.append((3 * v + 1, 3 * v, h))
        arcs.append((3 * v, 3 * v + 2, h))
    for u, v, c in g.edges:
        arcs.append((3 * u + 2, 3 * v + 1, c))
    aug = Digraph.from_edges(3 * g.n, arcs,
                             {**g.meta, "host_bottleneck": {"capacity": h}})
    mp = NodeMapping(host=tuple(3 * v for v in range(g.n)),
                     nic_in=tuple(3 * v + 1 for v in range(g.n)),
                     nic_out=tuple(3 * v + 2 for v in range(g.n)))
    return aug, mp


def all_pairs_distances(g) -> list:
    """BFS hop matrix, -1 = unreachable (src/graphs.py:481-496)."""
    out = []
    adj = [[] for _ in range(g.n)]
    for u, v, _ in g.edges:
        adj[u].append(v)
    for s in range(g.n):
        row = [-1] * g.n
        row[s] = 0
        q = deque([s])
        while q:
            u = q.popleft()
            for v in adj[u]:
                if row[v] < 0:
                    row[v] = row[u] + 1
                    q.append(v)
        out.append(row)
    return out


def distance_sum(g) -> int:
    """Sum of BFS distances over ordered pairs s != d (the Sigma-dist of
    reference src/bounds.py:79-90); raises if not strongly connected."""
    tot = 0
    for s, row in enumerate(all_pairs_distances(g)):
        for d, x in enumerate(row):
            if s == d:
                continue
            if x < 0:
                raise GraphError(f"graph is not strongly connected: {d} unreachable from {s}")
            tot += x
    return tot


def _open(path, mode="rt"):
    return gzip.open(path, mode) if str(path).endswith(".gz") else open(path, mode)


def _cap_str(c: float) -> str:
    f = Fraction(c).limit_denominator(10 ** 9)
    return str(f) if float(f) == c else repr(c)


def save_graph(g, path) -> None:
    """JSON graph file in the reference format (src/graphs.py:550-559)."""
    doc = {"n": g.n, "directed": True,
           "edges": [[u, v, _cap_str(c)] for u, v, c in g.edges],
           "meta": dict(getattr(g, "meta", {}) or {})}
    with _open(path, "wt") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def load_graph(path) -> Digraph:
    """Read a reference-format graph JSON (src/graphs.py:562-584); .gz ok."""
    try:
        with _open(path) as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise GraphError(f"{path}: not valid JSON: {exc}") from exc
    try:
        n = int(doc["n"])
        raw = doc["edges"]
    except (KeyError, TypeError) as exc:
        raise GraphError(f"{path}: missing required field: {exc}") from exc
    arcs = []
    for k, rec in enumerate(raw):
        try:
            u, v = int(rec[0]), int(rec[1])
            c = float(rec[2]) if isinstance(rec[2], (int, float)) else float(Fraction(rec[2]))
        except (ValueError, IndexError, TypeError, ZeroDivisionError) as exc:
            raise GraphError(f"{path}: bad edge record #{k}: {rec!r}") from exc
        if not (0 <= u < n and 0 <= v < n):
            raise GraphError(f"{path}: edge #{k} ({u},{v}) out of range for n={n}")
        if c < 0:
            raise GraphError(f"{path}: edge #{k} ({u},{v}) has capacity {c} < 0")
        arcs.append((u, v, c))
    return Digraph.from_edges(n, arcs, doc.get("meta", {}))
