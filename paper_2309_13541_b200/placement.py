"""Virtual-node -> GPU placement.

The multi-GPU bound is the cross-GPU bytes of the busiest GPU
(max_g max(egress_g, ingress_g), schedule link loads over NVLink).  Contiguous
blocks (``v*G//N``) are the default; ``optimized_placement`` searches balanced
placements for a smaller bound with the native optimiser
(``a2a_optimize_placement``: exhaustive for N <= 12, sampled swaps beyond).
"""
from __future__ import annotations

import numpy as np

from . import _native as N
from .executor import Plan, _raise, contiguous_placement

__all__ = ["edge_bytes", "cross_gpu_bytes", "optimized_placement"]


def edge_bytes(g, sched, m: int) -> np.ndarray:
    """Schedule bytes per edge (summed over steps) at shard size m."""
    with Plan(g, sched, m=m, copy_self=False) as p:
        return p.link_bytes().sum(axis=0).astype(np.int64)


def cross_gpu_bytes(g, eb: np.ndarray, placement) -> tuple:
    """(egress[G], ingress[G]) cross-GPU bytes of a placement."""
    G = max(placement) + 1
    eg, ing = [0] * G, [0] * G
    for e, (u, v, _) in enumerate(g.edges):
        a, b = placement[u], placement[v]
        if a != b:
            eg[a] += int(eb[e])
            ing[b] += int(eb[e])
    return eg, ing


def optimized_placement(g, sched, n_gpus: int, m: int = 1 << 20, iters: int = 400,
                        seed: int = 0, start=None) -> list:
    """Balanced placement minimising max_g max(egress, ingress); never worse
    than the start (contiguous blocks by default)."""
    place = np.ascontiguousarray(start if start is not None
                                 else contiguous_placement(g.n, n_gpus), dtype=np.int32)
    if n_gpus == 1:
        return place.tolist()
    eb = edge_bytes(g, sched, m)
    uv = np.ascontiguousarray([(u, v) for u, v, _ in g.edges], dtype=np.int32)
    rc = N.lib.a2a_optimize_placement(g.n, len(g.edges), uv.ctypes.data, eb.ctypes.data,
                                      int(n_gpus), int(iters), int(seed), place.ctypes.data)
    if rc:
        _raise(rc, "a2a_optimize_placement")
    return place.tolist()
