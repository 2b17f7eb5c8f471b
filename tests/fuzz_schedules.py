"""Random valid ts schedules for property tests (test infrastructure).

Each case: a random strongly connected digraph (a Hamiltonian ring plus
random chords), a random Q, and for every commodity (s, d) the chunk range
[0, Q) cut into 1..3 pieces, each sent along its own random simple path.  The
hop steps of one route are strictly increasing with random gaps (not only
hop i at step i), pieces of one commodity may take different routes, and a
route may re-split its chunk range mid-way, so forwarding ops read chunks that
arrived through several earlier ops.  Every schedule is valid by construction
(the reference's replay semantics: a chunk is forwarded only at a step after
it arrived, each chunk delivered exactly once).
"""
from __future__ import annotations

import numpy as np

from paper_2309_13541_b200.graphs import Digraph
from paper_2309_13541_b200.schedule import ChunkedSchedule, Instruction


def _random_path(rng, adj, s, d, n):
    """Random simple path s -> d (random-order DFS)."""
    stack = [(s, [s])]
    seen = {s}
    while stack:
        u, path = stack.pop()
        if u == d:
            return path
        nb = list(adj[u])
        rng.shuffle(nb)
        for v in nb:
            if v not in seen:
                seen.add(v)
                stack.append((v, path + [v]))
    raise AssertionError("graph not strongly connected")


def random_case(seed: int, n_max: int = 9, q_max: int = 48):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, n_max + 1))
    perm = rng.permutation(n)
    edges = {(int(perm[i]), int(perm[(i + 1) % n])) for i in range(n)}
    for _ in range(int(rng.integers(0, 2 * n))):
        u, v = (int(x) for x in rng.integers(0, n, 2))
        if u != v:
            edges.add((u, v))
    g = Digraph.from_edges(n, [(u, v, 1.0) for u, v in sorted(edges)])
    adj = [[] for _ in range(n)]
    for u, v in sorted(edges):
        adj[u].append(v)
    Q = int(rng.integers(1, q_max + 1))
    ins = []
    for s in range(n):
        for d in range(n):
            if s == d:
                continue
            cuts = sorted(set(int(x) for x in rng.integers(1, Q, int(rng.integers(0, 3))))) if Q > 1 else []
            bounds = [0] + cuts + [Q]
            for c0, c1 in zip(bounds[:-1], bounds[1:]):
                path = _random_path(rng, adj, s, d, n)
                # (c0, c1, hop index, step of the previous hop) work list: a
                # range may be re-split at an intermediate node
                work = [(c0, c1, 0, -1)]
                while work:
                    a, b, h, t_prev = work.pop()
                    t = t_prev + 1 + int(rng.integers(0, 2))
                    ins.append(Instruction(t, path[h], path[h + 1], s, d, a, b))
                    if h + 1 == len(path) - 1:
                        continue
                    if b - a > 1 and rng.random() < 0.3:
                        mid = int(rng.integers(a + 1, b))
                        work += [(a, mid, h + 1, t), (mid, b, h + 1, t)]
                    else:
                        work.append((a, b, h + 1, t))
    nsteps = max(i.t for i in ins) + 1
    order = rng.permutation(len(ins))
    sched = ChunkedSchedule(n=n, nsteps=nsteps, chunk_bytes=1.0, Q=Q, mode="ts",
                            instructions=[ins[i] for i in order])
    m = int(rng.choice([1, 7, 64, 1000, 4096 + 3, 3 * Q + 1]))
    G = int(rng.integers(1, min(n, 8) + 1))
    placement = [int(x) for x in rng.integers(0, G, n)]
    for gpu in range(G):          # every GPU hosts at least one node
        if gpu not in placement:
            placement[int(rng.integers(0, n))] = gpu
    if len(set(placement)) < G:
        placement = [v % G for v in range(n)]
    return g, sched, m, G, placement
