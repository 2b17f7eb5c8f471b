"""Drop-in-side lowering helpers the reference does not have.

``compile_path_schedule`` (reference src/schedule.py:244-312) emits a
``mode="path"`` schedule: one instruction per route, ``dst`` = route id,
``nsteps = 1``.  The reference replay only accepts ``mode="ts"``
(src/evaluate.py:70-71).  The executor runs the paper's hop-by-hop semantics
("copy it from the source buffer of v1 to the scratch buffer of
v2, then ... v3 and so on"): hop i of every route at step i.  The result is a
legal ts schedule that the reference replay accepts unchanged.

For the host-augmented ("without extra NIC-forwarding bandwidth") lowering
(src/graphs.py:447-475), routes live on augmented ids host=3v, nic_in=3v+1,
nic_out=3v+2 and must be collapsed to physical node sequences first.
"""
from __future__ import annotations

from .schedule import ChunkedSchedule, Instruction, ScheduleError

__all__ = ["lower_path_to_steps", "balanced_offsets", "split_path_schedule", "step_sync_cost",
           "collapse_aug_routes",
           "collapse_aug_schedule", "schedule_link_chunks", "hop_histogram"]


def _ts_key(i):
    # the ts sort key of reference src/schedule.py:237
    return (i.t, i.src, i.dst, i.s, i.d, i.c0)


def lower_path_to_steps(routes, sched, n: int | None = None, offsets=None) -> ChunkedSchedule:
    """Expand each route instruction into one hop-op per link, hop i at step i.

    ``routes`` is the route list returned by compile_path_schedule (or its
    ``.routes.json`` sidecar); ``sched`` the ``mode="path"`` schedule.
    ``offsets`` (one per instruction, default 0) delays a whole route: hop i
    at step offsets[k] + i (e.g. from ``balanced_offsets``).
    """
    if sched.mode != "path":
        raise ScheduleError(f"expected a path-mode schedule, got {sched.mode!r}")
    if offsets is not None and len(offsets) != len(sched.instructions):
        raise ScheduleError("one offset per path instruction")
    ops = []
    nsteps = 0
    for k, ins in enumerate(sched.instructions):
        off = 0 if offsets is None else int(offsets[k])
        if off < 0:
            raise ScheduleError(f"negative offset {off}")
        nodes = _route_nodes(routes, ins)
        for i in range(len(nodes) - 1):
            ops.append(Instruction(t=off + i, src=nodes[i], dst=nodes[i + 1],
                                   s=ins.s, d=ins.d, c0=ins.c0, c1=ins.c1))
        nsteps = max(nsteps, off + len(nodes) - 1)
    ops.sort(key=_ts_key)
    return ChunkedSchedule(n=sched.n if n is None else n, nsteps=nsteps,
                           chunk_bytes=sched.chunk_bytes, Q=sched.Q, mode="ts",
                           instructions=ops)


def split_path_schedule(sched, parts: int) -> ChunkedSchedule:
    """The same path schedule with every instruction's chunk range [c0, c1)
    cut into up to `parts` near-equal sub-ranges (one instruction each, same
    route).  Routes, links and bytes per link are unchanged; the pieces can
    then start at different steps (balanced_offsets), which balances the
    per-step NVLink load at a finer grain than whole routes."""
    if sched.mode != "path":
        raise ScheduleError(f"expected a path-mode schedule, got {sched.mode!r}")
    parts = max(1, int(parts))
    ins = []
    for i in sched.instructions:
        n = i.c1 - i.c0
        k = max(1, min(parts, n))
        for j in range(k):
            a, b = i.c0 + n * j // k, i.c0 + n * (j + 1) // k
            if b > a:
                ins.append(Instruction(t=i.t, src=i.src, dst=i.dst, s=i.s, d=i.d, c0=a, c1=b))
    return ChunkedSchedule(n=sched.n, nsteps=sched.nsteps, chunk_bytes=sched.chunk_bytes,
                           Q=sched.Q, mode="path", instructions=ins)


def _route_nodes(routes, ins) -> list:
    """Node sequence of the route a path instruction names (dst = route id),
    checked: the id exists, the route joins the instruction's shard, it has
    at least one hop."""
    if not 0 <= ins.dst < len(routes):
        raise ScheduleError(f"route id {ins.dst} out of range")
    r = routes[ins.dst]
    nodes = list(r["nodes"])
    if (r["s"], r["d"]) != (ins.s, ins.d) or nodes[0] != ins.s or nodes[-1] != ins.d:
        raise ScheduleError(
            f"route {ins.dst} {nodes} does not join shard ({ins.s},{ins.d})")
    if len(nodes) < 2:
        raise ScheduleError(f"route {ins.dst} has no hops")
    return nodes


def _route_egress(routes, ins, node_gpu, m, Q):
    """[(hop i, source GPU, destination GPU, bytes)] of the cross-GPU hops of
    one path instruction."""
    nodes = routes[ins.dst]["nodes"]
    nb = (ins.c1 * m) // Q - (ins.c0 * m) // Q
    return [(i, node_gpu[nodes[i]], node_gpu[nodes[i + 1]], nb) for i in range(len(nodes) - 1)
            if node_gpu[nodes[i]] != node_gpu[nodes[i + 1]]]


def step_sync_cost(sched, node_gpu, m: int) -> int:
    """Sum over steps of the busiest NVLink direction in that step (max over
    GPUs of cross-GPU egress and ingress bytes): the time (x NVLink bandwidth
    per direction) of a ts schedule executed step-synchronously."""
    G = max(node_gpu) + 1
    load = [[0] * (2 * G) for _ in range(sched.nsteps)]
    for i in sched.instructions:
        g, h = node_gpu[i.src], node_gpu[i.dst]
        if 0 <= i.t < sched.nsteps and g != h:
            nb = (i.c1 * m) // sched.Q - (i.c0 * m) // sched.Q
            load[i.t][g] += nb
            load[i.t][G + h] += nb
    return sum(max(x) for x in load)


def balanced_offsets(routes, sched, node_gpu, m: int, extra_steps: int = 0,
                     passes: int = 4) -> list:
    """Per-route start steps for ``lower_path_to_steps`` that balance each
    step's cross-GPU egress over the GPUs of a placement.

    Hop-indexed lowering puts every route's first hop at step 0, so step 0 is
    the heaviest and the last step nearly empty; a step-synchronous execution
    pays sum_t max_g egress(t, g).  Greedy: routes by cross-GPU bytes x hops,
    largest first, each at the offset in [0, L - hops] (L = longest route +
    extra_steps) that minimises that sum so far (ties: earliest).  Egress and
    ingress both count (each step costs its busiest NVLink direction).  Hop
    order within a route, the links and the bytes per link are unchanged; only
    steps move; ``passes`` rounds of single-route moves then lower the sum
    further.  The objective is step_sync_cost of the lowered schedule."""
    if sched.mode != "path":
        raise ScheduleError(f"expected a path-mode schedule, got {sched.mode!r}")
    if len(node_gpu) != sched.n or min(node_gpu, default=0) < 0:
        raise ScheduleError(f"placement must list one GPU >= 0 per node ({sched.n})")
    G = max(node_gpu) + 1
    hops = [len(_route_nodes(routes, i)) - 1 for i in sched.instructions]
    L = max(hops, default=0) + int(extra_steps)
    load = [[0] * (2 * G) for _ in range(L)]
    eg = [_route_egress(routes, i, node_gpu, m, sched.Q) for i in sched.instructions]
    order = sorted(range(len(eg)), key=lambda k: (-sum(x[3] for x in eg[k]) * hops[k], k))
    offs = [0] * len(eg)

    def place(k, o, sign):
        for i, g, h, b in eg[k]:
            load[o + i][g] += sign * b
            load[o + i][G + h] += sign * b

    def best_offset(k):
        best = None
        for o in range(L - hops[k] + 1):
            add: dict = {}
            for i, g, h, b in eg[k]:
                add[(o + i, g)] = add.get((o + i, g), 0) + b
                add[(o + i, G + h)] = add.get((o + i, G + h), 0) + b
            delta = 0
            for t in {t for t, _ in add}:
                row = load[t]
                delta += max(0, max(row[c] + b for (tt, c), b in add.items() if tt == t) - max(row))
            if best is None or delta < best[0]:
                best = (delta, o)
        return best[1]

    for k in order:
        offs[k] = best_offset(k)
        place(k, offs[k], 1)
    # improvement passes: take each route out and put it back at its best
    # offset given all the others; keep a move only if the total drops
    total = sum(max(r) for r in load)
    for _ in range(int(passes)):
        moved = False
        for k in order:
            if not eg[k]:
                continue
            place(k, offs[k], -1)
            o = best_offset(k)
            place(k, o, 1)
            t = sum(max(r) for r in load)
            if t < total:
                offs[k], total, moved = o, t, True
            else:
                place(k, o, -1)
                place(k, offs[k], 1)
        if not moved:
            break
    return offs


def _phys_of(mapping):
    phys = {}
    for v, (h, a, b) in enumerate(zip(mapping.host, mapping.nic_in, mapping.nic_out)):
        phys[h] = phys[a] = phys[b] = v
    return phys


def collapse_aug_routes(routes, mapping) -> list:
    """Map augmented node ids to physical nodes and drop repeats.

    host_u -> nic_out_u -> nic_in_v -> host_v collapses to the physical hop
    u -> v.  A simple augmented path visits each host at most once, so the
    collapsed sequence is simple.
    """
    phys = _phys_of(mapping)
    out = []
    for r in routes:
        seq = []
        for x in r["nodes"]:
            v = phys[x]
            if not seq or seq[-1] != v:
                seq.append(v)
        if len(set(seq)) != len(seq):
            raise ScheduleError(f"collapsed route {seq} is not simple")
        out.append({"s": phys[r["s"]], "d": phys[r["d"]], "nodes": seq})
    return out


def collapse_aug_schedule(routes, sched, mapping):
    """(physical routes, physical path schedule) for an augmented lowering."""
    phys = _phys_of(mapping)
    routes_p = collapse_aug_routes(routes, mapping)
    ins = [Instruction(t=i.t, src=phys[i.src], dst=i.dst, s=phys[i.s], d=phys[i.d],
                       c0=i.c0, c1=i.c1) for i in sched.instructions]
    sp = ChunkedSchedule(n=len(mapping.host), nsteps=sched.nsteps,
                         chunk_bytes=sched.chunk_bytes, Q=sched.Q, mode="path",
                         instructions=ins)
    return routes_p, sp


def schedule_link_chunks(sched, g) -> dict:
    """{(t, edge id): chunks} of a ts schedule (what the executor must move)."""
    eidx = g.edge_index
    out: dict = {}
    for i in sched.instructions:
        if 0 <= i.t < sched.nsteps and i.c1 > i.c0:
            k = (i.t, eidx[(i.src, i.dst)])
            out[k] = out.get(k, 0) + (i.c1 - i.c0)
    return out


def hop_histogram(sched) -> list:
    """Hop-ops per step of a ts schedule."""
    h = [0] * sched.nsteps
    for i in sched.instructions:
        if 0 <= i.t < sched.nsteps:
            h[i.t] += 1
    return h
