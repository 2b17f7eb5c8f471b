"""Step-balanced lowering (lowering.balanced_offsets): routes start at later
steps so that each step's cross-GPU egress is spread over the GPUs.  The
result is still a schedule the reference replay accepts (native replay), with
the same links, chunks and bytes per link as hop-indexed lowering, never a
higher step-synchronous cost, and the device protocol (CPU emulation) still
delivers the transpose."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2309_13541_b200.executor import Plan, replay_timestep_schedule
from paper_2309_13541_b200.lowering import (balanced_offsets, lower_path_to_steps,
                                            schedule_link_chunks, step_sync_cost)
from paper_2309_13541_b200.dist import local_nodes
from paper_2309_13541_b200.schedule import ScheduleError
from replay_bytes import make_send

CASES = [("gk8_2", 2), ("gk8_2", 4), ("gk8_2", 8), ("hypercube3", 4), ("hypercube3", 8),
         ("torus2x4", 8), ("torus4x4x4", 8), ("gk64_4", 4)]


def _lowered(a, G, m, extra=0):
    with Plan(a.g, a.sched, m=m, n_gpus=G, placement="optimized") as p:
        gpu = p.placement.tolist()
    offs = balanced_offsets(a.routes, a.path_sched, gpu, m, extra_steps=extra)
    return gpu, offs, lower_path_to_steps(a.routes, a.path_sched, n=a.g.n, offsets=offs)


@pytest.mark.parametrize("name,G", CASES)
def test_balanced_lowering_is_valid_and_no_worse(name, G, artifacts):
    a = artifacts(name)
    m = 1 << 20
    gpu, offs, s = _lowered(a, G, m)
    assert min(offs) >= 0
    assert s.nsteps == a.sched.nsteps                         # no extra steps asked for
    T, ok = replay_timestep_schedule(a.g, s)                  # reference replay semantics
    assert ok and T > 0
    # same links, chunks and bytes per link (summed over steps)
    def per_link(sc):
        out = {}
        for (t, e), c in schedule_link_chunks(sc, a.g).items():
            out[e] = out.get(e, 0) + c
        return out
    assert per_link(s) == per_link(a.sched)
    assert sorted((i.src, i.dst, i.s, i.d, i.c0, i.c1) for i in s.instructions) == \
        sorted((i.src, i.dst, i.s, i.d, i.c0, i.c1) for i in a.sched.instructions)
    assert step_sync_cost(s, gpu, m) <= step_sync_cost(a.sched, gpu, m)


def test_balanced_lowering_gains_on_gk8_2(artifacts):
    """GenKautz(8,2), one node per GPU: hop-indexed steps load step 0 with every
    first hop; balancing cuts the step-synchronous egress by > 5 %."""
    a = artifacts("gk8_2")
    m = 16 << 20
    gpu, _, s = _lowered(a, 8, m)
    assert step_sync_cost(s, gpu, m) < 0.95 * step_sync_cost(a.sched, gpu, m)


@pytest.mark.parametrize("name,G", [("gk8_2", 2), ("gk8_2", 8), ("hypercube3", 4), ("torus2x4", 8)])
@pytest.mark.parametrize("extra", [0, 2])
def test_balanced_lowering_emulation_delivers(name, G, extra, artifacts):
    a = artifacts(name)
    m = 4096 + 3
    _, _, s = _lowered(a, G, m, extra)
    send = make_send(a.g.n, m, seed=G + extra)
    want = np.swapaxes(send, 0, 1)
    for sched in ("static", "cp"):
        with Plan(a.g, s, m=m, n_gpus=G, placement="optimized") as p:
            if sched != "static":
                p.set_schedule(sched, 1024)
            nodes = [local_nodes(p, r) for r in range(G)]
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=7, seed=3)
            for r in range(G):
                assert np.array_equal(recvs[r], want[nodes[r]]), (sched, r)


def test_offsets_rejects(artifacts):
    a = artifacts("gk8_2")
    with pytest.raises(ScheduleError, match="one offset"):
        lower_path_to_steps(a.routes, a.path_sched, offsets=[0])
    with pytest.raises(ScheduleError, match="negative"):
        lower_path_to_steps(a.routes, a.path_sched, offsets=[-1] * len(a.path_sched.instructions))
    with pytest.raises(ScheduleError, match="path-mode"):
        balanced_offsets(a.routes, a.sched, [0] * a.g.n, 1)


@pytest.mark.parametrize("name", ["gk8_2", "hypercube3", "torus2x4_h2"])
@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("sched", ["static", "mix:1024", "cp:1024", "ready:1024", "cp:1024:64",
                                   "spread:1024", "ll", "ll128", "chain:1024", "chaind:1024"])
def test_every_autotune_order_delivers(name, G, sched, artifacts):
    """bench.balanced_artifact + every execution schedule bench.py's autotune
    tries, emulated at 13 and 148 CTAs per GPU."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    a = artifacts(name)
    m = 4096 + 7
    art, pl = bench.balanced_artifact(a, 16 << 20, G, "optimized")
    send = make_send(a.g.n, m, seed=G)
    want = np.swapaxes(send, 0, 1)
    with bench.make_plan(art, m, G, pl, sched, copy_self=True) as p:
        nodes = [local_nodes(p, r) for r in range(G)]
        for nc in (13, 148):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nc, seed=nc)
            for r in range(G):
                assert np.array_equal(recvs[r], want[nodes[r]]), (nc, r)


def test_balanced_offsets_validates_routes(artifacts):
    """Bad routes fail with the lowering's ScheduleError texts, not IndexError."""
    import copy

    from paper_2309_13541_b200.schedule import ScheduleError
    a = artifacts("gk8_2")
    gpu = [v % 2 for v in range(a.g.n)]
    bad = copy.deepcopy(a.path_sched)
    bad.instructions[0] = bad.instructions[0]._replace(dst=len(a.routes) + 5) \
        if hasattr(bad.instructions[0], "_replace") else type(bad.instructions[0])(
            t=0, src=bad.instructions[0].src, dst=len(a.routes) + 5, s=bad.instructions[0].s,
            d=bad.instructions[0].d, c0=bad.instructions[0].c0, c1=bad.instructions[0].c1)
    with pytest.raises(ScheduleError, match="out of range"):
        balanced_offsets(a.routes, bad, gpu, 4096)
    routes = copy.deepcopy(a.routes)
    routes[0]["nodes"] = list(reversed(routes[0]["nodes"]))
    with pytest.raises(ScheduleError, match="does not join"):
        balanced_offsets(routes, a.path_sched, gpu, 4096)
    with pytest.raises(ScheduleError, match="one GPU"):
        balanced_offsets(a.routes, a.path_sched, gpu[:-1], 4096)


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4", "gk8_2_h1"])
@pytest.mark.parametrize("parts", [2, 4])
def test_split_path_schedule(name, parts, artifacts):
    """Cutting every path instruction's chunk range into pieces keeps the
    routes, the per-link bytes and the modelled T's acceptance; the pieces can
    start at different steps."""
    from paper_2309_13541_b200.lowering import split_path_schedule
    a = artifacts(name)
    ps = split_path_schedule(a.path_sched, parts)
    assert len(ps.instructions) >= len(a.path_sched.instructions)
    gpu = [v % 2 for v in range(a.g.n)]
    offs = balanced_offsets(a.routes, ps, gpu, 4096, extra_steps=1)
    s = lower_path_to_steps(a.routes, ps, n=a.g.n, offsets=offs)
    T, ok = replay_timestep_schedule(a.g, s)          # the reference replay's checks, native
    assert ok and T > 0
    m = 4096 + 7
    with Plan(a.g, s, m=m, copy_self=False) as p, Plan(a.g, a.sched, m=m, copy_self=False) as q:
        assert np.array_equal(p.link_bytes().sum(axis=0), q.link_bytes().sum(axis=0))


@pytest.mark.parametrize("G", [2, 4, 8])
@pytest.mark.parametrize("sched", ["chain:262144", "chaind:262144"])
def test_balanced_lowering_linked_chains_deliver(G, sched, artifacts):
    """Chains at a size where hops link, on the balanced lowering with route
    pieces and extra steps (at 2 and 4 GPUs the hypercube keeps local hops)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    a = artifacts("hypercube3")
    m = 1 << 20
    art, pl = bench.balanced_artifact(a, 16 << 20, G, "optimized")
    send = make_send(a.g.n, m, seed=G)
    want = np.swapaxes(send, 0, 1)
    with bench.make_plan(art, m, G, pl, sched, copy_self=False) as p:
        nodes = [local_nodes(p, r) for r in range(G)]
        recvs = p.emulate([send[ns] for ns in nodes], num_ctas=37, seed=G)
        for r in range(G):
            for i, v in enumerate(nodes[r]):
                off = [s for s in range(a.g.n) if s != v]
                assert np.array_equal(recvs[r][i, off], want[v, off]), (r, v)
