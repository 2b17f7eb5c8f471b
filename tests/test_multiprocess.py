"""Gloo tests of the multi-GPU host logic (CPU only), world sizes 2, 4 and 8.

The processes each build the plan for G=world (as bench.py ranks do), prove they
built identical layouts (plan digest), exchange fixed-size handles through the
same all_gather_object path bench.py uses, and check that the per-rank pieces
compose: each rank's recv rows from the oracle equal the transpose rows of its
own virtual nodes, and egress/ingress agree pairwise.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, m, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch.distributed as dist
    from c_oracle import replay_bytes_c
    from replay_bytes import make_send

    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.dist import check_same_plan, local_nodes, plan_digest
    from paper_2309_13541_b200.executor import Plan
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                                rank=rank, world_size=world)
        a = load_artifact(name)
        plan = Plan(a.g, a.sched, m=m, n_gpus=world)
        check_same_plan(plan)
        fake = bytes([rank]) * 64                       # stands in for the IPC handle
        hs = [None] * world
        dist.all_gather_object(hs, fake)
        assert [h[0] for h in hs] == list(range(world)) and all(len(h) == 64 for h in hs)
        nodes = local_nodes(plan, rank)
        info = plan.gpu_info(rank)
        assert info["n_local_nodes"] == len(nodes) and info["first_node"] == nodes[0]
        send = make_send(a.g.n, m, seed=9)
        _, recv, _ = replay_bytes_c(a.g, a.sched, send, m, nthreads=2)
        mine = recv[nodes]                                # this rank's [V, N, m] recv
        want = np.swapaxes(send, 0, 1)[nodes]
        ok = bool(np.array_equal(mine, want))
        eg = [plan.gpu_info(g)["egress_bytes"] for g in range(world)]
        ing = [plan.gpu_info(g)["ingress_bytes"] for g in range(world)]
        flags = [None] * world
        dist.all_gather_object(flags, (ok, plan_digest(plan), info["egress_bytes"]))
        q.put((rank, all(f[0] for f in flags), len({f[1] for f in flags}) == 1,
               sum(eg) == sum(ing), [f[2] for f in flags] == eg))
        dist.destroy_process_group()
    except Exception as ex:  # surface worker errors to the test
        q.put((rank, repr(ex)))


@pytest.mark.parametrize("name,m,world", [("torus2x4", 96, 2), ("gk8_2", 4096 + 1, 2),
                                          ("hypercube3", 4096, 4), ("gk8_2", 4096 + 1, 8)])
def test_multi_rank_host_logic(name, m, world):
    """world=8 is the driver's 8-GPU bench shape: one virtual node per rank."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, name, m, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for p in ps:
        if p.is_alive():
            p.kill()
            p.join(timeout=10)
    for r in res:
        assert len(r) == 5, r
        assert all(r[1:]), r
