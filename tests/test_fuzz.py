"""Property tests on random valid schedules (tests/fuzz_schedules.py).

Random digraphs, Q, shard sizes, routes with random step gaps and mid-route
re-splits, random placements on 1..8 GPUs.  CPU: the native validation accepts
them with the oracle's modelled T, and the device protocol emulated in random
interleavings (static programs, dynamic unit queues, LL lines) delivers the
transpose (chain mode with a 32-byte TMA ring, so the random routes' local hops
link into chains).  GPU: bit-exact against the oracle for every protocol and
engine.
"""
from __future__ import annotations

import numpy as np
import pytest

from fuzz_schedules import random_case
from paper_2309_13541_b200.dist import local_nodes
from paper_2309_13541_b200.executor import Plan
from replay_bytes import make_send, replay_bytes

SEEDS = list(range(200))


@pytest.mark.parametrize("seed", SEEDS)
def test_random_schedule_emulation(seed):
    g, sched, m, G, placement = random_case(seed)
    send = make_send(g.n, m, seed=seed)
    T, want, _ = replay_bytes(g, sched, send, m)
    assert np.array_equal(want, np.swapaxes(send, 0, 1))     # generator sanity
    for proto, mode, reuse in (("simple", "static", False), ("simple", "static", True),
                               ("simple", "dynamic", False), ("simple", "list", True),
                               ("simple", "cp", False), ("simple", "mix", True),
                               ("simple", "ready", False), ("simple", "ready", True),
                               ("simple", "spread", False),
                               ("simple", "chain", False), ("simple", "chaind", False),
                               ("ll", "static", False), ("ll128", "static", False)):
        with Plan(g, sched, m=m, n_gpus=G, placement=placement, protocol=proto,
                  reuse_scratch=reuse) as p:
            if mode.startswith("chain"):
                p.set_engine("tma", 16, 2)    # a 32-byte ring: hops of >= 32 B link
            if mode != "static":
                p.set_schedule(mode, 256)
            assert p.model_time(m) == pytest.approx(T, rel=0, abs=0)
            nodes = [local_nodes(p, r) for r in range(G)]
            for nc in (1, 2, 7, 37):
                recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nc, seed=seed + nc)
                for r in range(G):
                    assert np.array_equal(recvs[r], want[nodes[r]]), (proto, mode, reuse, nc, r)
                p.check_bounds(nc)


def test_random_schedules_form_chains():
    """Sanity of the chain fuzzing above: with the 32-byte ring, many random
    schedules do link hops into chains (a linked hop drops its wait entries)."""
    linked = 0
    for seed in SEEDS[:60]:
        g, sched, m, _, _ = random_case(seed)
        waits = {}
        for mode in ("cp", "chain"):
            with Plan(g, sched, m=m) as p:
                p.set_engine("tma", 16, 2)
                p.set_schedule(mode, 256)
                waits[mode] = p.dyn_stats(0, 7)["wait_entries"]
        assert waits["chain"] <= waits["cp"]
        linked += waits["chain"] < waits["cp"]
    assert linked >= 15


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[:30])
def test_random_schedule_gpu(seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g, sched, m, _, _ = random_case(seed)
    send = make_send(g.n, m, seed=seed)
    _, want, _ = replay_bytes(g, sched, send, m)
    s = torch.from_numpy(send).cuda()
    for proto, mode, engine, nc in (("simple", "static", "tma", 0), ("simple", "static", "lsu", 5),
                                    ("simple", "cp", "tma", 0), ("simple", "dynamic", "lsu", 1),
                                    ("simple", "list", "tma", 2), ("simple", "ready", "tma", 0),
                                    ("simple", "ready", "lsu", 3), ("ll", "static", "lsu", 0),
                                    ("ll", "static", "tma", 3), ("ll128", "static", "lsu", 0),
                                    ("ll128", "static", "tma", 2), ("simple", "chain", "tma16", 0),
                                    ("simple", "chaind", "tma16", 3), ("simple", "chain", "lsu", 2)):
        with Plan(g, sched, m=m, protocol=proto) as p:
            if engine == "tma16":
                p.set_engine("tma", 16, 2)
            else:
                p.set_engine(engine)
            if mode != "static":
                p.set_schedule(mode, 256)
            p.bind(0, num_ctas=nc)
            p.set_timeout(10.0)
            for rep in range(2):
                r = torch.zeros_like(s)
                p.execute(s, r, count_links=True)
                p.sync()
                assert np.array_equal(r.cpu().numpy(), want), (proto, mode, engine, rep)
            assert np.array_equal(p.read_link_counters(), 2 * p.link_bytes())


@pytest.mark.gpu
@pytest.mark.multigpu
@pytest.mark.parametrize("seed", SEEDS[:20])
def test_random_schedule_two_gpus(seed):
    """Random schedules and placements over two GPUs driven from one process
    (peer pointers): simple static, dynamic queues and LL, bit-exact."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    g, sched, m, _, _ = random_case(seed)
    rng = np.random.default_rng(seed + 1000)
    placement = [int(x) for x in rng.integers(0, 2, g.n)]
    placement[0], placement[-1] = 0, 1
    send = make_send(g.n, m, seed=seed)
    _, want, _ = replay_bytes(g, sched, send, m)
    for proto, mode in (("simple", "static"), ("simple", "cp"), ("simple", "ready"), ("ll", "static"),
                        ("ll128", "static")):
        plans = []
        for r in range(2):
            p = Plan(g, sched, m=m, n_gpus=2, placement=placement, protocol=proto)
            if mode != "static":
                p.set_schedule(mode, 256)
            plans.append(p.bind(r, device=r))
        ptrs = [p.arena_ptr() for p in plans]
        for p in plans:
            p.import_pointers(ptrs)
            p.set_timeout(10.0)
        nodes = [local_nodes(p, r) for r, p in enumerate(plans)]
        sends = [torch.from_numpy(np.ascontiguousarray(send[nodes[r]])).cuda(r) for r in range(2)]
        recvs = [p.recv_buffer() for p in plans]
        for rep in range(2):
            for r, p in enumerate(plans):
                p.execute(sends[r], recvs[r])
            for p in plans:
                p.sync()
            for r in range(2):
                assert np.array_equal(recvs[r].cpu().numpy(), want[nodes[r]]), (proto, mode, rep, r)
        for p in plans:
            p.close()
