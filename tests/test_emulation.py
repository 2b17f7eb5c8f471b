"""CPU proof of the device synchronisation protocol.

a2a_plan_emulate runs the exact per-CTA byte ranges the kernel runs, for every
GPU of a G-GPU placement, in random interleavings constrained ONLY by the
host-computed producer-dependency lists (no step barriers).  If a list missed a
producer, some interleaving would read scratch/recv bytes before they are
written and the receive buffers would differ from the transpose.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2309_13541_b200.dist import local_nodes
from paper_2309_13541_b200.executor import Plan
from replay_bytes import make_send


def _run(a, m, G, nC, seed):
    send = make_send(a.g.n, m, seed=seed)
    with Plan(a.g, a.sched, m=m, n_gpus=G) as p:
        nodes = [local_nodes(p, g) for g in range(G)]
        recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nC, seed=seed)
        stats = [p.sync_stats(g) for g in range(G)]
    want = np.swapaxes(send, 0, 1)
    for g in range(G):
        assert np.array_equal(recvs[g], want[nodes[g]]), (G, nC, seed, g)
    return stats


@pytest.mark.parametrize("name", ["torus2x4", "hypercube3", "gk8_2", "torus2x4_h2",
                                  "gk8_2_h1", "ts_torus2x4", "ts_hypercube3", "ts_gk8_2",
                                  "ts_torus3x3", "ts_ring3"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nC", [1, 5, 37, 148])
def test_random_interleavings_deliver_transpose(name, G, nC, artifacts):
    a = artifacts(name)
    if G > a.g.n:
        pytest.skip("more GPUs than nodes")
    for seed in range(3):
        _run(a, 1000 + 64 * seed, G, nC, seed)


@pytest.mark.parametrize("name,G", [("torus4x4x4", 8), ("gk64_4", 4), ("gk64_4_h2", 8)])
def test_n64_interleavings(name, G, artifacts):
    a = artifacts(name)
    stats = _run(a, 2048, G, 148, 1)
    assert all(s["wait_flags"] > 0 for s in stats)


def test_dependency_lists_are_needed(artifacts):
    """Sanity of the test itself: with dependency lists the first-hop-only
    steps have no waits, later steps do."""
    a = artifacts("gk8_2")
    with Plan(a.g, a.sched, m=4096) as p:
        p.prepare(8)
        st = p.sync_stats(0)
    assert st["wait_flags"] > 0


@pytest.mark.parametrize("name,G", [("gk8_2", 2), ("gk8_2", 8), ("torus4x4x4", 4),
                                    ("hypercube3", 4), ("torus2x4_h2", 2)])
@pytest.mark.parametrize("split", [64, 4096, 0])
def test_interleaved_order_interleavings(name, G, split, artifacts):
    """Destination-interleaved item order (split pieces) keeps bytes and deps exact."""
    a = artifacts(name)
    m = 5000 if a.g.n <= 8 else 1024
    send = make_send(a.g.n, m, seed=2)
    with Plan(a.g, a.sched, m=m, n_gpus=G, order="interleaved", split_bytes=split) as p:
        nodes = [local_nodes(p, g) for g in range(G)]
        for seed in range(2):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=37, seed=seed)
            want = np.swapaxes(send, 0, 1)
            for g in range(G):
                assert np.array_equal(recvs[g], want[nodes[g]])
        lb = p.link_bytes()
    with Plan(a.g, a.sched, m=m, n_gpus=G) as q:
        assert np.array_equal(lb, q.link_bytes())


@pytest.mark.parametrize("name,G", [("gk8_2", 2), ("gk8_2", 4), ("hypercube3", 4),
                                    ("gk64_4", 8), ("torus2x4_h2", 4)])
def test_optimized_placement(name, G, artifacts):
    """f4: the optimiser keeps per-GPU node counts, never raises the NVLink
    bound, and the executor stays exact under the new placement."""
    from paper_2309_13541_b200.executor import contiguous_placement
    from paper_2309_13541_b200.placement import (cross_gpu_bytes, edge_bytes,
                                                 optimized_placement)
    a = artifacts(name)
    c = contiguous_placement(a.g.n, G)
    o = optimized_placement(a.g, a.sched, G)
    assert sorted(np.bincount(o, minlength=G)) == sorted(np.bincount(c, minlength=G))
    eb = edge_bytes(a.g, a.sched, 1 << 20)
    bound = lambda pl: max(max(x) for x in cross_gpu_bytes(a.g, eb, pl))  # noqa: E731
    assert bound(o) <= bound(c)
    m = 3000
    send = make_send(a.g.n, m, seed=1)
    with Plan(a.g, a.sched, m=m, n_gpus=G, placement=o) as p:
        nodes = [local_nodes(p, g) for g in range(G)]
        recvs = p.emulate([send[ns] for ns in nodes], num_ctas=29, seed=3)
    want = np.swapaxes(send, 0, 1)
    for g in range(G):
        assert np.array_equal(recvs[g], want[nodes[g]])


def test_placement_known_optimum():
    """GK(8,2) on 2 GPUs: exhaustive search finds the 16-chunk-MiB optimum."""
    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.placement import (cross_gpu_bytes, edge_bytes,
                                                 optimized_placement)
    a = load_artifact("gk8_2")
    eb = edge_bytes(a.g, a.sched, 1 << 20)
    o = optimized_placement(a.g, a.sched, 2)
    assert max(max(x) for x in cross_gpu_bytes(a.g, eb, o)) == 16 << 20


@pytest.mark.parametrize("name,G", [("gk8_2", 1), ("gk8_2", 2), ("gk8_2", 8), ("torus4x4x4", 4),
                                    ("torus4x4x4", 1), ("gk64_4_h2", 8), ("ts_torus2x4", 2),
                                    ("ts_hypercube3", 4), ("ts_torus3x3", 1), ("torus2x4_h2", 8)])
@pytest.mark.parametrize("nC", [7, 148])
def test_scratch_reuse_interleavings(name, G, nC, artifacts):
    """Liveness-reused scratch + WAR/WAW dependencies: exact under random
    interleavings (per-GPU flag visibility), and never larger than static."""
    a = artifacts(name)
    m = 4096 if a.g.n <= 9 else 512
    send = make_send(a.g.n, m, seed=4)
    with Plan(a.g, a.sched, m=m, n_gpus=G, reuse_scratch=True) as p:
        nodes = [local_nodes(p, g) for g in range(G)]
        for seed in range(3):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nC, seed=seed)
            want = np.swapaxes(send, 0, 1)
            for g in range(G):
                assert np.array_equal(recvs[g], want[nodes[g]]), (seed, g)
        reused = [p.gpu_info(g)["scratch_bytes"] for g in range(G)]
    with Plan(a.g, a.sched, m=m, n_gpus=G) as q:
        static = [q.gpu_info(g)["scratch_bytes"] for g in range(G)]
    assert all(r <= s for r, s in zip(reused, static))


def test_scratch_reuse_saves_memory(artifacts):
    a = artifacts("torus4x4x4")
    m = 1 << 20
    with Plan(a.g, a.sched, m=m, reuse_scratch=True) as p:
        r = p.gpu_info(0)["scratch_bytes"]
    with Plan(a.g, a.sched, m=m) as q:
        s = q.gpu_info(0)["scratch_bytes"]
    assert r < 0.8 * s


@pytest.mark.parametrize("name,G", [("gk8_2", 1), ("gk8_2", 2), ("gk8_2", 8), ("hypercube3", 4),
                                    ("torus4x4x4", 4), ("gk64_4_h2", 8), ("ts_torus2x4", 2),
                                    ("ts_torus3x3", 1), ("torus2x4_h2", 4)])
@pytest.mark.parametrize("unit", [0, 256, 1000 * 64])
@pytest.mark.parametrize("reuse", [False, True])
@pytest.mark.parametrize("mode", ["dynamic", "list", "cp", "mix", "ready", "spread"])
def test_dynamic_schedule_interleavings(name, G, unit, reuse, mode, artifacts):
    """Dynamic unit queues (f2): in-order grabbing + per-unit producer flags
    deliver the transpose under random interleavings, with and without
    scratch reuse, and never deadlock."""
    a = artifacts(name)
    m = 5000 if a.g.n <= 9 else 640
    send = make_send(a.g.n, m, seed=6)
    with Plan(a.g, a.sched, m=m, n_gpus=G, reuse_scratch=reuse) as p:
        p.set_schedule(mode, unit)
        nodes = [local_nodes(p, g) for g in range(G)]
        for seed in range(2):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=11, seed=seed)
            want = np.swapaxes(send, 0, 1)
            for g in range(G):
                assert np.array_equal(recvs[g], want[nodes[g]]), (seed, g)
        st = p.dyn_stats(0, 11)
        assert st["units"] > 0


@pytest.mark.parametrize("name,G", [("gk8_2", 1), ("gk8_2", 2), ("gk8_2", 8), ("hypercube3", 4),
                                    ("torus4x4x4", 4), ("torus2x4_h2", 4), ("ts_torus2x4", 2)])
@pytest.mark.parametrize("mode", ["dynamic", "list", "cp"])
@pytest.mark.parametrize("remote_ctas,nC", [(1, 11), (3, 11), (10, 11), (40, 11), (1, 2), (32, 148)])
def test_pinned_queue_split_interleavings(name, G, mode, remote_ctas, nC, artifacts):
    """Pinned two-queue split (a2a_plan_set_queue_split): CTAs never switch
    queues; every non-empty queue keeps a CTA, so random interleavings still
    deliver the transpose and never deadlock (emulator mirrors the kernel)."""
    a = artifacts(name)
    m = 5000 if a.g.n <= 9 else 640
    send = make_send(a.g.n, m, seed=12)
    with Plan(a.g, a.sched, m=m, n_gpus=G, placement="optimized") as p:
        p.set_schedule(mode, 1024).set_queue_split(remote_ctas)
        p.check_bounds(nC)
        nodes = [local_nodes(p, g) for g in range(G)]
        for seed in range(2):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nC, seed=seed)
            want = np.swapaxes(send, 0, 1)
            for g in range(G):
                assert np.array_equal(recvs[g], want[nodes[g]]), (seed, g)


def test_queue_split_rejects(artifacts):
    a = artifacts("gk8_2")
    with Plan(a.g, a.sched, m=4096, n_gpus=2) as p:
        with pytest.raises(ValueError):
            p.set_queue_split(-1)
        with pytest.raises(ValueError):
            p.set_schedule_spec("cp:1:2:3")
        with pytest.raises(KeyError):
            p.set_schedule_spec("nope")
        p.set_schedule_spec("spread:65536")
        assert p.schedule == "spread"
        p.set_schedule_spec("cp:1048576:64")
        assert (p.schedule, p.remote_ctas) == ("cp", 64)


@pytest.mark.parametrize("name,G", [("gk8_2", 2), ("gk8_2", 4), ("torus4x4x4", 4), ("hypercube3", 8),
                                    ("torus2x4_h2", 4), ("ts_hypercube3", 2)])
@pytest.mark.parametrize("w", [1, 3, 8])
def test_weighted_split_interleavings(name, G, w, artifacts):
    """Cost-weighted CTA split (NVLink bytes weighted w): still an exact
    partition of every step's bytes, dependencies still sufficient."""
    a = artifacts(name)
    m = 5000 if a.g.n <= 8 else 1024
    send = make_send(a.g.n, m, seed=8)
    with Plan(a.g, a.sched, m=m, n_gpus=G, placement="optimized") as p:
        p.set_split(w)
        nodes = [local_nodes(p, g) for g in range(G)]
        for seed in range(2):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=23, seed=seed)
            want = np.swapaxes(send, 0, 1)
            for g in range(G):
                assert np.array_equal(recvs[g], want[nodes[g]])


# ---- A2A_PROTO_LL: cross-GPU bytes as {data, epoch} lines polled by the receiver
@pytest.mark.parametrize("name", ["torus2x4", "hypercube3", "gk8_2", "gk8_2_h1",
                                  "ts_torus2x4", "ts_gk8_2", "ts_torus3x3", "ts_ring3"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nC", [1, 5, 148])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ll_interleavings_deliver_transpose(name, G, nC, proto, artifacts):
    """LL everywhere: every hop lands as lines, forwarders poll them, same-step
    decodes of remote final hops come last in each CTA step; lines in the
    device format; odd shard sizes exercise partial lines and unaligned
    payload addresses."""
    a = artifacts(name)
    if G > a.g.n:
        pytest.skip("more GPUs than nodes")
    for seed, m in enumerate((4096, 1000, 77, 123457)):
        send = make_send(a.g.n, m, seed=seed)
        with Plan(a.g, a.sched, m=m, n_gpus=G, protocol=proto) as p:
            nodes = [local_nodes(p, g) for g in range(G)]
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nC, seed=seed)
            p.check_bounds(nC)
            stats = [p.sync_stats(g) for g in range(G)]
            with Plan(a.g, a.sched, m=m, n_gpus=G) as q:
                assert np.array_equal(p.link_bytes(), q.link_bytes())
                for g in range(G):
                    pi, qi = p.gpu_info(g), q.gpu_info(g)
                    assert pi["egress_bytes"] == qi["egress_bytes"]
                    assert pi["hop_bytes"] == qi["hop_bytes"]
        want = np.swapaxes(send, 0, 1)
        for g in range(G):
            assert np.array_equal(recvs[g], want[nodes[g]]), (G, nC, m, g)
        # no step flags at all: every dependency is a polled line
        assert all(s["wait_flags"] == 0 and s["exit_flags"] == 0 for s in stats)


@pytest.mark.parametrize("name,G", [("torus4x4x4", 8), ("gk64_4", 4)])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ll_n64_interleavings(name, G, proto, artifacts):
    a = artifacts(name)
    send = make_send(a.g.n, 512, seed=3)
    with Plan(a.g, a.sched, m=512, n_gpus=G, protocol=proto) as p:
        nodes = [local_nodes(p, g) for g in range(G)]
        recvs = p.emulate([send[ns] for ns in nodes], num_ctas=148, seed=3)
    want = np.swapaxes(send, 0, 1)
    for g in range(G):
        assert np.array_equal(recvs[g], want[nodes[g]])


def test_ll128_landing_region_and_lines(artifacts):
    """LL128 slots start on 120-byte payload boundaries, the landing region is
    128 bytes per 120 payload bytes (vs 16 per 8 for LL): ~1.07x the payload."""
    a = artifacts("gk8_2")
    m = 1 << 20
    with Plan(a.g, a.sched, m=m, n_gpus=4, protocol="ll128") as p128, \
            Plan(a.g, a.sched, m=m, n_gpus=4, protocol="ll") as p16:
        for g in range(4):
            s128, s16 = p128.gpu_info(g)["scratch_bytes"], p16.gpu_info(g)["scratch_bytes"]
            assert s128 < 0.56 * s16
        assert np.array_equal(p128.link_bytes(), p16.link_bytes())


def test_ll_rejects(artifacts):
    a = artifacts("gk8_2")
    with pytest.raises(ValueError, match="PROTO_LL"):
        Plan(a.g, a.sched, m=4096, n_gpus=2, protocol="ll", reuse_scratch=True)
    with pytest.raises(ValueError, match="PROTO_LL"):
        Plan(a.g, a.sched, m=4096, n_gpus=2, protocol="ll", order="interleaved")
    with Plan(a.g, a.sched, m=4096, n_gpus=2, protocol="ll") as p:
        with pytest.raises(ValueError, match="static"):
            p.set_schedule("dynamic")
    with pytest.raises(ValueError):
        Plan(a.g, a.sched, m=4096, n_gpus=2, protocol="bogus")


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4_h2", "ts_hypercube3"])
@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("sched", ["static", "cp", "spread"])
def test_without_self_copy(name, G, sched, artifacts):
    """copy_self=False (what bench.py times: the reference transpose skips
    s == d, evaluate.py:114-118): every s != d shard delivered, the self
    rows of recv untouched."""
    a = artifacts(name)
    m = 4096 + 24
    send = make_send(a.g.n, m, seed=5)
    with Plan(a.g, a.sched, m=m, n_gpus=G, copy_self=False) as p:
        if sched != "static":
            p.set_schedule(sched, 1024)
        nodes = [local_nodes(p, g) for g in range(G)]
        recvs = p.emulate([send[ns] for ns in nodes], num_ctas=7, seed=3)
    want = np.swapaxes(send, 0, 1)
    for g in range(G):
        for i, v in enumerate(nodes[g]):
            for s in range(a.g.n):
                if s == v:
                    assert not recvs[g][i, s].any()
                else:
                    assert np.array_equal(recvs[g][i, s], want[v, s]), (g, v, s)


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4", "hypercube3", "torus2x4_h2", "ts_gk8_2",
                                  "ts_torus3x3"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("m,unit", [(1 << 20, 262144), (262144 + 48, 196608), (1000, 0)])
@pytest.mark.parametrize("mode", ["chain", "chaind"])
def test_chain_interleavings_deliver_transpose(name, G, m, unit, mode, artifacts):
    """Chain mode (schedule "chain"): a route's consecutive local hops run on
    one CTA with no flag between them, tasks wait only at their head, all
    unit flags are published when the task ends; random interleavings of all
    CTAs of all GPUs over three executes deliver the transpose."""
    a = artifacts(name)
    if G > a.g.n:
        pytest.skip("more GPUs than nodes")
    send = make_send(a.g.n, m, seed=G)
    with Plan(a.g, a.sched, m=m, n_gpus=G) as p:
        p.set_schedule(mode, unit)
        nodes = [local_nodes(p, g) for g in range(G)]
        for nc in (1, 7, 148):
            recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nc, seed=nc)
            for g in range(G):
                assert np.array_equal(recvs[g], np.swapaxes(send, 0, 1)[nodes[g]]), (nc, g)
        p.check_bounds(37)


def test_chain_links_routes(artifacts):
    """On one GPU the path schedules' routes become single tasks: every hop
    after the first has no wait list (GK(8,2): 4 of 7814 units keep one)."""
    a = artifacts("gk8_2")
    with Plan(a.g, a.sched, m=16 << 20, copy_self=False) as p:
        p.set_schedule("chain", 262144)
        st = p.dyn_stats(0, 148)
    assert st["units"] > 7000 and st["wait_entries"] < 16
