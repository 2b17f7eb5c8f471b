"""GPU parity: the sm_100a executor vs the CPU oracle and the schedule.

Bit-exact receive buffers against oracle/replay_bytes.py (itself pinned to the
reference replay by tests/test_oracle.py) on every small artifact at several
shard sizes, including sizes that break 16-byte alignment; device-counted
per-(step, link) bytes equal to the plan's schedule bytes; at full sizes the
size-independent transpose property recv[d][s] == send[s][d].
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

SMALL = ["torus2x4", "hypercube3", "gk8_2", "torus2x4_h1", "torus2x4_h2", "gk8_2_h1",
         "ts_ring3", "ts_torus2x4", "ts_hypercube3", "ts_gk8_2", "ts_torus3x3"]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


def _send(n, m, seed=0):
    from replay_bytes import make_send
    return make_send(n, m, seed=seed)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("m", [1, 7, 1000, 4096, 65536 + 3])
def test_recv_bit_exact_vs_oracle(name, m, artifacts):
    from paper_2309_13541_b200.executor import execute_timestep_schedule
    from replay_bytes import replay_bytes
    a = artifacts(name)
    send = _send(a.g.n, m, seed=m)
    _, want, _ = replay_bytes(a.g, a.sched, send, m)
    s = torch.from_numpy(send).cuda()
    r = torch.zeros_like(s)
    T, ok = execute_timestep_schedule(a.g, a.sched, s, r)
    assert ok and T > 0
    assert np.array_equal(r.cpu().numpy(), want)


@pytest.mark.parametrize("name", SMALL)
def test_device_link_counters_equal_schedule(name, artifacts):
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    m = 3 * a.sched.Q + 5
    send = _send(a.g.n, m)
    _, _, ob = replay_bytes(a.g, a.sched, send, m)
    with Plan(a.g, a.sched, m=m) as p:
        p.bind(0)
        s = torch.from_numpy(send).cuda()
        r = torch.empty_like(s)
        p.execute(s, r, count_links=True)
        p.sync()
        dev = p.read_link_counters()
        want = p.link_bytes()
    ref = np.zeros_like(want)
    for (t, e), x in ob.items():
        ref[t, e] = x
    assert np.array_equal(want, ref)
    assert np.array_equal(dev, want)


@pytest.mark.parametrize("num_ctas", [1, 3, 64, 0])
def test_cta_counts_and_repeats(num_ctas, artifacts):
    """Any grid size gives the same bytes; repeated executes (epochs) stay exact."""
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("gk8_2")
    m = 12345
    with Plan(a.g, a.sched, m=m) as p:
        p.bind(0, num_ctas=num_ctas)
        for seed in range(4):
            s = torch.from_numpy(_send(a.g.n, m, seed)).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r)
            p.sync()
            assert torch.equal(r, s.transpose(0, 1).contiguous())


@pytest.mark.parametrize("name,m", [("torus4x4x4", 65536), ("gk64_4", 65536 + 48),
                                    ("gk64_4_h2", 4096), ("torus4x4x4", 1000)])
def test_n64_transpose_and_counters(name, m, artifacts):
    from paper_2309_13541_b200.artifacts import list_artifacts
    from paper_2309_13541_b200.executor import Plan
    if name not in list_artifacts():
        pytest.skip(f"artifact {name} not generated")
    a = artifacts(name)
    n = a.g.n
    g = torch.Generator(device="cuda").manual_seed(7)
    s = torch.randint(0, 256, (n, n, m), dtype=torch.uint8, device="cuda", generator=g)
    r = torch.zeros_like(s)
    with Plan(a.g, a.sched, m=m) as p:
        p.bind(0)
        p.execute(s, r, count_links=True)
        p.sync()
        dev = p.read_link_counters()
        assert np.array_equal(dev, p.link_bytes())
    assert torch.equal(r, s.transpose(0, 1).contiguous())


def test_full_size_gk8_16mib(artifacts):
    """configs[1] workload on one GPU: GenKautz(8,2), 16 MiB per pair."""
    from paper_2309_13541_b200.executor import execute_timestep_schedule
    a = artifacts("gk8_2")
    m = 16 << 20
    g = torch.Generator(device="cuda").manual_seed(1)
    s = torch.randint(0, 256, (8, 8, m), dtype=torch.uint8, device="cuda", generator=g)
    r = torch.zeros_like(s)
    T, ok = execute_timestep_schedule(a.g, a.sched, s, r)
    assert ok
    assert torch.equal(r, s.transpose(0, 1).contiguous())


def test_execute_rejects_wrong_buffers(artifacts):
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("torus2x4")
    with Plan(a.g, a.sched, m=64) as p:
        p.bind(0)
        s = torch.zeros((8, 8, 64), dtype=torch.uint8, device="cuda")
        with pytest.raises(ValueError):
            p.execute(s[:, :, :32].contiguous())
        with pytest.raises(TypeError):
            p.execute(s.float())
        with pytest.raises(TypeError):
            p.execute(s.cpu())


@pytest.mark.parametrize("name", ["torus2x4", "gk8_2", "torus2x4_h2", "ts_hypercube3"])
@pytest.mark.parametrize("m,ring", [(7, (0, 0)), (4096 + 5, (0, 0)), (65536, (4096, 2)),
                                    ((1 << 20) + 48, (32768, 6)), (300000, (16, 1))])
def test_tma_engine_bit_exact(name, m, ring, artifacts):
    """TMA bulk-copy engine (cp.async.bulk ring) == oracle, incl. odd sizes and
    degenerate rings (1 stage of 16 bytes)."""
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    send = _send(a.g.n, m, seed=m % 97)
    _, want, _ = replay_bytes(a.g, a.sched, send, m)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_engine("tma", *ring)
        p.bind(0)
        s = torch.from_numpy(send).cuda()
        for rep in range(2):
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want)
        dev = p.read_link_counters()
        assert np.array_equal(dev, 2 * p.link_bytes())


def test_tma_engine_n64(artifacts):
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("torus4x4x4")
    m = 65536 + 16
    g = torch.Generator(device="cuda").manual_seed(3)
    s = torch.randint(0, 256, (64, 64, m), dtype=torch.uint8, device="cuda", generator=g)
    r = torch.zeros_like(s)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_engine("tma")
        p.bind(0)
        p.execute(s, r)
        p.sync()
    assert torch.equal(r, s.transpose(0, 1).contiguous())


@pytest.mark.parametrize("name", ["torus2x4", "gk8_2", "torus2x4_h2", "ts_hypercube3", "ts_torus3x3"])
@pytest.mark.parametrize("engine", ["tma", "lsu"])
@pytest.mark.parametrize("m,unit", [(7, 0), (4096 + 5, 0), (65536, 4096), ((1 << 20) + 48, 0)])
@pytest.mark.parametrize("reuse", [False, True])
@pytest.mark.parametrize("mode", ["dynamic", "list", "cp", "mix", "ready", "spread"])
def test_dynamic_schedule_bit_exact(name, engine, m, unit, reuse, mode, artifacts):
    """Dynamic unit queues (f2) on the device: exact over repeated executes
    (the grab counter carries across epochs), with and without scratch reuse."""
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    with Plan(a.g, a.sched, m=m, reuse_scratch=reuse) as p:
        p.set_schedule(mode, unit)
        p.set_engine(engine)
        p.bind(0)
        for rep in range(3):
            send = _send(a.g.n, m, seed=rep + m % 13)
            _, want, _ = replay_bytes(a.g, a.sched, send, m)
            s = torch.from_numpy(send).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), rep
        assert np.array_equal(p.read_link_counters(), 3 * p.link_bytes())


@pytest.mark.parametrize("reuse", [False, True])
def test_dynamic_n64(reuse, artifacts):
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("gk64_4_h2")
    m = 32768 + 16
    g = torch.Generator(device="cuda").manual_seed(5)
    s = torch.randint(0, 256, (64, 64, m), dtype=torch.uint8, device="cuda", generator=g)
    with Plan(a.g, a.sched, m=m, reuse_scratch=reuse) as p:
        p.set_schedule("dynamic")
        p.bind(0)
        for _ in range(2):
            r = torch.zeros_like(s)
            p.execute(s, r)
            p.sync()
            assert torch.equal(r, s.transpose(0, 1).contiguous())


def test_missing_peer_times_out_instead_of_hanging(artifacts):
    """A 2-GPU plan whose peer never launches: the entry barrier spin is bounded
    by the device timeout and reports A2A_ERR_TIMEOUT (no hang); the plan then
    refuses further executes."""
    from paper_2309_13541_b200.executor import ExecutorError, Plan
    a = artifacts("gk8_2")
    m = 4096
    p0 = Plan(a.g, a.sched, m=m, n_gpus=2).bind(0, device=0)
    p1 = Plan(a.g, a.sched, m=m, n_gpus=2).bind(1, device=0)   # never executes
    ptrs = [p0.arena_ptr(), p1.arena_ptr()]
    p0.import_pointers(ptrs)
    p0.set_timeout(0.3)
    info = p0.gpu_info(0)
    s = torch.zeros(info["send_bytes"], dtype=torch.uint8, device="cuda")
    p0.execute(s, p0.recv_buffer().reshape(-1))
    with pytest.raises(ExecutorError, match="TIMEOUT"):
        p0.sync()
    with pytest.raises(ExecutorError):
        p0.execute(s, p0.recv_buffer().reshape(-1))
    p0.close()
    p1.close()


def test_call_order_errors(artifacts):
    from paper_2309_13541_b200.executor import ExecutorError, Plan
    a = artifacts("torus2x4")
    with Plan(a.g, a.sched, m=64) as p:
        s = torch.zeros((8, 8, 64), dtype=torch.uint8, device="cuda")
        with pytest.raises((ExecutorError, TypeError)):
            p.execute(s)                      # not bound
        p.bind(0)
        with pytest.raises(ExecutorError):
            p.set_engine("lsu")               # after bind
        with pytest.raises(ExecutorError):
            p.bind(0)                         # twice


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4_h2", "ts_hypercube3"])
@pytest.mark.parametrize("sched", ["static", "cp", "mix", "ll", "ll128"])
@pytest.mark.parametrize("engine", ["tma", "lsu"])
def test_cuda_graph_capture_and_replay(name, sched, engine, artifacts):
    """Executes captured into a CUDA graph replay as fresh all-to-alls: the
    epoch lives in device memory (advanced by the kernel), so every replay
    re-synchronises correctly without host involvement; the send buffer's
    contents change between replays, the pointers do not."""
    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    m = 4096 + 64
    with Plan(a.g, a.sched, m=m, protocol=sched if sched in ("ll", "ll128") else "simple") as p:
        p.set_engine(engine)
        if sched not in ("static", "ll", "ll128"):
            p.set_schedule(sched, 4096)
        p.bind(0)
        s = torch.empty((a.g.n, a.g.n, m), dtype=torch.uint8, device="cuda")
        r1, r2 = torch.zeros_like(s), torch.zeros_like(s)
        p.execute(s.zero_(), r1)      # warm-up outside capture
        p.sync()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            p.execute(s, r1)
            p.execute(r1, r2)         # transpose of the transpose = the input
        for rep in range(4):
            s.copy_(torch.from_numpy(_send(a.g.n, m, seed=rep)).cuda())
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(r1, s.transpose(0, 1).contiguous()), rep
            assert torch.equal(r2, s), rep
        # and direct executes still work after replays (same device epoch)
        p.execute(s, r1)
        p.sync()
        assert torch.equal(r1, s.transpose(0, 1).contiguous())


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("m", [7, 1000, 4096 + 5, 65536, 123457])
@pytest.mark.parametrize("engine", ["tma", "lsu"])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ll_protocol_bit_exact(name, m, engine, proto, artifacts):
    """A2A_PROTO_LL on one GPU: every hop through polled landing lines (no
    flags); bit-exact vs the oracle over repeated executes (both landing
    parities), device link counters equal the schedule."""
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    with Plan(a.g, a.sched, m=m, protocol=proto) as p:
        p.set_engine(engine)
        p.bind(0)
        p.set_timeout(10.0)
        for rep in range(3):
            send = _send(a.g.n, m, seed=rep + 11)
            _, want, _ = replay_bytes(a.g, a.sched, send, m)
            s = torch.from_numpy(send).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), rep
        assert np.array_equal(p.read_link_counters(), 3 * p.link_bytes())


@pytest.mark.parametrize("name,m", [("torus4x4x4", 4096 + 8), ("gk64_4", 2048 + 5), ("gk64_4_h2", 1000)])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ll_protocol_n64(name, m, proto, artifacts):
    """LL on the N=64 schedules (13 943 / 27k hop-ops, forwards split across
    several arrivals): transpose on one GPU, twice (both landing parities)."""
    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    g = torch.Generator(device="cuda").manual_seed(9)
    s = torch.randint(0, 256, (64, 64, m), dtype=torch.uint8, device="cuda", generator=g)
    with Plan(a.g, a.sched, m=m, protocol=proto) as p:
        p.bind(0)
        for _ in range(2):
            r = torch.zeros_like(s)
            p.execute(s, r)
            p.sync()
            assert torch.equal(r, s.transpose(0, 1).contiguous())


@pytest.mark.parametrize("name,G", [("gk8_2", 4), ("gk8_2", 8), ("hypercube3", 8), ("torus4x4x4", 8)])
@pytest.mark.parametrize("mode", ["static", "mix", "cp", "ready"])
def test_balanced_lowering_one_gpu(name, G, mode, artifacts):
    """The step-balanced lowering (bench.py autotune at >= 2 GPUs) of a
    G-GPU placement, run with every node on one GPU: bit-exact vs the oracle
    replaying the same lowered schedule, link counters exact."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    m = 4096 + 5 if a.g.n == 8 else 1024
    b, _ = bench.balanced_artifact(a, 16 << 20, G, "optimized")
    with Plan(b.g, b.sched, m=m) as p:
        if mode != "static":
            p.set_schedule(mode, 1024)
        p.bind(0)
        for rep in range(2):
            send = _send(b.g.n, m, seed=rep + G)
            _, want, _ = replay_bytes(b.g, b.sched, send, m)
            s = torch.from_numpy(send).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), rep
        assert np.array_equal(p.read_link_counters(), 2 * p.link_bytes())


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4", "hypercube3", "torus2x4_h2", "ts_gk8_2"])
@pytest.mark.parametrize("m,unit", [(1 << 20, 262144), ((1 << 20) + 48, 262144), (4096 + 5, 0),
                                    (4 << 20, 196608)])
@pytest.mark.parametrize("engine", ["tma", "lsu"])
@pytest.mark.parametrize("mode", ["chain", "chaind"])
def test_chain_schedule_bit_exact(name, m, unit, engine, mode, artifacts):
    """Chain mode on the device (a2a_chain_kernel): the TMA ring streams each
    route's local hops through L2 (hop u+1 loads a chunk once hop u's store of
    it completed); odd sizes take the all-thread path.  Bit-exact vs the
    oracle over repeated executes, link counters exact."""
    from paper_2309_13541_b200.executor import Plan
    from replay_bytes import replay_bytes
    a = artifacts(name)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_schedule(mode, unit)
        p.set_engine(engine)
        p.bind(0)
        for rep in range(3):
            send = _send(a.g.n, m, seed=rep + 21)
            _, want, _ = replay_bytes(a.g, a.sched, send, m)
            s = torch.from_numpy(send).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), rep
        assert np.array_equal(p.read_link_counters(), 3 * p.link_bytes())


@pytest.mark.parametrize("name,m", [("torus4x4x4", 4 << 20), ("gk64_4", 1 << 20), ("gk256_4", 65536)])
@pytest.mark.parametrize("mode", ["chain", "chaind"])
def test_chain_large_transpose(name, m, mode, artifacts):
    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    n = a.g.n
    g = torch.Generator(device="cuda").manual_seed(13)
    s = torch.randint(0, 256, (n, n, m), dtype=torch.uint8, device="cuda", generator=g)
    r = torch.zeros_like(s)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_schedule(mode, 262144)
        p.bind(0)
        for _ in range(2):
            p.execute(s, r, count_links=True)
            p.sync()
        assert np.array_equal(p.read_link_counters(), 2 * p.link_bytes())
    assert torch.equal(r, s.transpose(0, 1).contiguous())


@pytest.mark.parametrize("mode", ["chain", "chaind"])
def test_chain_with_self_copy_and_graph(mode, artifacts):
    """Chains with the self shards copied too, and captured into a CUDA graph:
    every replay is a fresh all-to-all (the grab counter base follows the
    device epoch)."""
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("gk8_2")
    m = 1 << 20
    with Plan(a.g, a.sched, m=m, copy_self=True) as p:
        p.set_schedule(mode, 262144)
        p.bind(0)
        s = torch.empty((8, 8, m), dtype=torch.uint8, device="cuda")
        r = torch.zeros_like(s)
        p.execute(s.zero_(), r)
        p.sync()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            p.execute(s, r)
        for rep in range(3):
            s.copy_(torch.from_numpy(_send(8, m, seed=40 + rep)).cuda())
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(r, s.transpose(0, 1).contiguous()), rep
