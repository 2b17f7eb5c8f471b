"""Multi-GPU parity: one process per GPU, CUDA IPC arenas, NVLink peer stores.

Each rank binds the G-GPU plan to its own device, exchanges arena handles
through torch.distributed (gloo, plumbing only), executes, and checks its recv
rows against the oracle's; device link counters summed over ranks equal the
schedule.  A single-process variant drives G devices with peer pointers.
Skipped when fewer than 2 GPUs are visible.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _reap(ps):
    """Join the rank processes; kill any that linger (so no child keeps a GPU
    context alive after the test)."""
    for p in ps:
        p.join(timeout=60)
    for p in ps:
        if p.is_alive():
            p.kill()
            p.join(timeout=10)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, name, m, reps, q, engine="lsu", sched="static", reuse=False,
               proto="simple", graph=False, lowering="hop", sync_mode=None):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import torch
        import torch.distributed as dist
        from replay_bytes import make_send, replay_bytes

        from paper_2309_13541_b200.artifacts import load_artifact
        from paper_2309_13541_b200.dist import connect, disconnect, local_nodes
        from paper_2309_13541_b200.executor import Plan
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                                rank=rank, world_size=world)
        a = load_artifact(name)
        placement = "optimized"
        if lowering == "balanced":            # bench.py's step-balanced lowering
            sys.path.insert(0, ROOT)
            import bench
            a, placement = bench.balanced_artifact(a, m, world, "optimized")
        plan = Plan(a.g, a.sched, m=m, n_gpus=world, reuse_scratch=reuse, placement=placement,
                    protocol=proto)
        plan.set_engine(engine)
        plan.set_schedule_spec(sched)      # "<mode>[:<unit bytes>[:<pinned NVLink CTAs>]]"
        plan.bind(rank, device=rank)
        plan.set_timeout(20.0)
        if sync_mode is not None:
            plan.set_sync_mode(sync_mode)
        connect(plan)
        nodes = local_nodes(plan, rank)
        # LL: only local CTAs write recv, so any device buffer works
        recv = plan.recv_buffer() if proto not in ("ll", "ll128") else torch.empty(
            (len(nodes), a.g.n, m), dtype=torch.uint8, device=f"cuda:{rank}")
        ok = True
        if proto in ("ll", "ll128"):
            # back-to-back all-to-alls, no host sync in between: exercises the
            # epoch-parity landing regions and the lagged entry flags
            K = 6
            sends_all = [make_send(a.g.n, m, seed=300 + k) for k in range(K)]
            sends = [torch.from_numpy(np.ascontiguousarray(x[nodes])).cuda(rank) for x in sends_all]
            outs = [torch.empty_like(recv) for _ in range(K)]
            for k in range(K):
                plan.execute(sends[k], outs[k])
            plan.sync()
            for k in range(K):
                ok &= bool(np.array_equal(outs[k].cpu().numpy(), np.swapaxes(sends_all[k], 0, 1)[nodes]))
            dist.barrier()
        for rep in range(reps):
            send_all = make_send(a.g.n, m, seed=100 + rep)
            send = torch.from_numpy(np.ascontiguousarray(send_all[nodes])).cuda(rank)
            plan.execute(send, recv, count_links=True)
            plan.sync()
            want = np.swapaxes(send_all, 0, 1)[nodes]
            ok &= bool(np.array_equal(recv.cpu().numpy(), want))
            dist.barrier()
        if graph:
            # one execute captured into a CUDA graph, replayed with new send
            # contents: device-side epochs keep the ranks in step
            send = torch.empty((len(nodes), a.g.n, m), dtype=torch.uint8, device=f"cuda:{rank}")
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                plan.execute(send, recv)
            for rep in range(4):
                send_all = make_send(a.g.n, m, seed=700 + rep)
                send.copy_(torch.from_numpy(np.ascontiguousarray(send_all[nodes])))
                dist.barrier()
                g.replay()
                torch.cuda.synchronize(rank)
                ok &= bool(np.array_equal(recv.cpu().numpy(), np.swapaxes(send_all, 0, 1)[nodes]))
                dist.barrier()
        counters = plan.read_link_counters()
        tot = [None] * world
        dist.all_gather_object(tot, counters)
        summed = sum(tot)
        _, _, ob = replay_bytes(a.g, a.sched, make_send(a.g.n, m), m)
        ref = np.zeros_like(summed)
        for (t, e), x in ob.items():
            ref[t, e] = x * reps
        q.put((rank, ok, bool(np.array_equal(summed, ref))))
        disconnect(plan)
        dist.destroy_process_group()
    except Exception as ex:
        import traceback
        q.put((rank, f"{ex!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("engine", ["lsu", "tma"])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,m", [("torus2x4", 4096 + 7), ("gk8_2", 65536),
                                    ("hypercube3", 1 << 20), ("torus4x4x4", 8192)])
def test_multiprocess_ipc(world, name, m, engine):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main, args=(r, world, port, name, m, 3, q, engine))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,m,engine", [
    ("torus2x4", 4096 + 7, "tma"), ("gk8_2", 65536, "tma"), ("hypercube3", 4096, "tma"),
    ("torus4x4x4", 2048, "tma"), ("ts_gk8_2", 1000, "tma"), ("gk8_2", 20000, "lsu"),
    ("torus2x4", 333, "lsu"), ("hypercube3", 1 << 20, "lsu")])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_multiprocess_ll(world, name, m, engine, proto):
    """A2A_PROTO_LL / LL128 across GPUs: bit-exact recv (also back-to-back
    without host sync), device link counters equal the schedule."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, name, m, 3, q, engine, "static", False, proto))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("proto,sched", [("simple", "static"), ("ll", "static"), ("ll128", "static"),
                                         ("simple", "cp")])
def test_multiprocess_cuda_graph(world, proto, sched):
    """Executes captured into CUDA graphs on every rank, replayed repeatedly."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, "gk8_2", 20000, 1, q, "tma", sched, False, proto, True))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


def test_single_process_peer_pointers():
    """One process drives two GPUs through cudaDeviceEnablePeerAccess pointers."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    from replay_bytes import make_send

    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.dist import local_nodes
    from paper_2309_13541_b200.executor import Plan
    a = load_artifact("gk8_2")
    m = 10000
    plans = [Plan(a.g, a.sched, m=m, n_gpus=2).bind(r, device=r) for r in range(2)]
    ptrs = [p.arena_ptr() for p in plans]
    for p in plans:
        p.import_pointers(ptrs)
    send_all = make_send(8, m, seed=4)
    sends, recvs = [], []
    for r, p in enumerate(plans):
        nodes = local_nodes(p, r)
        sends.append(torch.from_numpy(np.ascontiguousarray(send_all[nodes])).cuda(r))
        recvs.append(p.recv_buffer())
    for r, p in enumerate(plans):
        p.execute(sends[r], recvs[r])
    for p in plans:
        p.sync()
    for r, p in enumerate(plans):
        want = np.swapaxes(send_all, 0, 1)[local_nodes(p, r)]
        assert np.array_equal(recvs[r].cpu().numpy(), want)
    for p in plans:
        p.close()


def _alt_main(rank, world, port, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    try:
        import torch
        import torch.distributed as dist
        from replay_bytes import make_send

        from paper_2309_13541_b200.artifacts import load_artifact
        from paper_2309_13541_b200.dist import connect, disconnect, local_nodes
        from paper_2309_13541_b200.executor import Plan
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                                rank=rank, world_size=world)
        a = load_artifact("gk8_2")
        m = 20000
        plan = Plan(a.g, a.sched, m=m, n_gpus=world).set_recv_buffers(2)
        plan.bind(rank, device=rank)
        connect(plan)
        nodes = local_nodes(plan, rank)
        bufs = [plan.recv_buffer(0), plan.recv_buffer(1)]
        ok = True
        wants = []
        for k in range(4):
            send_all = make_send(8, m, seed=50 + k)
            send = torch.from_numpy(np.ascontiguousarray(send_all[nodes])).cuda(rank)
            plan.execute(send, bufs[k & 1])
            wants.append(np.swapaxes(send_all, 0, 1)[nodes])
            plan.sync()
            if k >= 1:  # the other buffer still holds the previous all-to-all
                ok &= bool(np.array_equal(bufs[(k - 1) & 1].cpu().numpy(), wants[k - 1]))
            ok &= bool(np.array_equal(bufs[k & 1].cpu().numpy(), wants[k]))
        q.put((rank, ok))
        disconnect(plan)
        dist.destroy_process_group()
    except Exception as ex:
        import traceback
        q.put((rank, f"{ex!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("world,engine,reuse,name,m", [
    (2, "tma", False, "gk8_2", 65536 + 64), (4, "tma", True, "torus4x4x4", 8192),
    (2, "lsu", True, "torus2x4_h2", 4099), (4, "lsu", False, "gk8_2", 65536 + 64),
    (4, "tma", False, "torus2x4_h2", 4099)])
@pytest.mark.parametrize("mode", ["dynamic", "list", "cp", "mix", "ready", "spread"])
def test_multiprocess_dynamic(world, engine, reuse, name, m, mode):
    """Dynamic unit queues across GPUs (+ scratch reuse, optimized placement)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, name, m, 3, q, engine, mode, reuse))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,m", [("gk8_2", 65536 + 64), ("hypercube3", 4099)])
@pytest.mark.parametrize("mode", ["static", "mix:4096", "cp:4096:64", "spread:4096", "ready:4096"])
def test_multiprocess_balanced_lowering(world, name, m, mode):
    """The step-balanced lowering bench.py's autotune tries at >= 4 GPUs:
    bit-exact recv and exact link counters across processes."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, name, m, 2, q, "tma", mode, False, "simple", False,
                            "balanced"))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("world,engine,name,m", [(2, "tma", "gk8_2", 65536 + 64),
                                                 (4, "lsu", "torus2x4_h2", 4099)])
@pytest.mark.parametrize("mode", ["cp:0:3", "dynamic:4096:40"])
def test_multiprocess_pinned_split(world, engine, name, m, mode):
    """Pinned NVLink/HBM queue split (a2a_plan_set_queue_split) across GPUs,
    repeated executes (the per-epoch grab-counter base of pinned queues)."""
    test_multiprocess_dynamic(world, engine, False, name, m, mode)


def test_alternating_recv_buffers():
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_alt_main, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in res:
        assert r[1] is True, r


def _gk256_main(rank, world, port, name, sched, q):
    sys.path.insert(0, ROOT)
    try:
        import torch
        import torch.distributed as dist

        from paper_2309_13541_b200.artifacts import load_artifact
        from paper_2309_13541_b200.dist import connect, disconnect, local_nodes
        from paper_2309_13541_b200.executor import Plan
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                                rank=rank, world_size=world)
        a = load_artifact(name, native=True)
        m = 8192 + 64
        plan = Plan(a.g, a.sched, m=m, n_gpus=world, placement="optimized",
                    protocol="ll" if sched == "ll" else "simple")
        if sched != "ll":
            plan.set_schedule(sched)
        plan.bind(rank, device=rank)
        plan.set_timeout(30.0)
        connect(plan)
        nodes = local_nodes(plan, rank)
        n = a.g.n

        def row(s):   # deterministic shard rows of node s, generated on the device
            gen = torch.Generator(device="cuda").manual_seed(977 * (s + 1))
            return torch.randint(0, 256, (n, m), dtype=torch.uint8, device="cuda", generator=gen)
        send = torch.stack([row(v) for v in nodes])
        recv = plan.recv_buffer()
        plan.execute(send, recv, count_links=True)
        plan.sync()
        ok = True
        for s in range(n):
            r = row(s)
            ok &= bool(torch.equal(recv[:, s], r[nodes]))
        counters = plan.read_link_counters()
        tot = [None] * world
        dist.all_gather_object(tot, counters)
        q.put((rank, ok, bool(np.array_equal(sum(tot), plan.link_bytes()))))
        disconnect(plan)
        dist.destroy_process_group()
    except Exception as ex:
        import traceback
        q.put((rank, f"{ex!r}\n{traceback.format_exc()}"))


@pytest.mark.parametrize("name", ["gk256_4", "gk256_4_h2"])
@pytest.mark.parametrize("sched", ["static", "dynamic", "ll"])
def test_gk256_four_gpus(name, sched):
    """Config 4 (GenKautz N=256, with / without extra NIC forwarding) on 4 GPUs:
    transpose of device-generated shards, device link counters == schedule."""
    if _ngpu() < 4:
        pytest.skip("needs 4 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_gk256_main, args=(r, 4, port, name, sched, q)) for r in range(4)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("name,m", [("gk8_2", 65536), ("hypercube3", 4096 + 7), ("gk64_4", 2048)])
@pytest.mark.parametrize("proto,sched", [("simple", "static"), ("simple", "cp"), ("simple", "mix"),
                                         ("simple", "ready"), ("ll", "static"), ("ll128", "static"),
                                         ("simple", "spread"), ("simple", "chain")])
@pytest.mark.parametrize("lowering", ["hop", "balanced"])
def test_eight_ranks_single_process(name, m, proto, sched, lowering):
    """The 8-GPU code paths (8 peers, 8-bit destination masks, per-GPU exit
    lists) on real hardware with fewer devices: 8 plans of an 8-GPU placement
    in one process, rank r on device r % ndev, each with a reduced CTA count so
    the ranks sharing a device are co-resident, launched on their own streams."""
    ndev = _ngpu()
    if ndev < 2:
        pytest.skip("needs 2 GPUs")
    from replay_bytes import make_send

    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.dist import local_nodes
    from paper_2309_13541_b200.executor import Plan
    a = load_artifact(name)
    R = 8
    placement = "optimized"
    if lowering == "balanced":        # bench.py's 8-GPU lowering (route pieces, extra step)
        sys.path.insert(0, ROOT)
        import bench
        a, placement = bench.balanced_artifact(a, 16 << 20, R, "optimized")
    per_dev = -(-R // ndev)
    nc = max(8, 144 // per_dev)
    plans = []
    # plain (non-cooperative) launches: kernels of ranks sharing a device must
    # run concurrently from different streams
    old_env = os.environ.get("A2A_NONCOOP")
    os.environ["A2A_NONCOOP"] = "1"
    try:
        for r in range(R):
            p = Plan(a.g, a.sched, m=m, n_gpus=R, placement=placement, protocol=proto)
            if sched != "static":
                p.set_schedule(sched, 4096)
            plans.append(p.bind(r, device=r % ndev, num_ctas=nc))
    finally:
        if old_env is None:
            os.environ.pop("A2A_NONCOOP", None)
        else:
            os.environ["A2A_NONCOOP"] = old_env
    ptrs = [p.arena_ptr() for p in plans]
    for p in plans:
        p.import_pointers(ptrs)
        p.set_timeout(20.0)
    send_all = make_send(a.g.n, m, seed=8)
    want = np.swapaxes(send_all, 0, 1)
    nodes = [local_nodes(p, r) for r, p in enumerate(plans)]
    streams = [torch.cuda.Stream(r % ndev) for r in range(R)]
    sends = [torch.from_numpy(np.ascontiguousarray(send_all[nodes[r]])).cuda(r % ndev) for r in range(R)]
    recvs = [p.recv_buffer() for p in plans]
    for rep in range(2):
        for r, p in enumerate(plans):
            p.execute(sends[r], recvs[r], stream=streams[r], count_links=True)
        for p in plans:
            p.sync()
        for r in range(R):
            assert np.array_equal(recvs[r].cpu().numpy(), want[nodes[r]]), (rep, r)
    total = sum(p.read_link_counters() for p in plans)
    assert np.array_equal(total, 2 * plans[0].link_bytes())
    for p in plans:
        p.close()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,m", [("gk8_2", 1 << 20), ("torus4x4x4", 262144), ("hypercube3", (1 << 20) + 48)])
@pytest.mark.parametrize("lowering", ["hop", "balanced"])
def test_multiprocess_chain(world, name, m, lowering):
    """Chain mode across GPUs: local hop chains stream on one CTA, chains break
    at GPU boundaries (flags + exit wait as for the unit queues)."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, name, m, 2, q, "tma", "chain:262144", False, "simple",
                            False, lowering))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("name,m,engine,proto,sched", [
    ("gk8_2", 1 << 20, "tma", "simple", "static"),
    ("gk8_2", 65536 + 64, "lsu", "simple", "static"),
    ("gk8_2", 1 << 20, "tma", "simple", "cp:262144"),
    ("hypercube3", 1 << 20, "tma", "simple", "spread:262144"),
    ("torus4x4x4", 65536, "tma", "simple", "mix:65536"),
    ("gk8_2", 1 << 20, "tma", "simple", "chain:262144"),
    ("hypercube3", 65536 + 40, "lsu", "ll128", "static"),
    ("torus2x4_h2", 4096 + 7, "lsu", "ll", "static")])
def test_multiprocess_perturbed(world, name, m, engine, proto, sched):
    """Race hunting across GPUs (tests/test_gpu_race.py): every CTA naps a
    pseudo-random 0-16 us (1 in 16: up to 260 us) before each step / unit /
    task (sync_mode bit 6), so producers and consumers on different GPUs
    finish in new orders every repeat; every repeat is bit-exact."""
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, name, m, 4, q, engine, sched, False, proto,
                            False, "hop", 2 | 64))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    for r in sorted(res, key=lambda x: x[0]):
        assert len(r) == 3, r
        assert r[1], f"rank {r[0]}: recv mismatch"
        assert r[2], f"rank {r[0]}: link counters differ from schedule"


@pytest.mark.parametrize("sched", ["static", "cp:262144"])
def test_multiprocess_mutation_without_waits_is_caught(sched, monkeypatch):
    """The same perturbation with the dependency waits skipped (bit 7) must
    give a wrong transpose on some rank."""
    world = 2
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    import torch.multiprocessing as mp
    monkeypatch.setenv("A2A_ALLOW_MUTATION", "1")     # inherited by the spawned ranks
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main,
                      args=(r, world, port, "gk8_2", 1 << 20, 8, q, "tma", sched, False, "simple",
                            False, "hop", 2 | 64 | 128))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    _reap(ps)
    assert all(len(r) == 3 for r in res), res
    assert not all(r[1] for r in res), "dropped dependencies went unnoticed"
