"""GPU parity on the BASELINE.json configurations, one GPU.

* config 4 — GenKautz N=256, d=4, with (``gk256_4``) and without
  (``gk256_4_h2``, host bottleneck 2.0, routes collapsed to physical nodes)
  extra NIC-forwarding bandwidth (reference graphs.py:130-153, :447-475;
  tests/test_acceptance.py:47-50): 255 890 hop-ops over 9 steps.  At a small
  odd shard size the receive buffers are compared byte for byte with the C
  oracle (oracle/replay_bytes.c, the restatement pinned to the reference's
  replay by tests/test_oracle.py; the Python oracle is too slow at this size)
  and the device per-(step, link) byte counters with the oracle's link bytes.
  At 64 KiB: transpose + counters == schedule.
* config 1 — 2x4 torus at exactly 1 MiB per pair: bit-exact vs the oracle.
* config 3 — 4x4x4 torus at exactly 4 MiB per pair (13 943 hop-ops):
  transpose + counters, static programs and the unit queues bench.py uses.
"""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _dev_send(n, m, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randint(0, 256, (n, n, m), dtype=torch.uint8, device="cuda", generator=g)


def _oracle_links(a, lb):
    return np.asarray(lb, dtype=np.int64).reshape(a.sched.nsteps, len(a.g.edges))


@pytest.mark.parametrize("name", ["gk256_4", "gk256_4_h2"])
@pytest.mark.parametrize("sched", ["static", "cp:1048576"])
def test_gk256_one_gpu_bit_exact_vs_c_oracle(name, sched, artifacts):
    """Config 4 on one GPU at m=4101 (breaks 16-byte alignment): recv and
    per-link bytes equal the C oracle's replay of the same schedule."""
    from c_oracle import replay_bytes_c
    from replay_bytes import make_send

    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    n, m = a.g.n, 4101
    send = make_send(n, m, seed=41)
    _, want, lb = replay_bytes_c(a.g, a.sched, send, m)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_schedule_spec(sched)
        p.bind(0)
        s = torch.from_numpy(send).cuda()
        r = torch.zeros_like(s)
        p.execute(s, r, count_links=True)
        p.sync()
        dev = p.read_link_counters()
        sched_bytes = p.link_bytes()
    assert np.array_equal(r.cpu().numpy(), want)
    assert np.array_equal(sched_bytes, _oracle_links(a, lb))
    assert np.array_equal(dev, sched_bytes)


@pytest.mark.parametrize("name", ["gk256_4", "gk256_4_h2"])
def test_gk256_one_gpu_64k_transpose_and_counters(name, artifacts):
    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    n, m = a.g.n, 65536
    s = _dev_send(n, m, seed=256)
    with Plan(a.g, a.sched, m=m) as p:
        p.bind(0)
        for rep in range(2):
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert torch.equal(r, s.transpose(0, 1).contiguous()), rep
        assert np.array_equal(p.read_link_counters(), 2 * p.link_bytes())
    del s, r


def test_torus2x4_1mib_bit_exact(artifacts):
    """Config 1 (2x4 torus, decomposed MCF, 1 MiB per pair) vs the oracle."""
    from replay_bytes import make_send, replay_bytes

    from paper_2309_13541_b200.executor import Plan
    a = artifacts("torus2x4")
    m = 1 << 20
    send = make_send(a.g.n, m, seed=1)
    _, want, ob = replay_bytes(a.g, a.sched, send, m)
    ref = np.zeros((a.sched.nsteps, len(a.g.edges)), dtype=np.int64)
    for (t, e), x in ob.items():
        ref[t, e] = x
    for sched in ("static", "cp:1048576", "ll", "ll128"):
        proto = sched if sched in ("ll", "ll128") else "simple"
        with Plan(a.g, a.sched, m=m, protocol=proto) as p:
            if proto == "simple":
                p.set_schedule_spec(sched)
            p.bind(0)
            s = torch.from_numpy(send).cuda()
            r = torch.zeros_like(s)
            p.execute(s, r, count_links=True)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), sched
            assert np.array_equal(p.read_link_counters(), ref), sched


@pytest.mark.parametrize("sched", ["static", "cp:1048576", "mix:1048576"])
def test_torus4x4x4_4mib_transpose_and_counters(sched, artifacts):
    """Config 3 workload (4x4x4 torus, 4 MiB per pair) with all 64 virtual
    nodes on one GPU: 16 GiB send + 16 GiB recv + forwarding scratch."""
    from paper_2309_13541_b200.executor import Plan
    a = artifacts("torus4x4x4")
    n, m = a.g.n, 4 << 20
    s = _dev_send(n, m, seed=64)
    r = torch.zeros_like(s)
    with Plan(a.g, a.sched, m=m) as p:
        p.set_schedule_spec(sched)
        p.bind(0)
        p.execute(s, r, count_links=True)
        p.sync()
        assert np.array_equal(p.read_link_counters(), p.link_bytes())
    assert torch.equal(r, s.transpose(0, 1).contiguous())
    del s, r


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4_h2", "ts_hypercube3"])
@pytest.mark.parametrize("sched", ["static", "cp:1048576", "spread:1048576", "ll", "ll128"])
def test_without_self_copy(name, sched, artifacts):
    """copy_self=False, as bench.py times it: every s != d shard bit-exact vs
    the oracle, the self rows of recv untouched (the reference transpose
    skips s == d, evaluate.py:114-118)."""
    from replay_bytes import make_send, replay_bytes

    from paper_2309_13541_b200.executor import Plan
    a = artifacts(name)
    m = 65536 + 40
    send = make_send(a.g.n, m, seed=3)
    _, want, _ = replay_bytes(a.g, a.sched, send, m, copy_self=False)
    with Plan(a.g, a.sched, m=m, copy_self=False,
              protocol=sched if sched in ("ll", "ll128") else "simple") as p:
        if sched not in ("ll", "ll128"):
            p.set_schedule_spec(sched)
        p.bind(0)
        s = torch.from_numpy(send).cuda()
        for rep in range(2):
            r = torch.full_like(s, 0xA5)
            p.execute(s, r)
            p.sync()
            got = r.cpu().numpy()
            for v in range(a.g.n):
                assert (got[v, v] == 0xA5).all(), (rep, v)
                got[v, v] = 0
            assert np.array_equal(got, want), rep
