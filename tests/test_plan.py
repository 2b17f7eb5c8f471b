"""Native plan builder (host side of the C ABI) against the reference and the oracle.

No GPU needed: a2a_plan_create validates exactly like the reference replay
(evaluate.py:56-127), a2a_plan_model_time reproduces its T bit-for-bit, and
a2a_plan_link_bytes is the per-(step, link) byte load the kernels must move.
"""
from __future__ import annotations

import copy

import numpy as np
import pytest

from conftest import apply_edit
from paper_2309_13541_b200.executor import (EvalError, Plan, contiguous_placement,
                                            replay_timestep_schedule)
from replay_bytes import make_send, replay_bytes

ALL = ["torus2x4", "hypercube3", "gk8_2", "torus2x4_h1", "torus2x4_h2", "gk8_2_h1",
       "ts_ring3", "ts_torus2x4", "ts_hypercube3", "ts_gk8_2", "ts_torus3x3",
       "torus4x4x4", "gk64_4", "gk64_4_h2", "gk256_4", "gk256_4_h2"]


def _available(names):
    import json
    import os
    from paper_2309_13541_b200.artifacts import list_artifacts
    have = set(list_artifacts())
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.json")) as fh:
        gold = set(json.load(fh)["configs"])
    return [n for n in names if n in have and n in gold]


@pytest.mark.parametrize("name", _available(ALL))
def test_native_T_bit_identical_to_reference(name, golden, artifacts):
    a = artifacts(name)
    for (m, b, sync), want in zip(golden["params"], golden["configs"][name]["replay"]):
        T, ok = replay_timestep_schedule(a.g, a.sched, m=m, b=b, sync_latency=sync)
        assert ok is True and repr(T) == want["T"]


@pytest.mark.parametrize("name", _available(ALL))
def test_native_link_bytes_equal_schedule(name, golden, artifacts):
    a = artifacts(name)
    Q = a.sched.Q
    m = Q * 3
    with Plan(a.g, a.sched, m=m) as p:
        lb = p.link_bytes()
    want = np.zeros_like(lb)
    for k, c in golden["configs"][name]["link_chunks"].items():
        t, e = map(int, k.split(","))
        want[t, e] = c * 3
    assert np.array_equal(lb, want)


@pytest.mark.parametrize("name", ["torus2x4", "gk8_2", "ts_torus3x3", "torus2x4_h2"])
@pytest.mark.parametrize("m", [1, 5, 999])
def test_native_link_bytes_equal_oracle_any_m(name, m, artifacts):
    a = artifacts(name)
    _, _, ob = replay_bytes(a.g, a.sched, make_send(a.g.n, m), m)
    with Plan(a.g, a.sched, m=m) as p:
        lb = p.link_bytes()
    want = np.zeros_like(lb)
    for (t, e), x in ob.items():
        want[t, e] = x
    assert np.array_equal(lb, want)


@pytest.mark.parametrize("name", ["torus2x4", "gk8_2", "ts_ring3", "ts_hypercube3",
                                  "torus2x4_h2"])
def test_native_rejects_like_reference(name, golden, artifacts):
    a = artifacts(name)
    for case in golden["configs"][name]["corruptions"]:
        s = apply_edit(a.sched, case["edit"])
        want = case["replay"]
        if "error" in want:
            with pytest.raises(EvalError) as ei:
                Plan(a.g, s, m=64)
            assert str(ei.value) == want["error"], case["label"]
        else:
            T, ok = replay_timestep_schedule(a.g, s, m=1.0)
            assert ok and repr(T) == want["T"], case["label"]


def test_mode_and_node_count_errors(artifacts):
    a = artifacts("torus2x4")
    with pytest.raises(EvalError, match="expects a ts-mode schedule"):
        replay_timestep_schedule(a.g, a.path_sched)
    s = copy.deepcopy(a.sched)
    s.n = 9
    with pytest.raises(EvalError, match="graph has 8 nodes, schedule says 9"):
        replay_timestep_schedule(a.g, s)


def test_reference_replay_kats(artifacts):
    """tests/test_evaluate.py:22-37 of the reference, on the native replay."""
    a = artifacts("ts_ring3")
    T, ok = replay_timestep_schedule(a.g, a.sched, m=1.0, b=1.0)
    assert ok and T == pytest.approx(3.0)
    T2, _ = replay_timestep_schedule(a.g, a.sched, b=2.0)
    assert T2 == pytest.approx(T / 2)
    T3, _ = replay_timestep_schedule(a.g, a.sched, sync_latency=0.25)
    assert T3 == pytest.approx(T + 0.25 * a.sched.nsteps)


def test_reference_missing_chunk_kat(artifacts):
    """tests/test_evaluate.py:39-59: drop node 0's step-0 sends of shard (*,2)."""
    a = artifacts("ts_ring3")
    s = copy.deepcopy(a.sched)
    s.instructions = [i for i in s.instructions if not (i.t == 0 and i.src == 0 and i.d == 2)]
    with pytest.raises(EvalError):
        Plan(a.g, s, m=4)
    from paper_2309_13541_b200.schedule import Instruction
    s = copy.deepcopy(a.sched)
    s.instructions.append(Instruction(t=0, src=0, dst=2, s=0, d=2, c0=0, c1=1))
    with pytest.raises(EvalError, match="no link"):
        Plan(a.g, s, m=4)


@pytest.mark.parametrize("name,G", [("torus2x4", 2), ("hypercube3", 4), ("gk8_2", 8),
                                    ("torus4x4x4", 8), ("gk64_4", 8)])
def test_gpu_info_consistent(name, G, artifacts):
    a = artifacts(name)
    m = 1 << 20
    with Plan(a.g, a.sched, m=m, n_gpus=G) as p:
        infos = [p.gpu_info(g) for g in range(G)]
        lb = p.link_bytes()
    assert sum(i["n_local_nodes"] for i in infos) == a.g.n
    assert sum(i["egress_bytes"] for i in infos) == sum(i["ingress_bytes"] for i in infos)
    assert sum(i["hop_bytes"] for i in infos) == int(lb.sum())
    place = contiguous_placement(a.g.n, G)
    # egress per GPU from the schedule's links directly
    eg = [0] * G
    for t in range(a.sched.nsteps):
        for e, (u, v, _) in enumerate(a.g.edges):
            if place[u] != place[v]:
                eg[place[u]] += int(lb[t, e])
    assert eg == [i["egress_bytes"] for i in infos]
    for i in infos:
        assert i["send_bytes"] == i["n_local_nodes"] * a.g.n * m


def test_exact_quantization_link_loads_equal_mcf(artifacts, golden):
    """Q exact (2x4 torus, hypercube): schedule bytes per link == MCF load x m."""
    for name in ("torus2x4", "hypercube3"):
        a = artifacts(name)
        m = 1 << 20
        with Plan(a.g, a.sched, m=m) as p:
            per_link = p.link_bytes().sum(axis=0)
        fluid = [float(x) for x in golden["configs"][name]["fluid_link_load"]]
        for e, x in enumerate(per_link):
            assert x == round(fluid[e] * m)
        assert set(per_link.tolist()) == {4 * m}


def test_plan_rejects_bad_args(artifacts):
    a = artifacts("torus2x4")
    with pytest.raises(ValueError):
        Plan(a.g, a.sched, m=-1)
    with pytest.raises(ValueError):
        Plan(a.g, a.sched, m=16, n_gpus=9)
    with pytest.raises(ValueError):
        Plan(a.g, a.sched, m=16, placement=[0] * 7)


def test_sync_mode_range(artifacts, monkeypatch):
    """Sync-mode bits 0-7 (bit 6 = perturbation, bit 7 = skipped waits for the
    mutation self-test); anything wider is rejected before it reaches a kernel."""
    a = artifacts("torus2x4")
    with Plan(a.g, a.sched, m=16) as p:
        for mode in (0, 2, 2 | 64, 63 | 64):
            p.set_sync_mode(mode)
        for bad in (-1, 256, 2 | 128, 255):     # bit 7 only with A2A_ALLOW_MUTATION=1
            with pytest.raises(ValueError, match="bad sync mode"):
                p.set_sync_mode(bad)
        monkeypatch.setenv("A2A_ALLOW_MUTATION", "1")
        p.set_sync_mode(2 | 64 | 128)
        p.set_sync_mode(255)
