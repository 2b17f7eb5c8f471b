"""Degenerate inputs of the executor path: one node (no commodities), two
nodes, empty shards (m = 0), shards smaller than Q, and an empty schedule.

The reference replay's contract on these (pkg/src/a2aflow/evaluate.py:56-127):
a 1-node graph has no shards, so the empty schedule is accepted with T = 0;
an empty schedule on >= 2 nodes fails the final delivery scan (:114-126) with
"shard (0,1) chunk 0 never delivered".  CPU: native validation, the oracle and
the emulated device protocol agree (T, acceptance and the message were checked
against the reference replay imported in the build container); GPU: the
kernels move the same bytes.
"""
from __future__ import annotations

import numpy as np
import pytest

from paper_2309_13541_b200.dist import local_nodes
from paper_2309_13541_b200.executor import EvalError, Plan, replay_timestep_schedule
from paper_2309_13541_b200.graphs import Digraph
from paper_2309_13541_b200.schedule import ChunkedSchedule, Instruction
from replay_bytes import OracleEvalError, make_send, replay_bytes


def _one_node():
    return (Digraph.from_edges(1, []),
            ChunkedSchedule(n=1, nsteps=0, chunk_bytes=1.0, Q=1, mode="ts", instructions=[]))


def _two_nodes():
    """0 -> 1 in one op; 1 -> 0 split into two chunk ranges; Q = 2."""
    g = Digraph.from_edges(2, [(0, 1, 1.0), (1, 0, 1.0)])
    ins = [Instruction(0, 0, 1, 0, 1, 0, 2), Instruction(0, 1, 0, 1, 0, 0, 1),
           Instruction(0, 1, 0, 1, 0, 1, 2)]
    return g, ChunkedSchedule(n=2, nsteps=1, chunk_bytes=1.0, Q=2, mode="ts", instructions=ins)


CASES = {"one_node": _one_node, "two_nodes": _two_nodes}


@pytest.mark.parametrize("case", list(CASES))
def test_replay_T(case):
    g, s = CASES[case]()
    T, ok = replay_timestep_schedule(g, s, m=3)
    want, _, _ = replay_bytes(g, s, make_send(g.n, 3, seed=0), 3)
    assert ok and T == want == (0.0 if case == "one_node" else 3.0)


def test_empty_schedule_never_delivered():
    g, _ = _two_nodes()
    s = ChunkedSchedule(n=2, nsteps=1, chunk_bytes=1.0, Q=1, mode="ts", instructions=[])
    with pytest.raises(EvalError, match=r"^shard \(0,1\) chunk 0 never delivered$"):
        replay_timestep_schedule(g, s)
    with pytest.raises(OracleEvalError, match=r"^shard \(0,1\) chunk 0 never delivered$"):
        replay_bytes(g, s, make_send(2, 4, seed=0), 4)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("m", [0, 1, 3, 4096 + 7])
@pytest.mark.parametrize("mode", ["static", "cp", "spread", "ready", "ll"])
def test_emulated_edge_cases(case, m, mode):
    g, s = CASES[case]()
    send = make_send(g.n, m, seed=m)
    _, want, _ = replay_bytes(g, s, send, m)
    assert np.array_equal(want, np.swapaxes(send, 0, 1))
    for G in range(1, g.n + 1):
        with Plan(g, s, m=m, n_gpus=G, protocol="ll" if mode == "ll" else "simple") as p:
            if mode not in ("static", "ll"):
                p.set_schedule(mode, 64)
            p.check_bounds(5)
            nodes = [local_nodes(p, k) for k in range(G)]
            for nC in (1, 5):
                recvs = p.emulate([send[ns] for ns in nodes], num_ctas=nC, seed=nC)
                for k in range(G):
                    assert np.array_equal(recvs[k], want[nodes[k]]), (G, nC, k)


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("m", [0, 1, 4096 + 7])
@pytest.mark.parametrize("mode", ["static", "cp", "ll"])
@pytest.mark.parametrize("engine", ["tma", "lsu"])
def test_gpu_edge_cases(case, m, mode, engine):
    """One GPU, all nodes local: bit-exact recv over repeated executes."""
    import torch
    g, s = CASES[case]()
    with Plan(g, s, m=m, protocol="ll" if mode == "ll" else "simple") as p:
        if mode == "cp":
            p.set_schedule("cp", 64)
        p.set_engine(engine)
        p.bind(0)
        for rep in range(2):
            send = make_send(g.n, m, seed=rep)
            _, want, _ = replay_bytes(g, s, send, m)
            sd = torch.from_numpy(send).cuda()
            r = torch.zeros_like(sd)
            p.execute(sd, r)
            p.sync()
            assert np.array_equal(r.cpu().numpy(), want), rep
