"""Pin the CPU oracle (oracle/replay_bytes.py) to the reference.

The golden vectors in tests/golden/golden.json were produced by the read-only
reference replay (pkg/src/a2aflow/evaluate.py:56-127) via
tests/golden/make_golden.py.  The byte-moving restatement must give the same
T, the same acceptance and the same error text, and its receive buffers must
be the transpose of the send buffers.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import apply_edit
from replay_bytes import OracleEvalError, make_send, replay_bytes, transpose_expected

SMALL = ["torus2x4", "hypercube3", "gk8_2", "torus2x4_h1", "torus2x4_h2", "gk8_2_h1",
         "ts_ring3", "ts_torus2x4", "ts_hypercube3", "ts_gk8_2", "ts_torus3x3"]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_T_matches_reference(name, golden, artifacts):
    a = artifacts(name)
    rec = golden["configs"][name]
    send = make_send(a.g.n, 8)
    for (m, b, sync), want in zip(golden["params"], rec["replay"]):
        T, _, _ = replay_bytes(a.g, a.sched, send, 8, b=b, sync_latency=sync, m_model=m)
        assert want["ok"] is True and repr(T) == want["T"]


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("m", [1, 7, 1000, 4096])
def test_oracle_moves_bytes_to_transpose(name, m, artifacts, golden):
    a = artifacts(name)
    send = make_send(a.g.n, m, seed=3)
    T, recv, lbytes = replay_bytes(a.g, a.sched, send, m)
    assert np.array_equal(recv, transpose_expected(send))
    # per-(step, link) bytes: the integer rule summed over ops; when Q | m they
    # equal the reference's chunk counts x m/Q exactly
    chunks = golden["configs"][name]["link_chunks"]
    assert {f"{t},{e}" for (t, e) in lbytes} <= set(chunks)
    if m % a.sched.Q == 0:
        for k, c in chunks.items():
            t, e = map(int, k.split(","))
            assert lbytes.get((t, e), 0) == c * (m // a.sched.Q)


@pytest.mark.parametrize("name", ["torus2x4", "gk8_2", "ts_ring3", "ts_hypercube3",
                                  "torus2x4_h2"])
def test_oracle_errors_match_reference(name, golden, artifacts):
    a = artifacts(name)
    for case in golden["configs"][name]["corruptions"]:
        s = apply_edit(a.sched, case["edit"])
        want = case["replay"]
        if "error" in want:
            with pytest.raises(OracleEvalError) as ei:
                replay_bytes(a.g, s, make_send(a.g.n, 16), 16)
            assert str(ei.value) == want["error"], case["label"]
        else:
            send = make_send(a.g.n, 16)
            T, recv, _ = replay_bytes(a.g, s, send, 16)
            assert np.array_equal(recv, transpose_expected(send)), case["label"]


def test_oracle_mode_and_size_checks(artifacts):
    a = artifacts("torus2x4")
    with pytest.raises(OracleEvalError, match="ts-mode"):
        replay_bytes(a.g, a.path_sched, make_send(8, 4), 4)
    import copy
    s = copy.deepcopy(a.sched)
    s.n = 9
    with pytest.raises(OracleEvalError, match="graph has 8 nodes, schedule says 9"):
        replay_bytes(a.g, s, make_send(8, 4), 4)


def test_make_send_unique_bytes():
    x = make_send(4, 64, seed=0)
    assert x.shape == (4, 4, 64)
    rows = {x[s, d].tobytes() for s in range(4) for d in range(4)}
    assert len(rows) == 16
    assert not np.array_equal(make_send(4, 64, seed=1), x)


@pytest.mark.parametrize("name", SMALL)
@pytest.mark.parametrize("m", [1, 13, 4096])
def test_c_oracle_equals_python_oracle(name, m, artifacts, golden):
    """The multi-threaded C port (the CPU-baseline arm) agrees with the pinned
    Python restatement: recv, per-link bytes, T and error texts."""
    from c_oracle import OracleEvalError as CErr
    from c_oracle import replay_bytes_c
    a = artifacts(name)
    send = make_send(a.g.n, m, seed=5)
    T, recv, lb = replay_bytes(a.g, a.sched, send, m)
    Tc, recvc, lbc = replay_bytes_c(a.g, a.sched, send, m, nthreads=4)
    assert repr(T) == repr(Tc)
    assert np.array_equal(recv, recvc)
    want = np.zeros_like(lbc)
    for (t, e), x in lb.items():
        want[t, e] = x
    assert np.array_equal(lbc, want)
    # reused scratch workspace (the bench's CPU-baseline form), twice into one recv
    from c_oracle import workspace
    ws = workspace(a.sched, a.g.n, m)
    out = np.zeros_like(send)
    for k in range(2):
        Tw, _, lbw = replay_bytes_c(a.g, a.sched, make_send(a.g.n, m, seed=6 + k), m,
                                    nthreads=3, recv=out, ws=ws)
        assert repr(Tw) == repr(T) and np.array_equal(lbw, want)
        assert np.array_equal(out, np.swapaxes(make_send(a.g.n, m, seed=6 + k), 0, 1))
    for case in golden["configs"][name].get("corruptions", []):
        s = apply_edit(a.sched, case["edit"])
        if "error" in case["replay"]:
            with pytest.raises(CErr) as ei:
                replay_bytes_c(a.g, s, send, m, nthreads=2)
            assert str(ei.value) == case["replay"]["error"]


def test_c_oracle_workspace_too_small(artifacts):
    from c_oracle import replay_bytes_c, workspace
    a = artifacts("gk8_2")
    m = 64
    ws = workspace(a.sched, a.g.n, m)
    with pytest.raises(RuntimeError, match="workspace too small"):
        replay_bytes_c(a.g, a.sched, make_send(a.g.n, m), m, ws=ws[:len(ws) - m])


@pytest.mark.parametrize("m", [(1 << 20) + 3, (3 << 20) + 1])
def test_c_oracle_multi_piece_ops(m, artifacts):
    """Ops longer than the 1 MiB copy piece are cut and reassembled exactly."""
    from c_oracle import replay_bytes_c, workspace
    a = artifacts("hypercube3")
    send = make_send(a.g.n, m, seed=9)
    _, recv, _ = replay_bytes_c(a.g, a.sched, send, m, nthreads=5, ws=workspace(a.sched, a.g.n, m))
    assert np.array_equal(recv, np.swapaxes(send, 0, 1))
