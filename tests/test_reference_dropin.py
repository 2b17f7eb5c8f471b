"""The drop-in, proven with the reference's own code (skipped where
/root/reference is absent, e.g. on the GPU box).

1. The reference's executor tests (pkg/tests/test_evaluate.py, class
   TestReplay, :22-59) run UNCHANGED with ``a2aflow.evaluate.
   replay_timestep_schedule`` replaced by the ctypes stub of INTEGRATION.md §2
   (extracted from the document, bound to this repo's _a2a_exec.so).
2. The reference's own ``Digraph`` / ``ChunkedSchedule`` objects (built by its
   generators, MCF and compilers) go straight into ``executor.Plan``: same T
   as the reference replay, the device protocol (CPU emulation) delivers the
   transpose, per-link bytes equal the reference schedule's chunk counts.
3. With ``a2aflow`` importable, ``executor.EvalError`` IS-A
   ``a2aflow.evaluate.EvalError``: a caller catching the reference class
   catches the executor's rejects.
"""
from __future__ import annotations

import os
import re
import subprocess
import sys
import textwrap

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "src", "a2aflow")),
                                reason="reference tree not present")


def _env():
    return dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(REF, "src"), ROOT]),
                PYTHONDONTWRITEBYTECODE="1")


def test_reference_replay_tests_pass_through_the_stub(tmp_path):
    from paper_2309_13541_b200 import _native
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    stub = re.search(r"```python\n(# a2aflow/evaluate\.py.*?)```", text, re.S).group(1)
    stub = stub.replace('"paper_2309_13541_b200/_a2a_exec.so"', repr(_native.LIB_PATH))
    calls = tmp_path / "calls.txt"
    plugin = tmp_path / "dropin_plugin.py"
    plugin.write_text(textwrap.dedent(f'''
        import ctypes as C
        import a2aflow.evaluate as ev

        ns = {{"EvalError": ev.EvalError}}
        exec(compile({stub!r}, "INTEGRATION.md", "exec"), ns)
        ns["_lib"].a2a_last_error.restype = C.c_char_p
        _stub = ns["replay_timestep_schedule"]
        n_calls = [0]

        def replay_timestep_schedule(*a, **k):
            n_calls[0] += 1
            return _stub(*a, **k)

        ev.replay_timestep_schedule = replay_timestep_schedule   # before the tests import it

        def pytest_unconfigure(config):
            with open({str(calls)!r}, "w") as fh:
                fh.write(str(n_calls[0]))
    '''))
    out = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "dropin_plugin",
         "--rootdir", str(tmp_path), "-c", os.devnull,
         os.path.join(REF, "tests", "test_evaluate.py") + "::TestReplay"],
        capture_output=True, text=True, timeout=600, cwd=str(tmp_path),
        env=dict(_env(), PYTHONPATH=os.pathsep.join([str(tmp_path), _env()["PYTHONPATH"]])))
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "5 passed" in out.stdout, out.stdout[-2000:]
    assert int(calls.read_text()) >= 7        # every replay went through the stub


def test_reference_objects_into_plan():
    code = textwrap.dedent('''
        import sys
        import numpy as np
        sys.path.insert(0, "oracle")
        from a2aflow.evaluate import EvalError as RefEvalError, replay_timestep_schedule as ref_replay
        from a2aflow.graphs import gen_torus, gen_hypercube
        from a2aflow.mcf import mcf_timestepped
        from a2aflow.schedule import Instruction, compile_timestep_schedule
        from paper_2309_13541_b200.executor import EvalError, Plan, replay_timestep_schedule
        from paper_2309_13541_b200.dist import local_nodes
        from replay_bytes import make_send

        assert issubclass(EvalError, RefEvalError)
        for g in (gen_torus([3], bidirectional=False), gen_hypercube(3)):
            sched = compile_timestep_schedule(g, mcf_timestepped(g, l_max=3 if g.n == 8 else 2))
            for m, b, s in ((1.0, 1.0, 0.0), (4096.0, 2.0, 0.5)):
                assert replay_timestep_schedule(g, sched, m, b, s) == ref_replay(g, sched, m, b, s)
            m = 1000 + 3
            send = make_send(g.n, m, seed=1)
            for G in (1, 2):
                with Plan(g, sched, m=m, n_gpus=G) as p:
                    nodes = [local_nodes(p, r) for r in range(G)]
                    recvs = p.emulate([send[ns] for ns in nodes], num_ctas=5, seed=G)
                    lb = p.link_bytes()
                want = np.swapaxes(send, 0, 1)
                for r in range(G):
                    assert np.array_equal(recvs[r], want[nodes[r]])
                chunks = np.zeros_like(lb)
                for i in sched.instructions:
                    e = g.edge_index[(i.src, i.dst)]
                    chunks[i.t, e] += (i.c1 * m) // sched.Q - (i.c0 * m) // sched.Q
                assert np.array_equal(lb, chunks)
            bad = type(sched)(n=sched.n, nsteps=sched.nsteps, chunk_bytes=sched.chunk_bytes,
                              Q=sched.Q, mode="ts",
                              instructions=list(sched.instructions) + [Instruction(0, 0, 0, 0, 1, 0, 1)])
            try:
                Plan(g, bad, m=64)
            except RefEvalError as ex:
                msg = str(ex)
            else:
                raise AssertionError("no EvalError")
            try:
                ref_replay(g, bad)
            except RefEvalError as ex:
                assert str(ex) == msg, (str(ex), msg)
        print("DROPIN-OK")
    ''')
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=_env())
    assert out.returncode == 0 and "DROPIN-OK" in out.stdout, out.stdout[-2000:] + out.stderr[-3000:]
