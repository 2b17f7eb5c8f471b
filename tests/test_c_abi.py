"""include/a2a_exec.h from plain C99: tests/c/abi_from_c.c compiled with
gcc -std=c99 -Wall -Wextra -Werror against the executor library and run (no
GPU calls); its printed values must equal the Python binding's on the same
schedule."""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess

import pytest

from paper_2309_13541_b200 import _native
from paper_2309_13541_b200.executor import EvalError, replay_timestep_schedule
from paper_2309_13541_b200.graphs import Digraph
from paper_2309_13541_b200.schedule import ChunkedSchedule, Instruction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _py_case(first_src=0, first_dst=1):
    g = Digraph.from_edges(3, [(u, v, 1.0) for u in range(3) for v in range(3) if u != v])
    ins = [Instruction(0, s, d, s, d, 0, 2) for s in range(3) for d in range(3) if s != d]
    ins[0] = Instruction(0, first_src, first_dst, 0, 1, 0, 2)
    return g, ChunkedSchedule(n=3, nsteps=1, chunk_bytes=500.0, Q=2, mode="ts", instructions=ins)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="needs gcc")
def test_c_program_against_python_binding(tmp_path):
    libdir = os.path.dirname(_native.LIB_PATH)
    exe = tmp_path / "abi_from_c"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", "-pedantic",
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "abi_from_c.c"),
                    "-o", str(exe), "-L", libdir, "-l:" + os.path.basename(_native.LIB_PATH),
                    "-Wl,-rpath," + libdir], check=True)
    table = tmp_path / "t.a2at"
    out = subprocess.run([str(exe), str(table)], capture_output=True, text=True, check=True).stdout
    got = dict(line.split("=", 1) for line in out.strip().splitlines())
    g, sched = _py_case()
    T, ok = replay_timestep_schedule(g, sched, m=3.0, b=0.5, sync_latency=0.25)
    assert ok and float(got["T"]) == T
    assert int(got["link_bytes"]) == 6 * 1000          # every shard, one hop, m = 1000 B
    g, bad = _py_case(0, 0)
    with pytest.raises(EvalError) as e:
        replay_timestep_schedule(g, bad)
    rc, msg = got["reject"].split(":", 1)
    assert int(rc) == 2 and msg == str(e.value)
    assert got["table"] == "ok"
    assert got["sha256"] == hashlib.sha256(table.read_bytes()).hexdigest()
    assert got["version"] == _native.lib.a2a_version().decode()
