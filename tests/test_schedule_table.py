"""Binary op table (csrc/a2a_io.cpp) and the `pack`
CLI command.

The format is pinned independently of the C++ writer: ``_py_table`` builds the
bytes with ``struct`` + ``hashlib`` and the native writer must produce exactly
those bytes, the native reader must read them back.  Ops round-trip bit-exact
against the XML loader for every frozen artifact, and the reader applies the
XML loader's own rejects (reference src/schedule.py:370-378) with the same
texts.  ``sha256_file`` is checked against hashlib on the FIPS 180-4 padding
boundaries."""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import struct

import numpy as np
import pytest

from paper_2309_13541_b200.artifacts import ARTIFACT_DIR, list_artifacts, load_artifact
from paper_2309_13541_b200.cli import main
from paper_2309_13541_b200.native_io import (OpTableSchedule, is_schedule_table, load_schedule,
                                             load_schedule_table, load_schedule_xml,
                                             save_schedule_table, sha256_file)
from paper_2309_13541_b200.schedule import ScheduleError


def _py_table(n, nsteps, q, mode, chunk_bytes, ops) -> bytes:
    ops = np.ascontiguousarray(ops, dtype="<i4").reshape(-1, 7)
    body = (b"A2ATBL1\n" + struct.pack("<I5i", 48, n, nsteps, q, mode, 0)
            + struct.pack("<dq", chunk_bytes, ops.shape[0]) + ops.tobytes())
    return body + hashlib.sha256(body).digest()


def _row(i):
    return (i.t, i.src, i.dst, i.s, i.d, i.c0, i.c1)


def _small():
    ops = np.array([[0, 0, 1, 0, 1, 0, 2], [0, 1, 2, 1, 2, 0, 1], [1, 1, 2, 0, 2, 1, 2]], dtype=np.int32)
    return OpTableSchedule(3, 2, 0.5, 2, "ts", ops)


def test_header_layout_is_48_bytes():
    assert len(_py_table(3, 2, 2, 0, 0.5, np.zeros((0, 7)))) == 48 + 32


@pytest.mark.parametrize("size", [0, 1, 3, 55, 56, 57, 63, 64, 65, 119, 120, 128, 65536, (1 << 20) + 3])
def test_sha256_file_matches_hashlib(size, tmp_path):
    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8).tobytes()
    p = tmp_path / "x.bin"
    p.write_bytes(data)
    assert sha256_file(p) == hashlib.sha256(data).hexdigest()


def test_sha256_known_answers(tmp_path):
    p = tmp_path / "abc"
    p.write_bytes(b"abc")
    assert sha256_file(p) == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    p.write_bytes(b"")
    assert sha256_file(p) == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    with pytest.raises(ValueError, match="cannot open"):
        sha256_file(tmp_path / "missing")


def test_writer_bytes_equal_python_format(tmp_path):
    s = _small()
    p = tmp_path / "s.a2at"
    save_schedule_table(s, p)
    assert p.read_bytes() == _py_table(3, 2, 2, 0, 0.5, s.ops_array)
    assert not os.path.exists(str(p) + ".tmp")


def test_reader_reads_python_built_table(tmp_path):
    s = _small()
    p = tmp_path / "s.a2at"
    p.write_bytes(_py_table(3, 2, 2, 1, 0.5, s.ops_array))
    t = load_schedule_table(p)
    assert (t.n, t.nsteps, t.Q, t.mode, t.chunk_bytes) == (3, 2, 2, "path", 0.5)
    assert np.array_equal(t.ops_array, s.ops_array)
    assert [_row(i) for i in t.instructions] == [tuple(r) for r in s.ops_array.tolist()]


def test_empty_schedule_round_trip(tmp_path):
    s = OpTableSchedule(1, 0, 1.0, 1, "ts", np.zeros((0, 7), dtype=np.int32))
    p = tmp_path / "e.a2at"
    save_schedule_table(s, p)
    t = load_schedule_table(p)
    assert t.ops_array.shape == (0, 7) and (t.n, t.nsteps, t.Q) == (1, 0, 1)


def _xml_of(name):
    d = os.path.join(ARTIFACT_DIR, name)
    for x in ("ts.xml", "ts.xml.gz", "path.xml", "path.xml.gz"):
        if os.path.exists(os.path.join(d, x)):
            return os.path.join(d, x)
    raise FileNotFoundError(name)


@pytest.mark.parametrize("name", list_artifacts())
def test_round_trip_every_artifact(name, tmp_path):
    """The XML as parsed, and the lowered hop-step schedule the executor runs."""
    x = load_schedule_xml(_xml_of(name))
    p = tmp_path / "x.a2at"
    save_schedule_table(x, p)
    t = load_schedule(p)
    assert (t.n, t.nsteps, t.Q, t.mode, t.chunk_bytes) == (x.n, x.nsteps, x.Q, x.mode, x.chunk_bytes)
    assert np.array_equal(t.ops_array, x.ops_array)
    a = load_artifact(name, native=True)
    save_schedule_table(a.sched, p)
    t = load_schedule_table(p)
    assert t.mode == "ts" and np.array_equal(t.ops_array, a.sched.ops_array)


def test_reference_objects_accepted(tmp_path):
    """Instruction lists (no ops_array) are packed like op arrays."""
    a = load_artifact("gk8_2")                  # python loader: Instruction objects
    assert getattr(a.sched, "ops_array", None) is None
    p = tmp_path / "g.a2at"
    save_schedule_table(a.sched, p)
    t = load_schedule_table(p)
    assert [_row(i) for i in t.instructions] == [_row(i) for i in a.sched.instructions]


def test_gzip_table(tmp_path):
    s = _small()
    p = tmp_path / "s.a2at.gz"
    with gzip.open(p, "wb") as fh:
        fh.write(_py_table(3, 2, 2, 0, 0.5, s.ops_array))
    assert is_schedule_table(p)
    assert np.array_equal(load_schedule(p).ops_array, s.ops_array)


@pytest.mark.parametrize("corrupt,msg", [
    (lambda b: b[:-1], "truncated"),
    (lambda b: b + b"\0", "truncated"),
    (lambda b: b[:60], "truncated"),
    (lambda b: b"X" + b[1:], "not an A2ATBL1 file"),
    (lambda b: b[:50] + bytes([b[50] ^ 1]) + b[51:], "sha256 mismatch"),
    (lambda b: b[:-1] + bytes([b[-1] ^ 0x80]), "sha256 mismatch"),
])
def test_corruption_rejected(corrupt, msg, tmp_path):
    p = tmp_path / "c.a2at"
    p.write_bytes(corrupt(_py_table(3, 2, 2, 0, 0.5, _small().ops_array)))
    with pytest.raises(ValueError, match=msg):
        load_schedule_table(p)


def test_header_rejects(tmp_path):
    ops = _small().ops_array
    p = tmp_path / "h.a2at"
    p.write_bytes(_py_table(3, 2, 2, 7, 0.5, ops))
    with pytest.raises(ValueError, match="unknown mode"):
        load_schedule_table(p)
    b = bytearray(_py_table(3, 2, 2, 0, 0.5, ops)[:-32])
    b[8:12] = struct.pack("<I", 64)
    p.write_bytes(bytes(b) + hashlib.sha256(bytes(b)).digest())
    with pytest.raises(ValueError, match="unsupported header size"):
        load_schedule_table(p)


def _xml_reject_text(tmp_path, body):
    x = tmp_path / "r.xml"
    x.write_text('<schedule n="3" nsteps="2" chunkbytes="0.5" q="2" mode="ts">' + body + "</schedule>")
    with pytest.raises(ScheduleError) as e:
        load_schedule_xml(x)
    return str(e.value)


@pytest.mark.parametrize("row,xml", [
    ([2, 0, 1, 0, 1, 0, 1], '<step t="2"><send src="0" dst="1" s="0" d="1" c0="0" c1="1"/></step>'),
    ([-1, 0, 1, 0, 1, 0, 1], '<step t="-1"><send src="0" dst="1" s="0" d="1" c0="0" c1="1"/></step>'),
    ([0, 0, 1, 0, 1, 1, 1], '<step t="0"><send src="0" dst="1" s="0" d="1" c0="1" c1="1"/></step>'),
    ([0, 0, 1, 0, 1, 0, 3], '<step t="0"><send src="0" dst="1" s="0" d="1" c0="0" c1="3"/></step>'),
])
def test_op_rejects_match_xml_loader(row, xml, tmp_path):
    want = _xml_reject_text(tmp_path, xml)
    p = tmp_path / "r.a2at"
    p.write_bytes(_py_table(3, 2, 2, 0, 0.5, np.array([row])))
    with pytest.raises(ScheduleError) as e:
        load_schedule_table(p)
    assert str(e.value) == want
    with pytest.raises(ScheduleError) as e:       # the writer refuses it too
        save_schedule_table(OpTableSchedule(3, 2, 0.5, 2, "ts", np.array([row], dtype=np.int32)),
                            tmp_path / "w.a2at")
    assert str(e.value) == want
    assert not os.path.exists(tmp_path / "w.a2at")


def test_load_schedule_table_missing(tmp_path):
    with pytest.raises(ValueError, match="cannot open"):
        load_schedule_table(tmp_path / "nope.a2at")


# ---- CLI: pack, and eval on a packed table ----

def test_pack_ts_then_eval(tmp_path, capsys):
    d = os.path.join(ARTIFACT_DIR, "ts_torus2x4")
    graph, xml = os.path.join(d, "graph.json"), _xml_of("ts_torus2x4")
    out = str(tmp_path / "t.a2at")
    assert main(["pack", "--graph", graph, "--sched", xml, "-o", out]) == 0
    capsys.readouterr()
    man = json.load(open(out + ".manifest.json"))
    assert set(man) == {"command", "argv", "seed", "version", "inputs", "outputs", "wall_clock_s"}
    assert man["command"] == "pack"
    assert man["outputs"] == {out: hashlib.sha256(open(out, "rb").read()).hexdigest()}
    assert man["inputs"][xml] == hashlib.sha256(open(xml, "rb").read()).hexdigest()
    lines = []
    for sched in (xml, out):
        assert main(["eval", "--graph", graph, "--sched", sched, "--m", "3", "--sync", "0.5"]) == 0
        lines.append(capsys.readouterr().out.strip())
    assert lines[0] == lines[1] and lines[0].endswith("delivered = True")


def test_pack_path_with_routes(tmp_path, capsys):
    d = os.path.join(ARTIFACT_DIR, "gk8_2")
    out = str(tmp_path / "g.a2at")
    assert main(["pack", "--graph", os.path.join(d, "graph.json"), "--sched", _xml_of("gk8_2"),
                 "--routes", os.path.join(d, "path.xml.routes.json"), "-o", out]) == 0
    assert "mode ts" in capsys.readouterr().out
    t = load_schedule_table(out)
    assert np.array_equal(t.ops_array, load_artifact("gk8_2", native=True).sched.ops_array)


def test_pack_rejects_bad_schedule(tmp_path, capsys):
    d = os.path.join(ARTIFACT_DIR, "ts_ring3")
    text = open(os.path.join(d, "ts.xml")).read()
    bad = tmp_path / "bad.xml"
    bad.write_text(text.replace('src="0"', 'src="1"', 1))
    out = tmp_path / "b.a2at"
    assert main(["pack", "--graph", os.path.join(d, "graph.json"), "--sched", str(bad), "-o", str(out)]) == 1
    assert capsys.readouterr().err.startswith("error: ")
    assert not out.exists()


@pytest.mark.parametrize("seed", range(0, 200, 5))
def test_random_schedules_round_trip(seed, tmp_path):
    """Random valid schedules (tests/fuzz_schedules.py): the table reloads the
    same ops, and the plan built from it has the oracle's modelled T."""
    from fuzz_schedules import random_case
    from replay_bytes import make_send, replay_bytes

    from paper_2309_13541_b200.executor import Plan
    g, sched, m, _, _ = random_case(seed)
    p = tmp_path / "f.a2at"
    save_schedule_table(sched, p)
    t = load_schedule_table(p)
    assert [_row(i) for i in t.instructions] == [_row(i) for i in sched.instructions]
    T, _, _ = replay_bytes(g, sched, make_send(g.n, m, seed=seed), m)
    with Plan(g, t, m=m) as plan:
        assert plan.model_time(m) == T
