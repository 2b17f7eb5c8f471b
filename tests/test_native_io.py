"""Native loader (csrc/a2a_io.cpp) == the Python loader/lowering,
with the reference parser's rejects and messages."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2309_13541_b200.artifacts import list_artifacts, load_artifact
from paper_2309_13541_b200.native_io import load_schedule_xml
from paper_2309_13541_b200.schedule import ScheduleError, emit_schedule_xml, parse_schedule_xml


@pytest.mark.parametrize("name", list_artifacts())
def test_native_artifact_equals_python(name):
    py = load_artifact(name)
    nat = load_artifact(name, native=True)
    assert (nat.sched.n, nat.sched.nsteps, nat.sched.Q, nat.sched.mode) == \
        (py.sched.n, py.sched.nsteps, py.sched.Q, py.sched.mode)
    want = np.array([(i.t, i.src, i.dst, i.s, i.d, i.c0, i.c1) for i in py.sched.instructions],
                    dtype=np.int32).reshape(-1, 7)
    assert np.array_equal(nat.sched.ops_array, want)


def test_native_xml_roundtrip_gz(tmp_path):
    a = load_artifact("gk8_2")
    for fn in ("s.xml", "s.xml.gz"):
        p = tmp_path / fn
        emit_schedule_xml(a.sched, p)
        s = load_schedule_xml(p)
        assert s.instructions == parse_schedule_xml(p).instructions


@pytest.mark.parametrize("text,match", [
    ('<schedule n="3" chunkbytes="1.0" q="1" mode="ts"></schedule>', "missing attribute 'nsteps' on <schedule>"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="1" mode="ts"><step t="5"/></schedule>',
     r"step t=5 outside \[0, 2\)"),
    ("<schedule", "malformed XML"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="1" mode="zz"></schedule>', "unknown mode 'zz'"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="2" mode="ts"><step t="0">'
     '<send src="0" dst="1" s="0" d="1" c0="1" c1="1"/></step></schedule>', r"bad chunk range \[1,1\)"),
    ('<plan n="3"/>', "root element is <plan>, not <schedule>"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="2" mode="ts"><stp t="0"/></schedule>',
     "unexpected element <stp>"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="2" mode="ts"><step t="0">'
     '<send src="0" dst="1" s="0" d="1" c0="0"/></step></schedule>', "missing attribute 'c1' on <send>"),
])
def test_native_rejects_like_reference(tmp_path, text, match):
    p = tmp_path / "bad.xml"
    p.write_text(text)
    with pytest.raises(ScheduleError, match=match):
        load_schedule_xml(p)
    with pytest.raises(ScheduleError, match=match):
        parse_schedule_xml(p)


def test_native_faster_on_gk256():
    import time
    if "gk256_4" not in list_artifacts():
        pytest.skip("artifact missing")
    t0 = time.perf_counter()
    a = load_artifact("gk256_4", native=True, verify=False)
    t_nat = time.perf_counter() - t0
    assert a.sched.ops_array.shape == (255890, 7)
    assert t_nat < 5.0
