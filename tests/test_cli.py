"""`eval` command (paper_2309_13541_b200/cli.py) against the reference CLI's
output for the same files: ``T = <T:.9g>, delivered = True`` with T from the
reference replay (tests/golden/golden.json, made by the reference itself),
``error: ...`` + exit 1 on rejects, exit 2 on usage errors
(reference pkg/src/a2aflow/cli.py:326-343, :419-431)."""
from __future__ import annotations

import json
import os

import pytest

from paper_2309_13541_b200.artifacts import ARTIFACT_DIR
from paper_2309_13541_b200.cli import main

HERE = os.path.dirname(os.path.abspath(__file__))


def _golden():
    with open(os.path.join(HERE, "golden", "golden.json")) as fh:
        return json.load(fh)


def _files(name):
    d = os.path.join(ARTIFACT_DIR, name)
    for x in ("ts.xml", "ts.xml.gz"):
        if os.path.exists(os.path.join(d, x)):
            return ["--graph", os.path.join(d, "graph.json"), "--sched", os.path.join(d, x)]
    z = "" if os.path.exists(os.path.join(d, "path.xml")) else ".gz"
    return ["--graph", os.path.join(d, "graph.json"), "--sched", os.path.join(d, "path.xml" + z),
            "--path-routes", os.path.join(d, "path.xml.routes.json" + z)]


# augmented (host-bottleneck) configs need the node map: covered by test_native_io
NAMES = ["ts_ring3", "ts_torus2x4", "ts_hypercube3", "ts_gk8_2", "ts_torus3x3",
         "torus2x4", "hypercube3", "gk8_2", "torus4x4x4", "gk64_4"]


@pytest.mark.parametrize("name", NAMES)
def test_eval_prints_reference_T(name, capsys):
    gold = _golden()
    params, runs = gold["params"], gold["configs"][name]["replay"]
    for (m, b, sync), run in zip(params, runs):
        rc = main(["eval", *_files(name), "--m", repr(m), "--b", repr(b), "--sync", repr(sync)])
        out = capsys.readouterr().out.strip()
        assert rc == 0
        assert out == f"T = {float(run['T']):.9g}, delivered = True", (m, b, sync)


def test_eval_reject_exit_1(tmp_path, capsys):
    d = os.path.join(ARTIFACT_DIR, "ts_ring3")
    with open(os.path.join(d, "ts.xml")) as fh:
        text = fh.read()
    bad = tmp_path / "bad.xml"
    bad.write_text(text.replace('src="0"', 'src="1"', 1))    # first send now from a non-holder / non-edge
    rc = main(["eval", "--graph", os.path.join(d, "graph.json"), "--sched", str(bad)])
    err = capsys.readouterr().err
    assert rc == 1 and err.startswith("error: ")
    rc = main(["eval", "--graph", os.path.join(d, "graph.json"), "--sched", str(tmp_path / "nope.xml")])
    assert rc == 1 and capsys.readouterr().err.startswith("error: ")
    # a path-mode schedule without its routes: the replay's mode check (evaluate.py:70-71)
    g = os.path.join(ARTIFACT_DIR, "gk8_2")
    rc = main(["eval", "--graph", os.path.join(g, "graph.json"), "--sched", os.path.join(g, "path.xml")])
    assert rc == 1 and "ts-mode" in capsys.readouterr().err


def test_eval_usage_exit_2():
    with pytest.raises(SystemExit) as ex:
        main(["eval"])
    assert ex.value.code == 2


def test_eval_needs_sched_or_routes(capsys):
    """The reference raises GraphError("eval needs --sched or --routes") -> exit 1."""
    g = os.path.join(ARTIFACT_DIR, "gk8_2", "graph.json")
    rc = main(["eval", "--graph", g])
    assert rc == 1 and capsys.readouterr().err.strip() == "error: eval needs --sched or --routes"


@pytest.mark.parametrize("name", ["torus2x4", "hypercube3", "gk8_2", "torus4x4x4", "gk64_4"])
def test_eval_routes_fluid_time(name, capsys):
    """`eval --graph G --routes R`: the reference's cut-through fluid time
    eval_path_alltoall (cli.py:338-342, evaluate.py:130-139), same output line
    as the reference for its own widest-path set (golden fluid_max_load)."""
    gold = _golden()["configs"][name]
    d = os.path.join(ARTIFACT_DIR, name)
    wps = [os.path.join(d, x) for x in ("wps.json", "wps.json.gz") if os.path.exists(os.path.join(d, x))][0]
    for m, b in ((1.0, 1.0), (2.0, 1.0), (1048576.0, 3.0)):
        rc = main(["eval", "--graph", os.path.join(d, "graph.json"), "--routes", wps,
                   "--m", repr(m), "--b", repr(b)])
        out = capsys.readouterr().out.strip()
        assert rc == 0
        assert out == f"T = {float(gold['fluid_max_load']) * m / b:.9g}"


@pytest.mark.gpu
@pytest.mark.parametrize("name,m,sched", [("ts_torus2x4", 4096 + 3, "static"),
                                          ("gk8_2", 1 << 20, "cp:65536"),
                                          ("torus2x4", 7, "static")])
def test_eval_execute(name, m, sched, capsys):
    rc = main(["eval", *_files(name), "--m", str(m), "--execute", "--schedule", sched])
    out = capsys.readouterr()
    assert rc == 0, out.err
    lines = out.out.strip().splitlines()
    assert lines[0].endswith("delivered = True")
    assert lines[1].startswith("executed on cuda:0") and lines[1].endswith("recv == transpose(send): True")
