"""Drop-in side: generators, augmentation, XML dialect and the path->steps lowering.

Generators are checked against the graph files the reference itself wrote
(artifacts/*/graph.json, aug_graph.json via a2aflow.graphs.save_graph); the
XML reader against the reference's own reject tests
(tests/test_schedule.py:136-167); the lowering against the hop histograms of
SURVEY.md Appendix A.
"""
from __future__ import annotations

import os

import pytest

from paper_2309_13541_b200.artifacts import ARTIFACT_DIR, _find, load_artifact
from paper_2309_13541_b200.graphs import (augment_host_bottleneck, distance_sum,
                                          gen_gen_kautz, gen_hypercube, gen_torus, load_graph,
                                          save_graph)
from paper_2309_13541_b200.lowering import (collapse_aug_routes, hop_histogram,
                                            lower_path_to_steps)
from paper_2309_13541_b200.schedule import (ChunkedSchedule, Instruction, ScheduleError,
                                            emit_schedule_xml, parse_schedule_xml)

GENS = {
    "torus2x4": lambda: gen_torus([2, 4]),
    "hypercube3": lambda: gen_hypercube(3),
    "gk8_2": lambda: gen_gen_kautz(8, 2),
    "torus4x4x4": lambda: gen_torus([4, 4, 4]),
    "gk64_4": lambda: gen_gen_kautz(64, 4),
    "gk256_4": lambda: gen_gen_kautz(256, 4),
    "ts_ring3": lambda: gen_torus([3], bidirectional=False),
    "ts_torus3x3": lambda: gen_torus([3, 3]),
}


@pytest.mark.parametrize("name", sorted(GENS))
def test_generators_match_reference_files(name):
    d = os.path.join(ARTIFACT_DIR, name)
    if not os.path.isdir(d):
        pytest.skip("artifact missing")
    ref = load_graph(_find(d, "graph.json"))
    mine = GENS[name]()
    assert mine.n == ref.n and mine.edges == ref.edges
    assert mine.meta.get("self_loops", 0) == ref.meta.get("self_loops", 0)


@pytest.mark.parametrize("name,base,h", [("torus2x4_h2", "torus2x4", 2.0),
                                         ("gk8_2_h1", "gk8_2", 1.0),
                                         ("gk64_4_h2", "gk64_4", 2.0)])
def test_augmentation_matches_reference(name, base, h):
    d = os.path.join(ARTIFACT_DIR, name)
    ref = load_graph(_find(d, "aug_graph.json"))
    aug, mp = augment_host_bottleneck(GENS[base](), h)
    assert aug.n == ref.n and aug.edges == ref.edges
    assert mp.host[3] == 9 and mp.nic_in[3] == 10 and mp.nic_out[3] == 11


def test_graph_kats():
    """reference tests/test_graphs.py:43-118 style facts + SURVEY Σdist KATs."""
    gk = gen_gen_kautz(8, 2)
    assert gk.num_edges == 14 and gk.meta["self_loops"] == 2
    assert sorted(len(a) for a in gk.out_adj)[:2] == [1, 1]
    t = gen_torus([2, 4])
    assert t.num_edges == 24 and all(len(a) == 3 for a in t.out_adj)
    assert distance_sum(t) == 96 and distance_sum(gen_hypercube(3)) == 96
    assert distance_sum(gk) == 118
    assert distance_sum(gen_torus([4, 4, 4])) == 12288
    assert gen_gen_kautz(256, 4).num_edges == 1020


def test_graph_roundtrip(tmp_path):
    g = gen_gen_kautz(27, 4)
    p = tmp_path / "g.json"
    save_graph(g, p)
    assert load_graph(p).edges == g.edges


HOPS = {"torus2x4": [56, 32, 8], "hypercube3": [56, 32, 8], "gk8_2": [58, 44, 23, 3],
        "torus4x4x4": [4347, 3963, 3000, 1716, 730, 187],
        "gk64_4": [4214, 3972, 3099, 823, 94, 5],
        "gk256_4": [66028, 65021, 61155, 47489, 13011, 2749, 381, 55, 1]}


@pytest.mark.parametrize("name", sorted(HOPS))
def test_lowering_hop_histograms(name):
    if not os.path.isdir(os.path.join(ARTIFACT_DIR, name)):
        pytest.skip("artifact missing")
    a = load_artifact(name)
    assert hop_histogram(a.sched) == HOPS[name]
    assert a.sched.mode == "ts" and a.sched.n == a.g.n
    key = [(i.t, i.src, i.dst, i.s, i.d, i.c0) for i in a.sched.instructions]
    assert key == sorted(key)


def test_lowering_single_route_kat():
    """reference tests/test_schedule.py:87-95: one route, Q=1 -> one hop-op per link."""
    routes = [{"s": 0, "d": 2, "nodes": [0, 1, 2]}]
    ps = ChunkedSchedule(n=3, nsteps=1, chunk_bytes=1.0, Q=1, mode="path",
                         instructions=[Instruction(0, 0, 0, 0, 2, 0, 1)])
    ts = lower_path_to_steps(routes, ps)
    assert ts.nsteps == 2 and ts.instructions == [Instruction(0, 0, 1, 0, 2, 0, 1),
                                                  Instruction(1, 1, 2, 0, 2, 0, 1)]
    with pytest.raises(ScheduleError):
        lower_path_to_steps([{"s": 0, "d": 1, "nodes": [0, 2]}], ps)


def test_collapse_aug_route_example():
    """[0,2,4,3] = host0->nic_out0->nic_in1->host1 -> [0,1]."""
    _, mp = augment_host_bottleneck(gen_torus([2, 4]), 2.0)
    out = collapse_aug_routes([{"s": 0, "d": 3, "nodes": [0, 2, 4, 3]}], mp)
    assert out == [{"s": 0, "d": 1, "nodes": [0, 1]}]


def test_augmented_lowering_is_physical():
    a = load_artifact("torus2x4_h2")
    for i in a.sched.instructions:
        assert (i.src, i.dst) in a.g.edge_index and 0 <= i.s < 8 and 0 <= i.d < 8


def test_xml_roundtrip_and_gz(tmp_path):
    a = load_artifact("gk8_2")
    for fn in ("s.xml", "s.xml.gz"):
        p = tmp_path / fn
        emit_schedule_xml(a.sched, p)
        back = parse_schedule_xml(p)
        assert (back.n, back.nsteps, back.Q, back.mode) == (a.sched.n, a.sched.nsteps,
                                                            a.sched.Q, a.sched.mode)
        assert back.instructions == a.sched.instructions


@pytest.mark.parametrize("text,match", [
    ('<schedule n="3" chunkbytes="1.0" q="1" mode="ts"></schedule>', "nsteps"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="1" mode="ts"><step t="5"/></schedule>',
     "outside"),
    ("<schedule", "malformed"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="1" mode="zz"></schedule>', "unknown mode"),
    ('<schedule n="3" nsteps="2" chunkbytes="1.0" q="2" mode="ts"><step t="0">'
     '<send src="0" dst="1" s="0" d="1" c0="1" c1="1"/></step></schedule>', "bad chunk range"),
])
def test_xml_rejects(tmp_path, text, match):
    p = tmp_path / "bad.xml"
    p.write_text(text)
    with pytest.raises(ScheduleError, match=match):
        parse_schedule_xml(p)
