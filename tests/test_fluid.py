"""fluid.py against the reference's own numbers: per-link
normalised loads and the max load of every path config's widest-path set,
bit-identical (repr) to eval_link_load run by the reference in
tests/golden/make_golden.py; the EvalError / RouteError texts of
evaluate.py:134-136 and paths.py:49-57."""
from __future__ import annotations

import os

import pytest

from paper_2309_13541_b200.artifacts import ARTIFACT_DIR
from paper_2309_13541_b200.errors import EvalError, RouteError
from paper_2309_13541_b200.fluid import (WeightedPathSet, eval_link_load, eval_path_alltoall,
                                         load_routes)
from paper_2309_13541_b200.graphs import load_graph

PATH_CONFIGS = ["torus2x4", "hypercube3", "gk8_2", "torus4x4x4", "gk64_4", "gk256_4",
                "torus2x4_h1", "torus2x4_h2", "gk8_2_h1", "gk64_4_h2"]


def _f(d, base):
    for x in (base, base + ".gz"):
        if os.path.exists(os.path.join(d, x)):
            return os.path.join(d, x)
    return None


@pytest.mark.parametrize("name", PATH_CONFIGS)
def test_link_loads_bit_identical_to_reference(name, golden):
    rec = golden["configs"].get(name)
    if rec is None or "fluid_max_load" not in rec:
        pytest.skip("no golden fluid loads")
    d = os.path.join(ARTIFACT_DIR, name)
    aug = _f(d, "aug_graph.json")
    g = load_graph(aug or _f(d, "graph.json"))
    mx, loads = eval_link_load(g, load_routes(_f(d, "wps.json")))
    assert repr(mx) == rec["fluid_max_load"]
    if aug is None:
        assert [repr(float(x)) for x in loads] == rec["fluid_link_load"]
    else:   # golden keeps the physical links: nic_out_u -> nic_in_v of the augmented graph
        phys = load_graph(_f(d, "graph.json"))
        got = [repr(float(loads[g.edge_index[(3 * u + 2, 3 * v + 1)]])) for u, v, _ in phys.edges]
        assert got == rec["fluid_link_load"]


def test_eval_path_alltoall_errors(artifacts):
    g = artifacts("torus2x4").g
    with pytest.raises(EvalError, match=r"commodity \(0,1\) has zero total weight"):
        eval_path_alltoall(g, WeightedPathSet(paths={(0, 1): [((0, 1), 0.0)]}))
    with pytest.raises(RouteError, match="does not join"):
        eval_path_alltoall(g, WeightedPathSet(paths={(0, 1): [((0, 2), 1.0)]}))
    with pytest.raises(RouteError, match="nonexistent edge"):
        eval_link_load(g, WeightedPathSet(paths={(0, 5): [((0, 5), 1.0)]}))
    with pytest.raises(RouteError, match="not simple"):
        eval_link_load(g, WeightedPathSet(paths={(0, 1): [((0, 1, 0, 1), 1.0)]}))


def test_fluid_time_scales(artifacts):
    a = artifacts("hypercube3")
    wps = load_routes(_f(os.path.join(ARTIFACT_DIR, "hypercube3"), "wps.json"))
    t1 = eval_path_alltoall(a.g, wps)
    assert eval_path_alltoall(a.g, wps, m=2.0, b=4.0) == t1 * 2.0 / 4.0
