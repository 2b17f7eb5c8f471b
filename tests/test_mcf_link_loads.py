"""Per-link byte loads of the executed schedule vs the MCF solution (SURVEY §8 finding 1).

The executor moves exactly the lowered schedule's bytes per link (device
counters == a2a_plan_link_bytes, tests/test_gpu_executor.py).  Those equal the
MCF link loads m * sum_c f_ce / F exactly when quantisation is exact (Q = LCM,
2x4 torus / hypercube: every link 4*m).  With the Q = q_max fallback each route
is off by < 1/Q of a shard (src/schedule.py:108-131), so a link carrying k
routes deviates by < k/Q shards.  Both are checked here against the reference's
own eval_link_load numbers frozen in tests/golden/golden.json, and the maximum
relative deviation is written to profiles/r01_mcf_link_deviation.json.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from paper_2309_13541_b200.executor import Plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH_CONFIGS = ["torus2x4", "hypercube3", "gk8_2", "torus2x4_h1", "torus2x4_h2", "gk8_2_h1",
                "torus4x4x4", "gk64_4", "gk64_4_h2", "gk256_4"]


@pytest.mark.parametrize("name", PATH_CONFIGS)
def test_schedule_link_loads_vs_mcf(name, golden, artifacts):
    rec = golden["configs"].get(name)
    if rec is None or "fluid_link_load" not in rec:
        pytest.skip("no golden MCF loads")
    a = artifacts(name)
    Q = a.sched.Q
    with Plan(a.g, a.sched, m=Q, copy_self=False) as p:      # m = Q: one byte per chunk
        chunks = p.link_bytes().sum(axis=0).astype(np.float64)
    fluid = np.array([float(x) for x in rec["fluid_link_load"]])   # shards per link (MCF)
    routes_per_link = np.zeros(len(a.g.edges))
    for r in a.routes:
        for u, v in zip(r["nodes"], r["nodes"][1:]):
            routes_per_link[a.g.edge_index[(u, v)]] += 1
    dev = np.abs(chunks / Q - fluid)
    assert np.all(dev <= routes_per_link / Q + 1e-9)
    if name in ("torus2x4", "hypercube3"):
        assert np.all(dev == 0)                      # exact quantisation: identical loads
    out = os.path.join(ROOT, "profiles", "r01_mcf_link_deviation.json")
    data = json.load(open(out)) if os.path.exists(out) else {}
    nz = fluid > 0
    data[name] = {"Q": Q, "max_abs_dev_shards": float(dev.max()),
                  "max_rel_dev": float((dev[nz] / fluid[nz]).max()) if nz.any() else 0.0,
                  "max_schedule_load_shards": float((chunks / Q).max()),
                  "max_mcf_load_shards": float(fluid.max())}
    with open(out, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
