"""Fluid performance model (a2a_plan_simulate, Plan.simulate): runs every
modelled execution order at 1/2/4/8 GPUs, never beats the resource bounds it
models, rejects what it does not model, and is calibrated against measured
runs by tools/sim_calibrate.py (not re-checked here: no GPU numbers on CPU)."""
from __future__ import annotations

import os
import sys

import pytest

from paper_2309_13541_b200.executor import Plan

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("name,m", [("gk8_2", 16 << 20), ("hypercube3", 1 << 20), ("torus2x4_h2", 65536)])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("sched", ["static", "dynamic:1048576", "list:262144", "cp:1048576",
                                   "mix:1048576", "spread:1048576", "cp:1048576:24",
                                   "ready:1048576", "ready:262144"])
def test_simulate_respects_bounds(name, m, G, sched, artifacts):
    import bench
    a = artifacts(name)
    if a.g.n % G:
        pytest.skip("placement needs G | N")
    prm = dict(Plan.SIM_DEFAULTS, jitter=0.0, launch_us=0.0, flag_us=0.0, unit_us=0.0, unit_us_sys=0.0)
    with bench.make_plan(a, m, G, "optimized", sched) as p:
        t = p.simulate(37, **prm)
        bt = bench.bound_terms([p.gpu_info(g) for g in range(G)], a.g.n, m, 1, prm["hbm_gbs"])
    assert 0 < t < 1.0
    # neither the HBM bytes nor the NVLink bytes of the busiest GPU can move faster
    assert t >= bt["t_hbm"] * (1 - 1e-9)
    assert t >= bt["nvlink_bytes"] / (prm["nvlink_gbs"] * 1e9) * (1 - 1e-9)


def test_simulate_single_copy_exact(artifacts):
    """One GPU, one CTA, no fixed costs: the model is bytes / CTA rate."""
    a = artifacts("torus2x4")
    m = 1 << 20
    with Plan(a.g, a.sched, m=m) as p:
        hop = p.gpu_info(0)["hop_bytes"] + 8 * m        # every hop + self shards
        t = p.simulate(1, jitter=0.0, launch_us=0.0, flag_us=0.0, unit_us=0.0, cta_gbs=10.0)
    assert t == pytest.approx(hop / 10e9, rel=1e-9)


def test_simulate_rejects(artifacts):
    a = artifacts("gk8_2")
    with Plan(a.g, a.sched, m=4096, n_gpus=2, protocol="ll") as p:
        with pytest.raises(ValueError, match="LL"):
            p.simulate(8)
    with Plan(a.g, a.sched, m=4096, n_gpus=2) as p:
        with pytest.raises(ValueError):
            p.simulate(8, nvlink_gbs=0.0)


@pytest.mark.parametrize("sched", ["static", "cp:1048576", "mix:1048576"])
def test_simulate_incast_penalty_only_slows(sched, artifacts):
    """The optional ingress-oversubscription penalty never speeds an execute
    up, and is a no-op on one GPU (no NVLink ingress)."""
    import bench
    a = artifacts("gk8_2")
    for G in (1, 4):
        with bench.make_plan(a, 16 << 20, G, "optimized", sched) as p:
            t0, t1 = p.simulate(148), p.simulate(148, incast=0.5)
            assert t1 >= t0 * (1 - 1e-9)
            if G == 1:
                assert t1 == t0


@pytest.mark.parametrize("name", ["gk8_2", "torus2x4_h2", "hypercube3"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("nc", [1, 2, 148])
def test_simulate_ready_queue_completes(name, G, nc, artifacts):
    """Ready queue (mode 5) in the model: the k-th CTA to claim a position
    runs the k-th unit enqueued on its GPU; every unit runs, even with one CTA,
    and the time grows as CTAs are taken away."""
    import bench
    a = artifacts(name)
    if a.g.n % G:
        pytest.skip("placement needs G | N")
    with bench.make_plan(a, 1 << 20, G, "optimized", "ready:262144") as p:
        t = p.simulate(nc)
        assert t > 0
        if nc == 1:
            assert t >= p.simulate(148)
