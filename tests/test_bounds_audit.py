"""Host bounds audit of every device copy range (compute-sanitizer is closed on
this GPU pool; this is its address-math half): all artifacts, 1/2/4/8 GPUs,
static and dynamic schedules, chains, scratch reuse on/off, the LL protocols,
odd shard sizes."""
from __future__ import annotations

import pytest

from paper_2309_13541_b200.artifacts import list_artifacts
from paper_2309_13541_b200.executor import Plan

NAMES = [n for n in list_artifacts() if not n.startswith("gk256")]


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("sched", ["static", "cp", "mix", "spread", "chain", "chaind"])
@pytest.mark.parametrize("reuse", [False, True])
def test_every_copy_range_in_bounds(name, G, sched, reuse, artifacts):
    a = artifacts(name)
    if G > a.g.n:
        pytest.skip("more GPUs than nodes")
    for m in (1, 1000 + 7, 65536):
        with Plan(a.g, a.sched, m=m, n_gpus=G, reuse_scratch=reuse, placement="optimized") as p:
            p.set_schedule(sched, 0 if sched == "static" else 4096)
            assert p.check_bounds(37)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("proto", ["ll", "ll128"])
def test_ll_ranges_in_bounds(name, G, proto, artifacts):
    """A2A_PROTO_LL pieces: LL sources/destinations inside the landing regions
    (payload addresses, whole destination lines), plain stores GPU-local."""
    a = artifacts(name)
    if G > a.g.n:
        pytest.skip("more GPUs than nodes")
    for m in (1, 1000 + 7, 65536):
        with Plan(a.g, a.sched, m=m, n_gpus=G, placement="optimized", protocol=proto) as p:
            assert p.check_bounds(37)


def test_gk256_in_bounds(artifacts):
    if "gk256_4" not in list_artifacts():
        pytest.skip("artifact missing")
    from paper_2309_13541_b200.artifacts import load_artifact
    a = load_artifact("gk256_4", native=True, verify=False)
    with Plan(a.g, a.sched, m=4096 + 64, n_gpus=8, reuse_scratch=True) as p:
        assert p.check_bounds(148)


@pytest.mark.parametrize("name", ["gk8_2", "hypercube3", "torus4x4x4", "ts_torus3x3"])
@pytest.mark.parametrize("G", [1, 2, 4])
@pytest.mark.parametrize("mode", ["chain", "chaind"])
def test_linked_chains_in_bounds(name, G, mode, artifacts):
    """Chains at sizes where hops link (>= one TMA ring per unit), incl. a
    shard size that is not 16-byte clean."""
    a = artifacts(name)
    for m in (1 << 20, (1 << 20) + 48, 262144 + 4):
        with Plan(a.g, a.sched, m=m, n_gpus=G, placement="optimized") as p:
            p.set_schedule(mode, 262144)
            assert p.check_bounds(148)
