"""Device-side race hunting: perturbed interleavings on the GPU.

compute-sanitizer is closed on this pool, and the host emulator
(tests/test_emulation.py) is a model of the device, not the device.  This is
the on-hardware counterpart.  With sync_mode bit 6 every CTA naps a
pseudo-random 0-16 us (one time in 16 up to 260 us) before each step, unit or
chain task; the nap is keyed by the execute's epoch, so every repeat runs a
different interleaving.  Each
repeat uses a fresh send buffer, so a stale read of the previous repeat's
scratch or recv cannot pass by accident.  The check is the reference's
delivery postcondition, recv[d][s] == send[s][d] (evaluate.py:114-126).

The mutation self-test (bit 7: dependency waits skipped) must FAIL under the
same perturbation.  That shows the check can see a missing dependency on the
device.
"""
from __future__ import annotations

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

DEFAULT_SYNC = 2          # a2a_plan_set_sync_mode default
PERTURB, NO_WAITS = 64, 128


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


def _runs(a, m, sched, mode, reps, proto="simple", engine="tma", seed=0, ctas=0,
          stop_on_bad=False):
    """Execute `reps` all-to-alls with fresh random send buffers; return how
    many delivered the exact transpose (with `stop_on_bad`, stop at the first
    wrong one and return -1)."""
    from paper_2309_13541_b200.executor import Plan
    n = a.g.n
    g = torch.Generator(device="cuda").manual_seed(seed)
    good = 0
    with Plan(a.g, a.sched, m=m, protocol=proto) as p:
        p.set_engine(engine)
        if proto == "simple":
            p.set_schedule_spec(sched)
        p.bind(0, num_ctas=ctas)
        p.set_sync_mode(mode)
        p.set_timeout(20.0)
        r = torch.empty((n, n, m), dtype=torch.uint8, device="cuda")
        for _ in range(reps):
            s = torch.randint(0, 256, (n, n, m), dtype=torch.uint8, device="cuda", generator=g)
            p.execute(s, r)
            p.sync()
            ok = bool(torch.equal(r, s.transpose(0, 1).contiguous()))
            if stop_on_bad and not ok:
                return -1
            good += ok
    return good


CASES = [("gk8_2", 65536 + 40), ("gk8_2", 1 << 20), ("torus2x4_h2", 262144 + 16),
         ("hypercube3", 1 << 20), ("ts_torus3x3", 65536), ("torus4x4x4", 16384),
         ("gk8_2_h1", 4096 + 7), ("torus2x4", 300000), ("ts_gk8_2", 65536 + 16),
         ("ts_hypercube3", 1000), ("gk64_4", 8192)]


@pytest.mark.parametrize("name,m", CASES)
@pytest.mark.parametrize("sched,engine", [("static", "tma"), ("static", "lsu"),
                                          ("cp:65536", "tma"), ("mix:65536", "tma"),
                                          ("spread:65536", "lsu"), ("chain:262144", "tma"),
                                          ("ll", None), ("ll128", None)])
def test_perturbed_interleavings_deliver_transpose(name, m, sched, engine, artifacts):
    a = artifacts(name)
    proto = sched if sched in ("ll", "ll128") else "simple"
    reps = 6
    good = _runs(a, m, sched, DEFAULT_SYNC | PERTURB, reps, proto=proto,
                 engine=engine or "tma", seed=m)
    assert good == reps


@pytest.mark.parametrize("name,m", [("gk8_2", 1 << 20), ("hypercube3", 1 << 20),
                                    ("torus2x4_h2", 262144 + 16), ("torus4x4x4", 16384)])
@pytest.mark.parametrize("sched", ["static", "cp:65536", "mix:65536", "spread:65536"])
def test_mutation_without_waits_is_caught(name, m, sched, artifacts, monkeypatch):
    """Same perturbation with the dependency waits skipped: the transpose
    check must catch the missing dependencies in at least one repeat."""
    a = artifacts(name)
    monkeypatch.setenv("A2A_ALLOW_MUTATION", "1")
    reps = 24          # the first wrong transpose ends the test (usually the first repeat)
    good = _runs(a, m, sched, DEFAULT_SYNC | PERTURB | NO_WAITS, reps, seed=7, stop_on_bad=True)
    assert good < 0, f"{reps} perturbed runs without dependency waits all delivered"


@pytest.mark.parametrize("name,m", [("gk8_2", 1 << 20), ("torus4x4x4", 65536)])
@pytest.mark.parametrize("sched", ["static", "cp:65536", "spread:65536", "chain:262144"])
@pytest.mark.parametrize("ctas", [1, 3, 37])
def test_perturbed_few_ctas(name, m, sched, ctas, artifacts):
    """Few CTAs: each runs many steps / units in a row, so the naps reorder
    long per-CTA sequences rather than one item per SM."""
    a = artifacts(name)
    assert _runs(a, m, sched, DEFAULT_SYNC | PERTURB, 3, seed=ctas, ctas=ctas) == 3
