"""Fluid-model estimate of sub-unit cut-through before building it (VERDICT r1
item 5).  Publishing readiness per 128-256 KiB group inside a 1 MiB unit acts
like smaller units without the per-unit system-scope publication cost, so the
calibrated model (a2a_plan_simulate, csrc/a2a_sim.cpp) is run with small units
and a small per-unit cost as the proxy, against today's 1 MiB units at the
calibrated 10 us and the static programs.  One line per (config, GPUs,
lowering): modelled ms per all-to-all.

  python tools/sim_subunit.py > profiles/r02_sim_subunit.txt
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2309_13541_b200.artifacts import load_artifact  # noqa: E402

CASES = (("static", None), ("spread:1048576", 10.0), ("spread:262144", 10.0),
         ("spread:262144", 1.0), ("spread:131072", 1.0), ("spread:65536", 0.5))

if __name__ == "__main__":
    for name, m in (("gk8_2", 16 << 20), ("hypercube3", 16 << 20)):
        a = load_artifact(name)
        for G in (4, 8):
            for low in ("hop", "balanced"):
                art, pl = (a, "optimized") if low == "hop" else bench.balanced_artifact(a, m, G, "optimized")
                res = {}
                for sched, us in CASES:
                    with bench.make_plan(art, m, G, pl, sched) as p:
                        kw = {} if us is None else {"unit_us_sys": us}
                        res[f"{sched} unit_us_sys={us}"] = round(p.simulate(148, **kw) * 1e3, 4)
                print(name, f"G={G}", low, res, flush=True)
