"""Small single-GPU workload for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run): every copy engine and execution schedule on
small schedules, odd shard sizes, scratch reuse on/off; checks the transpose.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
from __future__ import annotations

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.executor import Plan
    bad = 0
    runs = 0
    for name in ("torus2x4", "gk8_2", "ts_hypercube3"):
        a = load_artifact(name)
        for m in (1000, 65536 + 16):
            for engine in ("tma", "lsu"):
                for sched in ("static", "cp", "mix"):
                    for reuse in (False, True):
                        with Plan(a.g, a.sched, m=m, reuse_scratch=reuse) as p:
                            p.set_engine(engine)
                            p.set_schedule(sched, 4096 if sched != "static" else 0)
                            p.bind(0, num_ctas=16)
                            gen = torch.Generator(device="cuda").manual_seed(m)
                            s = torch.randint(0, 256, (a.g.n, a.g.n, m), dtype=torch.uint8,
                                              device="cuda", generator=gen)
                            r = torch.zeros_like(s)
                            for _ in range(2):
                                p.execute(s, r)
                            p.sync()
                            runs += 1
                            if not torch.equal(r, s.transpose(0, 1).contiguous()):
                                bad += 1
                                print("MISMATCH", name, m, engine, sched, reuse, flush=True)
    print(f"sanitize_run: {runs} configurations, {bad} mismatches", flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
