"""Fluid model (Plan.simulate / a2a_plan_simulate) vs measured B200 runs.

Prints, for every measured (config, m, G, schedule) below, the measured p50
all-to-all time, the modelled time and their ratio, and per (config, G) whether
the model ranks the schedules in the measured order.  With --predict, prints the
model's times for GPU counts that were not measured (8 GPUs).

Measured numbers: profiles/r01_queue_split_ab_G{2,4}.jsonl,
r01_spread_ab_G4.jsonl, r01_schedule_ab_G{12,4}.jsonl, r01_bench_final6_b1.log,
r01_ready_queue_ab_G{2,4}.jsonl.
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (config, m, G, schedule) -> measured p50 ms
MEASURED = {
    ("gk8_2", 16 << 20, 1, "static"): 0.6887,
    ("gk8_2", 16 << 20, 1, "mix:1048576"): 0.6626,
    ("gk8_2", 16 << 20, 1, "cp:1048576"): 0.6612,
    ("gk8_2", 16 << 20, 2, "static"): 0.4437,
    ("gk8_2", 16 << 20, 2, "mix:1048576"): 0.4349,
    ("gk8_2", 16 << 20, 2, "cp:1048576"): 0.4484,
    ("gk8_2", 16 << 20, 2, "cp:1048576:16"): 0.525,
    ("gk8_2", 16 << 20, 2, "cp:1048576:64"): 0.4308,
    ("gk8_2", 16 << 20, 2, "cp:1048576:96"): 0.5322,
    ("gk8_2", 16 << 20, 4, "static"): 0.709,
    ("gk8_2", 16 << 20, 4, "mix:1048576"): 0.6468,
    ("gk8_2", 16 << 20, 4, "cp:1048576"): 0.682,
    ("gk8_2", 16 << 20, 4, "spread:1048576"): 0.6561,
    ("gk8_2", 16 << 20, 4, "cp:1048576:32"): 0.8416,
    ("gk8_2", 16 << 20, 4, "cp:1048576:96"): 0.6787,
    ("hypercube3", 16 << 20, 4, "static"): 0.5146,
    ("hypercube3", 16 << 20, 4, "mix:1048576"): 0.4692,
    ("hypercube3", 16 << 20, 4, "cp:1048576"): 0.5124,
    ("hypercube3", 16 << 20, 2, "static"): 0.4111,
    ("hypercube3", 16 << 20, 2, "mix:1048576"): 0.4202,
    ("torus4x4x4", 4 << 20, 2, "static"): 7.9773,
    ("torus4x4x4", 4 << 20, 2, "mix:1048576"): 7.8383,
    ("torus4x4x4", 4 << 20, 4, "static"): 6.7574,
    ("torus4x4x4", 4 << 20, 4, "mix:1048576"): 8.0595,
    ("torus4x4x4", 4 << 20, 4, "spread:1048576"): 6.6821,
    ("torus4x4x4", 4 << 20, 4, "cp:1048576"): 12.5188,
    # unit-size A/B (profiles/r01_unit_size_ab_G{2,4}.jsonl)
    ("gk8_2", 16 << 20, 2, "cp:262144"): 0.7338,
    ("gk8_2", 16 << 20, 2, "mix:262144"): 0.5673,
    ("gk8_2", 16 << 20, 2, "list:1048576"): 0.4485,
    ("gk8_2", 16 << 20, 2, "cp:4194304"): 0.4996,
    ("gk8_2", 16 << 20, 4, "cp:262144"): 0.902,
    ("gk8_2", 16 << 20, 4, "mix:262144"): 0.8016,
    ("gk8_2", 16 << 20, 4, "list:1048576"): 0.7454,
    ("gk8_2", 16 << 20, 4, "cp:4194304"): 0.7484,
    # ready queue (profiles/r01_ready_queue_ab_G{2,4}.jsonl; G=1: bench autotune, r01_bench_final6_b1.log)
    ("gk8_2", 16 << 20, 1, "ready:1048576"): 0.6764,
    ("gk8_2", 16 << 20, 2, "ready:1048576"): 0.4813,
    ("gk8_2", 16 << 20, 2, "ready:2097152"): 0.5313,
    ("gk8_2", 16 << 20, 4, "ready:1048576"): 0.6861,
    ("gk8_2", 16 << 20, 4, "ready:2097152"): 0.7321,
    ("hypercube3", 4 << 20, 2, "ready:1048576"): 0.1545,
    ("hypercube3", 4 << 20, 4, "ready:1048576"): 0.164,
    ("gk256_4", 1 << 20, 4, "static"): 34.0651,
    ("gk256_4", 1 << 20, 4, "mix:1048576"): 49.3659,
    ("gk256_4", 1 << 20, 4, "spread:1048576"): 34.1506,
}


def model(name, m, G, sched, num_ctas=148, lowering="hop", **params):
    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    art, placement = load_artifact(name), "optimized"
    if lowering == "balanced":
        art, placement = bench.balanced_artifact(art, m, G, placement)
    with bench.make_plan(art, m, G, placement, sched) as p:
        return p.simulate(num_ctas, **params) * 1e3


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--predict", action="store_true", help="also model 8 GPUs")
    ap.add_argument("--skip-large", action="store_true", help="skip GK(256,4)")
    ap.add_argument("--param", action="append", default=[], help="name=value model parameter")
    a = ap.parse_args(argv)
    params = {k: float(v) for k, v in (x.split("=") for x in a.param)}
    rows, by = [], {}
    for (name, m, G, sched), meas in MEASURED.items():
        if a.skip_large and name == "gk256_4":
            continue
        t = model(name, m, G, sched, **params)
        rows.append((name, m, G, sched, meas, t))
        by.setdefault((name, G), []).append((sched, meas, t))
        print(f"{name:11s} m={m:>9d} G={G} {sched:16s} measured {meas:8.4f} ms  model {t:8.4f} ms"
              f"  ratio {t / meas:5.2f}", flush=True)
    agree = tot = 0
    for key, v in by.items():
        for i in range(len(v)):
            for j in range(i + 1, len(v)):
                if abs(v[i][1] - v[j][1]) / min(v[i][1], v[j][1]) < 0.03:
                    continue            # measured tie: no ranking to check
                tot += 1
                ok = (v[i][1] < v[j][1]) == (v[i][2] < v[j][2])
                agree += ok
                if not ok:
                    print(f"  order differs: {key} {v[i][0]} vs {v[j][0]}: measured "
                          f"{v[i][1]:.4f}/{v[j][1]:.4f}, model {v[i][2]:.4f}/{v[j][2]:.4f}")
    import statistics
    ratios = [t / meas for *_, meas, t in rows]
    print(f"pairwise order agreement {agree}/{tot}; model/measured median {statistics.median(ratios):.3f}, "
          f"range {min(ratios):.2f}-{max(ratios):.2f}")
    if a.predict:
        for name, m in (("gk8_2", 16 << 20), ("hypercube3", 16 << 20), ("torus4x4x4", 4 << 20)):
            for sched in ("static", "mix:1048576", "cp:1048576", "spread:1048576", "cp:1048576:64",
                          "ready:1048576"):
                print(f"predict {name} G=8 {sched:16s} {model(name, m, 8, sched, **params):8.4f} ms"
                      f"   balanced lowering {model(name, m, 8, sched, lowering='balanced', **params):8.4f} ms",
                      flush=True)


if __name__ == "__main__":
    main()
