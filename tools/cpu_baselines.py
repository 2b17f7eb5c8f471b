"""CPU baselines of SURVEY.md §8d, timed in the build container (not the GPU box:
the reference tree exists only here).

Per frozen config, one core each:
  1. the reference's ``replay_timestep_schedule`` as-is (symbolic: chunk-id
     sets, no bytes; reference pkg/src/a2aflow/evaluate.py:56-127), wall time
     of one replay of its own parse of our XML;
  2. this package's ``executor.replay_timestep_schedule`` (same signature and
     result; validation + modelled T in csrc/a2a_plan.cpp), plan creation
     included;
  3. the byte-moving restatement (oracle/replay_bytes.c, 1 thread, reused
     scratch workspace) at m = 1 MiB per pair (N <= 64; GK(256,4) needs 128 GiB
     of host buffers at 1 MiB).
Writes a JSON object per config to stdout (and to --out).

Usage: python tools/cpu_baselines.py [--out profiles/r01_cpu_baselines_container.json] [CONFIG ...]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

DEFAULT = ["torus2x4", "hypercube3", "gk8_2", "ts_gk8_2", "torus4x4x4", "gk64_4", "gk256_4"]


def _best(fn, budget_s=2.0, max_iters=20):
    times, t0 = [], time.perf_counter()
    while len(times) < max_iters and (not times or time.perf_counter() - t0 < budget_s):
        a = time.perf_counter()
        out = fn()
        times.append(time.perf_counter() - a)
    return sorted(times)[len(times) // 2], len(times), out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("configs", nargs="*")
    args = ap.parse_args(argv)

    import numpy as np
    from make_golden import RE, RG, _find, plain, ref_sched   # imports the read-only reference

    from c_oracle import ops_array, replay_bytes_c, workspace
    from paper_2309_13541_b200.artifacts import ARTIFACT_DIR, load_artifact
    from paper_2309_13541_b200.executor import replay_timestep_schedule

    host = {"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count(),
            "where": "build container (no GPU); the GPU box's host cores are timed by bench.py"}
    try:
        with open("/proc/cpuinfo") as fh:
            host["cpu"] = next(x.split(":", 1)[1].strip() for x in fh if x.startswith("model name"))
    except (OSError, StopIteration):
        pass
    res = {"host": host, "configs": {}}
    for name in args.configs or DEFAULT:
        art = load_artifact(name, native=True)
        d = os.path.join(ARTIFACT_DIR, name)
        rg = RG.load_graph(plain(_find(d, "graph.json")))
        rs = ref_sched(art.sched)
        n_ops = len(art.sched.ops_array)
        big = n_ops > 100000
        t_ref, k_ref, (T_ref, _) = _best(lambda: RE.replay_timestep_schedule(rg, rs, m=1.0),
                                         budget_s=0 if big else 2.0, max_iters=1 if big else 20)
        t_nat, k_nat, (T_nat, _) = _best(lambda: replay_timestep_schedule(art.g, art.sched, m=1.0))
        rec = {"n": art.g.n, "hop_ops": n_ops,
               "reference_replay_s": t_ref, "reference_replay_runs": k_ref,
               "native_replay_s": t_nat, "native_replay_runs": k_nat,
               "speedup": round(t_ref / t_nat, 1), "T_identical": T_ref == T_nat}
        if art.g.n <= 64:
            m = 1 << 20
            n = art.g.n
            send = np.random.default_rng(0).integers(0, 256, size=(n, n, m), dtype=np.uint8)
            recv = np.zeros_like(send)
            ops = ops_array(art.sched)
            ws = workspace(art.sched, n, m, ops)
            t_b, k_b, _ = _best(lambda: replay_bytes_c(art.g, art.sched, send, m, nthreads=1,
                                                       recv=recv, ops=ops, ws=ws), budget_s=3.0)
            rec["bytes_1core"] = {"m": m, "s": t_b, "runs": k_b,
                                  "algbw_gbs": round(n * (n - 1) * m / t_b / 1e9, 3),
                                  "recv_ok": bool(np.array_equal(recv, np.swapaxes(send, 0, 1)))}
            del send, recv
        res["configs"][name] = rec
        print(name, json.dumps(rec), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)
            fh.write("\n")


if __name__ == "__main__":
    main()
