"""Scaling / message-size sweeps on B200 (BASELINE.json configs 2-5).

Runs bench.measure for a list of (artifact, m) cases on the GPUs of this job
(single process for G=1, torchrun for G>1) and appends one JSON line per case
to --out (rank 0).  Every line carries our algBW (whole job and per GPU), the
topology-bound fraction, the roofline and NCCL all_to_all_single on the same
bytes.

Presets:
  scaling         gk8_2 16 MiB, hypercube3 4 MiB, torus4x4x4 4 MiB, gk64_4 1 MiB
  hypercube       hypercube3, m = 4 KiB * 4^k, k = 0..7 (4 KiB .. 64 MiB)
  gk256           gk256_4 and gk256_4_h2 at 1 MiB (cases whose memory does not fit skip)

  torchrun --nproc-per-node 8 tools/sweep.py --preset scaling --out profiles/x.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PRESETS = {
    "scaling": [("gk8_2", 16 << 20), ("hypercube3", 4 << 20), ("torus4x4x4", 4 << 20),
                ("gk64_4", 1 << 20)],
    "hypercube": [("hypercube3", 4096 * 4 ** k) for k in range(8)],
    "gk256": [("gk256_4", 1 << 20), ("gk256_4_h2", 1 << 20)],
}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default=None)
    ap.add_argument("--cases", default="",
                    help="config:m[@schedule],... (a per-case schedule overrides --schedule)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--mem-limit-gib", type=float, default=150.0)
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--placement", default="optimized",
                    help="optimized | contiguous | explicit node->GPU list '0,1,0,...'")
    ap.add_argument("--num-ctas", type=int, default=0)
    ap.add_argument("--schedule", default=None,
                    help="static | dynamic[:bytes] | auto; default: $A2A_SCHED or static")
    ap.add_argument("--lowering", default="hop", choices=["hop", "balanced", "auto"],
                    help="path -> step lowering (bench.balanced_artifact for 'balanced'; 'auto' "
                         "with --schedule auto: time both, keep the faster, as bench.py does)")
    a = ap.parse_args(argv)
    if a.placement not in ("optimized", "contiguous"):
        a.placement = [int(x) for x in a.placement.split(",")]
    cases = [(name, m, None) for name, m in PRESETS.get(a.preset, [])] if a.preset else []
    for c in filter(None, a.cases.split(",")):
        c, _, case_sched = c.partition("@")
        name, m = c.split(":")
        cases.append((name, int(m), case_sched or None))

    import bench
    from paper_2309_13541_b200.artifacts import list_artifacts, load_artifact
    from paper_2309_13541_b200.executor import Plan

    ctx = bench.Ctx()
    have = set(list_artifacts())
    for name, m, case_sched in cases:
        rec = {"config": name, "m_bytes": m, "n_gpus": ctx.world}
        if name not in have:
            rec["skipped"] = "artifact not generated"
        else:
            art = load_artifact(name)
            placement = a.placement
            auto_low = a.lowering == "auto" and (case_sched or a.schedule) == "auto"
            if a.lowering == "balanced" and art.routes is not None:
                art, placement = bench.balanced_artifact(art, m, ctx.world, a.placement)
            rec["lowering"] = a.lowering if art.routes is not None else "ts artifact"
            with Plan(art.g, art.sched, m=m, n_gpus=ctx.world, placement=placement) as p:
                mem = max(p.gpu_info(g)["send_bytes"] * 2 + p.gpu_info(g)["scratch_bytes"]
                          for g in range(ctx.world))
            if mem > a.mem_limit_gib * 2 ** 30:
                rec["skipped"] = f"needs {mem / 2**30:.1f} GiB per GPU"
            else:
                t0 = time.time()
                sched = case_sched or a.schedule or os.environ.get("A2A_SCHED") or "static"
                tune = None
                if sched == "auto" and auto_low:
                    ns = argparse.Namespace(schedule="auto", lowering="auto", num_ctas=a.num_ctas,
                                            placement=a.placement if isinstance(a.placement, str)
                                            else "optimized")
                    art, placement, sched, low, tune, _ = bench.choose_execution(ctx, ns, art, m,
                                                                                 placement)
                    rec["lowering"] = low
                elif sched == "auto":
                    sched, tune = bench.autotune_schedule(ctx, art, m, placement=placement,
                                                          num_ctas=a.num_ctas)
                r = bench.measure(ctx, art, m, a.steps, a.warmup, nccl=not a.no_nccl,
                                  e2e=False, clocks=os.environ.get("A2A_NO_CLOCKS") != "1", placement=placement, schedule=sched,
                                  num_ctas=a.num_ctas)
                rec["schedule"] = sched
                rec["schedule_autotune_ms"] = tune
                rec.update({
                    "nodes": art.g.n, "hop_ops": len(art.sched.instructions),
                    "nsteps": art.sched.nsteps, "Q": art.sched.Q,
                    "ms": round(r["T"] * 1e3, 4), "step_ms_dist": r["step_ms_dist"],
                    "algbw_gbs": round(r["value"], 2),
                    "algbw_per_gpu_gbs": round(r["per_gpu"], 2),
                    "t_lb_ms": round(r["t_lb"] * 1e3, 4), "bound_frac": round(r["bound_frac"], 4),
                    "t_hbm_ms": round(r["t_hbm"] * 1e3, 4),
                    "bound_frac_both": round(r["t_both"] / r["T"], 4),
                    "roofline": r["roofline"], "nccl": r["nccl"], "recv_ok": r["recv_ok"],
                    "clocks": r["clocks"], "sync_flags": r["sync"],
                    "host_enqueue_us_per_step": r["host_enqueue_us_per_step"],
                    "flush_ms_p50_by_rank": r["flush_ms_p50_by_rank"],
                    "step_period_ms_p50_by_rank": r["step_period_ms_p50_by_rank"],
                    "step_ms_by_rank": r["step_ms_by_rank"],
                    "kernel_timeline": r["kernel_timeline"],
                    "egress_max_bytes": r["egress_max"], "scratch_bytes": r["scratch_bytes"],
                    "placement": a.placement, "l2": r["l2"], "num_ctas": r["num_ctas"],
                    "wall_s": round(time.time() - t0, 1)})
        if ctx.rank == 0:
            line = json.dumps(rec)
            print(line, flush=True)
            if a.out:
                with open(a.out, "a") as fh:
                    fh.write(line + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
