"""Where does the time of a small all-to-all go?  (one process, 1 or 2 GPUs)

Per variant: CUDA-event time per execute for back-to-back executes (no L2
flush), the same executes replayed from a CUDA graph, and the kernel's own
%globaltimer span (first CTA start -> last CTA exit).  The difference between
event time and kernel span is launch + completion overhead.
  python tools/latency_probe.py [--m 4096] [--config hypercube3]
Prints one JSON line per variant.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2309_13541_b200.artifacts import load_artifact
    from paper_2309_13541_b200.dist import local_nodes
    from paper_2309_13541_b200.executor import Plan, timeline_summary
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=4096)
    ap.add_argument("--config", default="hypercube3")
    ap.add_argument("--iters", type=int, default=50)
    a = ap.parse_args()
    art = load_artifact(a.config)
    n, m = art.g.n, a.m
    G_max = min(2, torch.cuda.device_count())
    ap_ctas = [int(x) for x in os.environ.get("PROBE_CTAS", "0").split(",")]
    variants = [(proto, eng, c) for proto, eng in
                [("simple", None), ("ll", None), ("ll", ("tma", 4096, 1))] for c in ap_ctas]
    for G in sorted({1, G_max}):
        for proto, eng, nctas in variants:
            plans = []
            for r in range(G):
                p = Plan(art.g, art.sched, m=m, n_gpus=G, protocol=proto)
                if eng:
                    p.set_engine(*eng)
                plans.append(p.bind(r, device=r, num_ctas=nctas))
            if G > 1:
                ptrs = [p.arena_ptr() for p in plans]
                for p in plans:
                    p.import_pointers(ptrs)
            sends = [torch.randint(0, 256, (len(local_nodes(p, r)), n, m), dtype=torch.uint8,
                                   device=f"cuda:{r}") for r, p in enumerate(plans)]
            recvs = [torch.empty_like(s) for s in sends] if proto == "ll" or G == 1 else \
                [p.recv_buffer() for p in plans]
            streams = [torch.cuda.Stream(r) for r in range(G)]

            def launch():
                for r, p in enumerate(plans):
                    p.execute(sends[r], recvs[r], stream=streams[r])

            for _ in range(5):
                launch()
            for p in plans:
                p.sync()
            # back-to-back executes
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[0])
            for _ in range(a.iters):
                launch()
            e1.record(streams[0])
            for p in plans:
                p.sync()
            t_b2b = e0.elapsed_time(e1) * 1e3 / a.iters
            tl = timeline_summary(plans[0].read_timeline(), "static")
            # single execute with events (after idle)
            singles = []
            for _ in range(10):
                for r in range(G):
                    torch.cuda.synchronize(r)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(streams[0])
                launch()
                a1.record(streams[0])
                for r in range(G):
                    torch.cuda.synchronize(r)
                singles.append(a0.elapsed_time(a1) * 1e3)
            tl1 = timeline_summary(plans[0].read_timeline(), "static")
            # CUDA graph of the same executes (one graph per GPU)
            graphs = []
            for r, p in enumerate(plans):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.device(r), torch.cuda.stream(streams[r]):
                    with torch.cuda.graph(g, stream=streams[r]):
                        for _ in range(a.iters):
                            p.execute(sends[r], recvs[r], stream=streams[r])
                graphs.append(g)
            for r in range(G):
                torch.cuda.synchronize(r)
            e0.record(streams[0])
            for r, g in enumerate(graphs):
                with torch.cuda.device(r), torch.cuda.stream(streams[r]):
                    g.replay()
            e1.record(streams[0])
            for r in range(G):
                torch.cuda.synchronize(r)
            t_graph = e0.elapsed_time(e1) * 1e3 / a.iters
            ok = all(torch.equal(recvs[r].cpu(), torch.cat([sends[q].cpu() for q in range(G)])
                                 .transpose(0, 1)[local_nodes(plans[r], r)]) for r in range(G))
            print(json.dumps({"config": a.config, "m": m, "G": G, "proto": proto, "engine": eng,
                              "num_ctas": nctas,
                              "noncoop": os.environ.get("A2A_NONCOOP", "0"),
                              "b2b_us": round(t_b2b, 2), "graph_us": round(t_graph, 2),
                              "single_us_p50": round(sorted(singles)[len(singles) // 2], 2),
                              "kernel_us_b2b_last": tl["kernel_us"], "kernel_us_single": tl1["kernel_us"],
                              "entry_us": tl1["entry_us"], "step_done_us": tl1["step_done_us"],
                              "ok": bool(ok)}), flush=True)
            del graphs
            for p in plans:
                p.close()


if __name__ == "__main__":
    main()
