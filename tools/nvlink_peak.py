"""NVLink peer bandwidth on this box (one process, two GPUs).

1. copy engine: torch peer copy cuda:0 -> cuda:1 (1 GiB), one direction and
   both directions at once;
2. this executor: a 2-node, 1-step full exchange (node 0 on GPU 0, node 1 on
   GPU 1; each sends one m-byte shard to the other) with the TMA engine and the
   LSU engine -- the SM-driven peer-store ceiling of a2a_exec_kernel.
Prints one JSON line.
"""
from __future__ import annotations

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _time(fn, iters=10):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iters)]
    fn()
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    ts = []
    for a, b in ev:
        a.record(torch.cuda.current_stream(0))
        fn()
        b.record(torch.cuda.current_stream(0))
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ts.append(a.elapsed_time(b) / 1e3)
    return sorted(ts)[len(ts) // 2]


def main():
    from paper_2309_13541_b200.executor import Plan
    from paper_2309_13541_b200.graphs import Digraph
    from paper_2309_13541_b200.schedule import ChunkedSchedule, Instruction
    out = {}
    n = 1 << 30
    a0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    a1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    b0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    t = _time(lambda: b1.copy_(a0, non_blocking=True))
    out["copy_engine_one_way_gbs"] = round(n / t / 1e9, 1)
    s1 = torch.cuda.Stream(1)

    def both():
        b1.copy_(a0, non_blocking=True)
        with torch.cuda.stream(s1):
            b0.copy_(a1, non_blocking=True)
    t = _time(both)
    out["copy_engine_bidir_per_direction_gbs"] = round(n / t / 1e9, 1)
    del a0, b1, a1, b0
    torch.cuda.empty_cache()

    g = Digraph.from_edges(2, [(0, 1, 1.0), (1, 0, 1.0)])
    m = 512 << 20
    both_ways = [Instruction(0, 0, 1, 0, 1, 0, 1), Instruction(0, 1, 0, 1, 0, 0, 1)]
    # one-way: shard (1,0) travels 1 -> 0 at step 0 as before, shard (0,1) only at step 1
    # (the timed step-0 traffic of the first all-to-all is then one direction at a time)
    variants = [("tma", (0, 0), "bidir"), ("lsu", (0, 0), "bidir"), ("tma", (65536, 3), "bidir"),
                ("tma", (16384, 12), "bidir"), ("tma", (0, 0), "oneway")]
    for engine, ring, mode in variants:
        ins = both_ways if mode == "bidir" else [Instruction(0, 0, 1, 0, 1, 0, 1),
                                                 Instruction(1, 1, 0, 1, 0, 0, 1)]
        sched = ChunkedSchedule(n=2, nsteps=1 if mode == "bidir" else 2, chunk_bytes=1.0, Q=1,
                                mode="ts", instructions=ins)
        plans = [Plan(g, sched, m=m, n_gpus=2, copy_self=False).set_engine(engine, *ring)
                 .bind(r, device=r) for r in range(2)]
        ptrs = [p.arena_ptr() for p in plans]
        for p in plans:
            p.import_pointers(ptrs)
        sends = [torch.randint(0, 256, (1, 2, m), dtype=torch.uint8, device=f"cuda:{r}")
                 for r in range(2)]
        recvs = [p.recv_buffer() for p in plans]

        def run():
            for r, p in enumerate(plans):
                p.execute(sends[r], recvs[r], stream=torch.cuda.current_stream(r))
        t = _time(run)
        for p in plans:
            p.sync()
        ok = all(torch.equal(recvs[r][0, 1 - r].cpu(), sends[1 - r][0, r].cpu()) for r in range(2))
        tag = f"a2a_exec_{engine}{'' if ring == (0, 0) else f'_{ring[0]}x{ring[1]}'}_{mode}"
        # bidir: m bytes each way in t; oneway: 2 sequential one-way transfers of m in t
        out[tag + "_gbs_per_direction"] = round((m if mode == "bidir" else 2 * m) / t / 1e9, 1)
        out[tag + "_ok"] = ok
        for p in plans:
            p.close()
        del sends, recvs
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
