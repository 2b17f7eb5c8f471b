"""`eval` command of the reference CLI, on the B200 executor.

Mirrors ``a2a eval --graph G (--sched X | --routes R) [--m M] [--b B] [--sync S]``
(reference pkg/src/a2aflow/cli.py:133-139, :326-343):

* ``--sched X``: load the graph JSON and the ts-mode XML schedule, replay it
  (same validation, same EvalError texts, bit-identical T) and print
  ``T = <T:.9g>, delivered = True``;
* ``--routes R`` (a weighted path set, the reference's route JSON): the
  cut-through fluid time ``eval_path_alltoall`` (evaluate.py:130-139), printed
  as ``T = <T:.9g>`` (fluid.py);
* neither: ``error: eval needs --sched or --routes``.

Any error prints ``error: <message>`` on stderr and exits 1, usage errors exit
2 (argparse), as the reference's ``main`` does (cli.py:419-431).  The
reference's run manifest (cli.py:40-55) is not written: it records the
reference's own pipeline runs.

Additions of this package (flags the reference does not have):

* ``--path-routes R`` with a path-mode ``--sched``: lower the path schedule and
  its route sidecar hop i -> step i natively (a2a_lower_path_files) and replay
  that (the reference replay only accepts ts schedules, evaluate.py:70-71).
* ``--execute``: also move real bytes on GPU ``--device`` (integer ``--m``
  bytes per shard, every virtual node on that GPU), check recv against the
  transpose of send and print the device time.  Multi-GPU runs go through
  ``bench.py`` / ``tools/sweep.py`` (one process per GPU).

* ``--sched`` may also be a binary op table written by ``pack``.
* ``pack --sched X [--routes R --graph G] -o OUT``: parse (and, with
  ``--routes``, lower) a schedule once and write it as a binary op table
   plus ``OUT.manifest.json`` in the shape of the
  reference's run manifest (command, argv, seed, version, sha256 of inputs and
  outputs, wall_clock_s; reference cli.py:38-55).

Usage: ``python -m paper_2309_13541_b200.cli eval --graph g.json --sched s.xml``.
"""
from __future__ import annotations

import argparse
import json
import sys
import time


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="b200-a2a")
    sub = p.add_subparsers(dest="command", required=True)
    e = sub.add_parser("eval", help="replay / evaluate / execute a schedule")
    e.add_argument("--graph", required=True)
    e.add_argument("--sched", default=None,
                   help="XML schedule or op table (ts mode, or path mode with --path-routes)")
    e.add_argument("--routes", default=None, help="route JSON (path mode): fluid eval_path_alltoall")
    e.add_argument("--path-routes", default=None,
                   help="route sidecar of a path-mode --sched: lower it hop i -> step i")
    e.add_argument("--m", type=float, default=1.0)
    e.add_argument("--b", type=float, default=1.0)
    e.add_argument("--sync", type=float, default=0.0)
    e.add_argument("--execute", action="store_true", help="also run it on a GPU with real bytes")
    e.add_argument("--device", type=int, default=0)
    e.add_argument("--schedule", default="static",
                   help="execution schedule for --execute: static | <mode>[:unit[:R]]")
    k = sub.add_parser("pack", help="write a schedule as a binary op table")
    k.add_argument("--sched", required=True, help="XML schedule or op table (ts, or path with --routes)")
    k.add_argument("--routes", default=None, help="route sidecar: lower the path schedule hop i -> step i")
    k.add_argument("--graph", default=None, help="graph JSON (node count for --routes; checked with replay)")
    k.add_argument("-o", "--out", required=True)
    return p


def _load(args):
    from .graphs import load_graph
    from .native_io import load_schedule, lower_path_files
    g = load_graph(args.graph)
    if args.path_routes:
        sched = lower_path_files(args.sched, args.path_routes, n_phys=g.n)
    else:
        sched = load_schedule(args.sched)
    return g, sched


def _execute(g, sched, args) -> str:
    import numpy as np
    import torch

    from .executor import Plan
    if args.m != int(args.m) or args.m < 0:
        raise ValueError(f"--execute needs an integer shard size in bytes, got --m {args.m}")
    m = int(args.m)
    n = g.n
    gen = torch.Generator().manual_seed(0)
    send = torch.randint(0, 256, (n, n, m), dtype=torch.uint8, generator=gen)
    dev = torch.device("cuda", args.device)
    with Plan(g, sched, m=m) as plan:
        if args.schedule != "static":
            plan.set_schedule_spec(args.schedule)
        plan.bind(0, device=args.device)
        s = send.to(dev)
        r = torch.zeros_like(s)
        stream = torch.cuda.current_stream(dev)
        plan.execute(s, r, stream=stream)          # warm-up (first launch)
        plan.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        plan.execute(s, r, stream=stream)
        e1.record(stream)
        plan.sync()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        ok = bool(np.array_equal(r.cpu().numpy(), send.transpose(0, 1).contiguous().numpy()))
    if not ok:
        raise RuntimeError("executed all-to-all: recv differs from the transpose of send")
    gbs = n * (n - 1) * m / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    return f"executed on cuda:{args.device}: {ms:.4f} ms, {gbs:.1f} GB/s algBW, recv == transpose(send): True"


def _cmd_eval(args) -> None:
    if not args.sched:
        if not args.routes:
            from .graphs import GraphError
            raise GraphError("eval needs --sched or --routes")
        from .fluid import eval_path_alltoall, load_routes
        from .graphs import load_graph
        T = eval_path_alltoall(load_graph(args.graph), load_routes(args.routes), m=args.m, b=args.b)
        print(f"T = {T:.9g}")
        return
    from .executor import replay_timestep_schedule
    g, sched = _load(args)
    T, ok = replay_timestep_schedule(g, sched, m=args.m, b=args.b, sync_latency=args.sync)
    print(f"T = {T:.9g}, delivered = {ok}")
    if args.execute:
        print(_execute(g, sched, args))


def _cmd_pack(args, argv) -> None:
    from . import __version__
    from .native_io import load_schedule, lower_path_files, save_schedule_table, sha256_file
    started = time.time()
    inputs = [args.sched] + [x for x in (args.routes, args.graph) if x]
    g = None
    if args.graph:
        from .graphs import load_graph
        g = load_graph(args.graph)
    if args.routes:
        sched = lower_path_files(args.sched, args.routes, n_phys=g.n if g is not None else 0)
    else:
        sched = load_schedule(args.sched)
    if g is not None and sched.mode == "ts":
        from .executor import replay_timestep_schedule
        replay_timestep_schedule(g, sched)        # same rejects as eval, before writing
    save_schedule_table(sched, args.out)
    manifest = {"command": "pack", "argv": list(argv), "seed": None, "version": __version__,
                "inputs": {p: sha256_file(p) for p in inputs},
                "outputs": {args.out: sha256_file(args.out)},
                "wall_clock_s": time.time() - started}
    with open(args.out + ".manifest.json", "w") as fh:
        json.dump(manifest, fh, indent=1)
        fh.write("\n")
    print(f"wrote {args.out}: mode {sched.mode}, n={sched.n}, nsteps={sched.nsteps}, "
          f"Q={sched.Q}, {len(sched.ops_array)} ops")


def main(argv: list[str] | None = None) -> int:
    argv = sys.argv[1:] if argv is None else list(argv)
    args = build_parser().parse_args(argv)
    try:
        if args.command == "pack":
            _cmd_pack(args, argv)
        else:
            _cmd_eval(args)
    except Exception as ex:   # noqa: BLE001 - CLI boundary, as the reference's main
        print(f"error: {ex}", file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
