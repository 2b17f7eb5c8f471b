"""Freeze reference-produced schedule artifacts (run in the build container only).

This script drives the UNMODIFIED reference package ``a2aflow`` (imported from
``/root/reference/pkg/src``) through its own public pipeline and writes the
results to ``artifacts/<config>/`` in the reference's own file formats:

  graph.json            a2aflow.graphs.save_graph            (src/graphs.py:550)
  aug_graph.json        host-augmented graph, if any          (src/graphs.py:447)
  wps.json              a2aflow.paths.save_routes(wps)        (src/paths.py:561)
  path.xml              emit_schedule_xml(compile_path_schedule(...))
                                                              (src/schedule.py:244, :318)
  path.xml.routes.json  the route sidecar `a2a compile` writes (src/cli.py:289-292)
  meta.json             F, Q, route counts, solver versions, wall times
  manifest.json         sha256 of every file (like src/cli.py:40-55)

MCF flows are solver-dependent (SURVEY.md finding 4), so these files are the
frozen inputs every test and benchmark runs on.  Files above 256 KiB are
gzip-compressed (``.gz``); the package's loaders read both.

Pipeline per config (SURVEY.md §3 call stacks A and B):
  g = gen_*(...) [; g_aug, mp = augment_host_bottleneck(g, h)]
  sol = mcf_decomposed(g_or_aug, commodities, workers)     (src/mcf.py:420)
  wps = extract_widest_paths(g_or_aug, sol)                (src/paths.py:263)
  routes, sched = compile_path_schedule(g_or_aug, wps, m=1.0)   (src/schedule.py:244)

tsMCF configs instead run mcf_timestepped +
compile_timestep_schedule and store ``ts.xml``.

Usage:  python tools/gen_artifacts.py CONFIG [CONFIG ...] [--workers 8]
"""
from __future__ import annotations

import argparse
import gzip
import hashlib
import json
import os
import shutil
import sys
import time
import warnings

REF_SRC = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

from a2aflow import graphs as G          # noqa: E402
from a2aflow import mcf as M             # noqa: E402
from a2aflow import paths as P           # noqa: E402
from a2aflow import schedule as S        # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "artifacts")

# name -> (kind, builder, host_capacity or None, extra)
CONFIGS = {
    # decomposed-MCF path schedules (the hot path's input)
    "torus2x4": ("path", lambda: G.gen_torus([2, 4]), None),
    "hypercube3": ("path", lambda: G.gen_hypercube(3), None),
    "gk8_2": ("path", lambda: G.gen_gen_kautz(8, 2), None),
    "torus4x4x4": ("path", lambda: G.gen_torus([4, 4, 4]), None),
    "gk64_4": ("path", lambda: G.gen_gen_kautz(64, 4), None),
    "gk256_4": ("path", lambda: G.gen_gen_kautz(256, 4), None),
    # "without extra NIC-forwarding bandwidth": host-augmented lowering
    "torus2x4_h1": ("path", lambda: G.gen_torus([2, 4]), 1.0),
    "torus2x4_h2": ("path", lambda: G.gen_torus([2, 4]), 2.0),
    "gk8_2_h1": ("path", lambda: G.gen_gen_kautz(8, 2), 1.0),
    "gk64_4_h2": ("path", lambda: G.gen_gen_kautz(64, 4), 2.0),
    "gk256_4_h2": ("path", lambda: G.gen_gen_kautz(256, 4), 2.0),
    # tsMCF schedules (row f1: same executor, different lowering)
    "ts_ring3": ("ts", lambda: G.gen_torus([3], bidirectional=False), None),
    "ts_torus2x4": ("ts", lambda: G.gen_torus([2, 4]), None),
    "ts_hypercube3": ("ts", lambda: G.gen_hypercube(3), None),
    "ts_gk8_2": ("ts", lambda: G.gen_gen_kautz(8, 2), None),
    "ts_torus3x3": ("ts", lambda: G.gen_torus([3, 3]), None),
}


class _IndexedFlows(M.LinkFlowSolution):
    """LinkFlowSolution whose flow_of(ci) is O(1).

    The reference's flow_of (src/mcf.py:79-80) scans the whole flows dict once
    per commodity, which makes extract_widest_paths quadratic (SURVEY.md §8a
    row a12; 838 s at N=256).  This subclass returns the *same* dicts in the
    *same* insertion order (one ordered pass over ``flows``), so extraction
    output is identical; only the scan is hoisted.
    """

    def __init__(self, sol):
        super().__init__(F=sol.F, commodities=sol.commodities,
                         flows=sol.flows, graph=sol.graph)
        per: dict[int, dict[int, float]] = {}
        for (c, e), v in sol.flows.items():
            per.setdefault(c, {})[e] = v
        self._per = per

    def flow_of(self, ci):
        return dict(self._per.get(ci, {}))


def _sha256(path):
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for blk in iter(lambda: fh.read(1 << 20), b""):
            h.update(blk)
    return h.hexdigest()


def _finish(dirpath, files):
    final = []
    for f in files:
        p = os.path.join(dirpath, f)
        if os.path.getsize(p) > 256 * 1024:
            with open(p, "rb") as src, gzip.GzipFile(p + ".gz", "wb", mtime=0) as dst:
                shutil.copyfileobj(src, dst)
            os.remove(p)
            f = f + ".gz"
        final.append(f)
    man = {f: _sha256(os.path.join(dirpath, f)) for f in final}
    with open(os.path.join(dirpath, "manifest.json"), "w") as fh:
        json.dump(man, fh, indent=1, sort_keys=True)
        fh.write("\n")


def gen(name, workers):
    kind, builder, h = CONFIGS[name]
    d = os.path.join(OUT, name)
    os.makedirs(d, exist_ok=True)
    import numpy
    import scipy
    meta = {"config": name, "kind": kind, "host_capacity": h,
            "scipy": scipy.__version__, "numpy": numpy.__version__,
            "reference": "a2aflow (read-only /root/reference/pkg)",
            "workers": workers}
    g = builder()
    G.save_graph(g, os.path.join(d, "graph.json"))
    files = ["graph.json"]
    meta["n"] = g.n
    meta["num_edges"] = g.num_edges
    t0 = time.time()
    if kind == "ts":
        l_max = G.diameter(g)
        ts = M.mcf_timestepped(g, l_max=l_max)
        meta["t_solve_s"] = time.time() - t0
        sched = S.compile_timestep_schedule(g, ts, m=1.0)
        S.emit_schedule_xml(sched, os.path.join(d, "ts.xml"))
        files.append("ts.xml")
        meta.update(l_max=l_max, U=[float(u) for u in ts.U],
                    total_utilization=ts.total_utilization, Q=sched.Q,
                    n_ops=len(sched.instructions))
    else:
        target = g
        comms = None
        if h is not None:
            target, mp = G.augment_host_bottleneck(g, h)
            G.save_graph(target, os.path.join(d, "aug_graph.json"))
            files.append("aug_graph.json")
            comms = M.all_to_all_commodities(mp.host)
        sol = M.mcf_decomposed(target, comms, workers=workers)
        meta["t_decomposed_s"] = time.time() - t0
        meta["F"] = sol.F
        t1 = time.time()
        wps = P.extract_widest_paths(target, _IndexedFlows(sol))
        meta["t_extract_s"] = time.time() - t1
        P.save_routes(wps, os.path.join(d, "wps.json"))
        files.append("wps.json")
        max_load, _ = P.eval_link_load(target, wps)
        meta["max_link_load"] = max_load
        with warnings.catch_warnings(record=True) as rec:
            warnings.simplefilter("always")
            routes, sched = S.compile_path_schedule(target, wps, m=1.0)
        meta["compile_warnings"] = [str(w.message) for w in rec]
        S.emit_schedule_xml(sched, os.path.join(d, "path.xml"))
        with open(os.path.join(d, "path.xml.routes.json"), "w") as fh:
            json.dump({"routes": routes}, fh, indent=1)
            fh.write("\n")
        files += ["path.xml", "path.xml.routes.json"]
        npaths = {}
        for plist in wps.paths.values():
            npaths[len(plist)] = npaths.get(len(plist), 0) + 1
        meta.update(Q=sched.Q, n_routes=len(routes),
                    n_instructions=len(sched.instructions),
                    paths_per_commodity=npaths)
    meta["t_total_s"] = time.time() - t0
    with open(os.path.join(d, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
        fh.write("\n")
    files.append("meta.json")
    _finish(d, files)
    print(f"[{name}] done in {meta['t_total_s']:.1f}s: "
          + json.dumps({k: meta.get(k) for k in ("F", "Q", "n_routes", "n_ops")}),
          flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--workers", type=int, default=8)
    a = ap.parse_args(argv)
    names = list(CONFIGS) if a.configs == ["all"] else a.configs
    for n in names:
        gen(n, a.workers)


if __name__ == "__main__":
    main()
