"""Generate golden vectors from the UNMODIFIED reference (build container only).

Imports ``a2aflow`` from the read-only ``/root/reference/pkg/src`` and records,
for every frozen artifact and for deterministic corruptions of a few of them,
what the reference executor ``replay_timestep_schedule``
(pkg/src/a2aflow/evaluate.py:56-127) answers: the modelled T (exact float
repr) for several (m, b, sync) triples, or the exact EvalError text.  The
reference reads the schedules through its own ``parse_schedule_xml``
(src/schedule.py:349) and graphs through ``load_graph`` (src/graphs.py:562);
hop-indexed schedules come from this repo's lowering (the reference has none,
SURVEY.md finding 2) and are written to a temp XML first so the reference
parses them itself.

Also recorded: the reference's fluid per-link loads for the path configs
(``eval_link_load``, src/paths.py:535-553) — the MCF link loads the executor's
per-link bytes are compared against.

Output: tests/golden/golden.json (committed).  Run:
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import copy
import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from a2aflow import evaluate as RE       # noqa: E402
from a2aflow import graphs as RG         # noqa: E402
from a2aflow import paths as RP          # noqa: E402
from a2aflow import schedule as RS       # noqa: E402

from paper_2309_13541_b200.artifacts import (ARTIFACT_DIR, _find,  # noqa: E402
                                             list_artifacts, load_artifact)
from paper_2309_13541_b200.schedule import (Instruction,  # noqa: E402
                                            emit_schedule_xml)

PARAMS = [(1.0, 1.0, 0.0), (1048576.0, 1.0, 0.0), (16777216.0, 2.0, 0.25), (3.0, 0.5, 1.5)]


def plain(path):
    """The reference readers take plain files; inflate .gz artifacts to /tmp."""
    if not path.endswith(".gz"):
        return path
    import gzip
    fd, out = tempfile.mkstemp(suffix=os.path.basename(path)[:-3])
    with gzip.open(path, "rb") as src, os.fdopen(fd, "wb") as dst:
        dst.write(src.read())
    return out


def ref_sched(sched):
    """Round-trip through XML so the reference parses it with its own reader."""
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "s.xml")
        emit_schedule_xml(sched, p)
        return RS.parse_schedule_xml(p)


def ref_replay(g, sched, m, b, sync):
    try:
        T, ok = RE.replay_timestep_schedule(g, sched, m=m, b=b, sync_latency=sync)
        return {"T": repr(T), "ok": ok}
    except RE.EvalError as ex:
        return {"error": str(ex)}


def corruptions(sched):
    """Deterministic corrupted variants, each as (label, edit, instructions).

    Edits mirror the reference's own negative tests
    (tests/test_evaluate.py:39-59): drop / append instructions."""
    ins = list(sched.instructions)
    out = []
    multi = [i for i, x in enumerate(ins) if x.t == 0 and x.dst != x.d]
    if multi:
        k = multi[0]
        out.append(("drop_first_hop_of_forwarded_shard", {"drop": [k]},
                    ins[:k] + ins[k + 1:]))
    out.append(("append_non_edge", {"append": [[0, 0, 0, 0, 1, 0, 1]]}, None))
    last = [i for i, x in enumerate(ins) if x.dst == x.d]
    k = last[-1]
    out.append(("drop_final_hop", {"drop": [k]}, ins[:k] + ins[k + 1:]))
    x = ins[k]
    out.append(("duplicate_final_hop", {"append": [[x.t, x.src, x.dst, x.s, x.d, x.c0, x.c1]]}, None))
    f = ins[0]
    out.append(("chunk_beyond_Q", {"append": [[f.t, f.src, f.dst, f.s, f.d, sched.Q, sched.Q + 1]]}, None))
    out.append(("step_beyond_nsteps_ignored",
                {"append": [[sched.nsteps + 3, f.src, f.dst, f.s, f.d, f.c0, f.c1]]}, None))
    out.append(("empty_range_noop", {"append": [[0, f.src, f.dst, f.s, f.d, 0, 0]]}, None))
    out.append(("self_shard_send", {"append": [[0, f.src, f.dst, f.src, f.src, 0, 1]]}, None))
    return out


def apply_edit(sched, edit):
    s = copy.deepcopy(sched)
    drop = set(edit.get("drop", []))
    s.instructions = [x for i, x in enumerate(s.instructions) if i not in drop]
    for a in edit.get("append", []):
        s.instructions.append(RS.Instruction(*a))
    return s


def main(argv=None):
    """make_golden.py [CONFIG ...]: (re)generate the given configs (default all)
    and merge them into golden.json.  Configs with > 100k hop-ops replay only
    the first (m, b, sync) triple (the reference replay takes minutes there)."""
    argv = sys.argv[1:] if argv is None else argv
    gpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    out = {"params": PARAMS, "configs": {}}
    if argv and os.path.exists(gpath):
        with open(gpath) as fh:
            out = json.load(fh)
    for name in (argv or list_artifacts()):
        art = load_artifact(name)
        d = os.path.join(ARTIFACT_DIR, name)
        g = RG.load_graph(plain(_find(d, "graph.json")))
        sched = ref_sched(art.sched)
        rec = {"n": g.n, "nsteps": sched.nsteps, "Q": sched.Q,
               "n_ops": len(sched.instructions),
               "replay": [ref_replay(g, sched, *p)
                          for p in (PARAMS if len(sched.instructions) <= 100000 else PARAMS[:1])]}
        # per-(t, edge) chunk counts straight from the reference objects
        lc = {}
        for x in sched.instructions:
            k = f"{x.t},{g.edge_index[(x.src, x.dst)]}"
            lc[k] = lc.get(k, 0) + (x.c1 - x.c0)
        rec["link_chunks"] = lc
        if art.meta["kind"] == "path":
            target = g
            wps = RP.load_routes(plain(_find(d, "wps.json")))
            if art.meta.get("host_capacity") is not None:
                target = RG.load_graph(plain(_find(d, "aug_graph.json")))
            max_load, loads = RP.eval_link_load(target, wps)
            rec["fluid_max_load"] = repr(max_load)
            if target is g:
                rec["fluid_link_load"] = [repr(float(x)) for x in loads]
            else:
                # physical link (u,v) == augmented nic_out_u -> nic_in_v
                phys = []
                for u, v, _ in g.edges:
                    phys.append(repr(float(loads[target.edge_index[(3 * u + 2, 3 * v + 1)]])))
                rec["fluid_link_load"] = phys
        if name in ("torus2x4", "gk8_2", "ts_ring3", "ts_hypercube3", "torus2x4_h2"):
            cs = []
            for label, edit, _ in corruptions(sched):
                cs.append({"label": label, "edit": edit,
                           "replay": ref_replay(g, apply_edit(sched, edit), 1.0, 1.0, 0.0)})
            rec["corruptions"] = cs
        out["configs"][name] = rec
        print(name, rec["replay"][0], flush=True)
    with open(gpath, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
        fh.write("\n")


if __name__ == "__main__":
    main()
