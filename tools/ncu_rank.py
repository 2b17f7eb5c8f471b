"""One rank of a G-GPU all-to-all for per-rank ncu captures (NVLink + DRAM bytes).

ncu serialises the kernels of the process it profiles, so a multi-GPU
execute cannot be profiled from one process (each GPU's kernel waits on its
peers' flags).  Here every rank is its own process, started by a shell loop
(no torchrun), each under its own ncu with a single-pass metric set; the
ranks exchange their CUDA-IPC arena handles through files in --dir.  The
gpurun ncu shim first runs the command once without ncu: both runs of a rank
rendezvous only with the same kind of run of their peers (file prefix
"plain" / "ncu", from the ncu injection variable).

  for r in 0 1; do ncu --metrics ... -k regex:a2a -s 3 -c 1 --csv --log-file out_$r.csv \
      python tools/ncu_rank.py --rank $r --world 2 & done; wait
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _wait_files(paths, timeout=120.0):
    t0 = time.time()
    while not all(os.path.exists(p) for p in paths):
        if time.time() - t0 > timeout:
            raise SystemExit(f"peer files missing after {timeout}s: {paths}")
        time.sleep(0.05)


def _put(path, data: bytes):
    tmp = path + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(data)
    os.replace(tmp, path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--config", default="gk8_2")
    ap.add_argument("--m", type=int, default=16 << 20)
    ap.add_argument("--schedule", default="spread:1048576")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dir", default="/tmp/a2a_ncu_rdv")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    phase = "ncu" if any(k.startswith(("CUDA_INJECTION64", "NV_NSIGHT", "NSYS_", "NV_COMPUTE_PROFILER"))
                         for k in os.environ) else "plain"
    os.makedirs(a.dir, exist_ok=True)
    G, r = a.world, a.rank
    torch.cuda.set_device(r)
    art = load_artifact(a.config)
    plan = bench.make_plan(art, a.m, G, "optimized", a.schedule)
    plan.bind(r, device=r)
    plan.set_timeout(5.0)
    _put(os.path.join(a.dir, f"{phase}_h{r}"), plan.export_handle())
    hs = [os.path.join(a.dir, f"{phase}_h{g}") for g in range(G)]
    _wait_files(hs)
    plan.import_handles([open(p, "rb").read() for p in hs])
    nodes = [v for v in range(art.g.n) if int(plan.placement[v]) == r]
    send = torch.randint(0, 256, (len(nodes), art.g.n, a.m), dtype=torch.uint8, device=f"cuda:{r}")
    recv = plan.recv_buffer()
    for _ in range(a.warmup + 1):      # the last one is the profiled launch (ncu -s warmup -c 1)
        plan.execute(send, recv)
        plan.sync()
    plan.close_peers()
    _put(os.path.join(a.dir, f"{phase}_done{r}"), b"1")
    _wait_files([os.path.join(a.dir, f"{phase}_done{g}") for g in range(G)])
    plan.close()
    print(f"rank {r} ({phase}) ok: {G} GPUs, {a.config} m={a.m} {a.schedule}", flush=True)


if __name__ == "__main__":
    main()
