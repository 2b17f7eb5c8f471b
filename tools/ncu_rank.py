"""One rank of a G-GPU all-to-all for ncu captures of the multi-GPU kernel
(NVLink tx/rx + DRAM bytes of one GPU).

ncu serialises the kernels it profiles (also across processes), so a
multi-GPU execute cannot be profiled on every rank at once: each GPU's kernel
waits on its peers' flags.  Here every rank is its own process (no torchrun;
CUDA-IPC arena handles are exchanged through files in --dir) and only ONE rank
runs under ncu with a single-pass metric set, its profiled launch running
concurrently with the peers' plain launches of the same all-to-all.  The
gpurun ncu shim first runs the profiled command once without ncu; the peers
therefore run twice (--phase plain --optional, then --phase ncu) and rendezvous
only with the same phase (the profiled rank's phase comes from the ncu
injection variable).

  python tools/ncu_rank.py --rank 1 --world 2 --phase plain --optional && \
      python tools/ncu_rank.py --rank 1 --world 2 --phase ncu &
  ncu --metrics ... -k regex:a2a -s 3 -c 1 python tools/ncu_rank.py --rank 0 --world 2
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _wait_files(paths, timeout=150.0, optional=False):
    t0 = time.time()
    while not all(os.path.exists(p) for p in paths):
        if time.time() - t0 > timeout:
            if optional:
                return False
            raise SystemExit(f"peer files missing after {timeout}s: {paths}")
        time.sleep(0.05)
    return True


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
    ap.add_argument("--phase", default=None, help="plain | ncu (default: from the ncu injection env)")
    ap.add_argument("--optional", action="store_true",
                    help="exit 0 if the peers of this phase never show up (no ncu shim pre-run)")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    phase = a.phase or ("ncu" if any(k.startswith(("CUDA_INJECTION64", "NV_NSIGHT", "NV_COMPUTE_PROFILER"))
                                     for k in os.environ) else "plain")
    os.makedirs(a.dir, exist_ok=True)
    G, r = a.world, a.rank
    torch.cuda.set_device(r)
    art = load_artifact(a.config)
    plan = bench.make_plan(art, a.m, G, "optimized", a.schedule)
    plan.bind(r, device=r)
    plan.set_timeout(60.0)      # the profiled launch starts seconds late (ncu set-up)
    _put(os.path.join(a.dir, f"{phase}_h{r}"), plan.export_handle())
    hs = [os.path.join(a.dir, f"{phase}_h{g}") for g in range(G)]
    if not _wait_files(hs, timeout=90.0 if a.optional else 150.0, optional=a.optional):
        plan.close()
        print(f"rank {r} ({phase}): no peers of this phase, skipped", flush=True)
        return
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
