"""One GPU: a few executes of one (config, m, execution schedule) plan, for
ncu captures of the executor kernel (`ncu -k regex:a2a -s <warmup> -c 1`).

  python tools/ncu_one.py --config gk8_2 --m 16777216 --schedule mix:1048576
"""
from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gk8_2")
    ap.add_argument("--m", type=int, default=16 << 20)
    ap.add_argument("--schedule", default="mix:1048576")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--copy-self", action="store_true")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    art = load_artifact(a.config)
    n = art.g.n
    plan = bench.make_plan(art, a.m, 1, "optimized", a.schedule, copy_self=a.copy_self)
    plan.bind(0, num_ctas=bench.spec_ctas(a.schedule)[1])
    g = torch.Generator(device="cuda").manual_seed(5)
    send = torch.randint(0, 256, (n, n, a.m), dtype=torch.uint8, device="cuda", generator=g)
    recv = torch.zeros_like(send)
    for _ in range(a.warmup + 1):     # the last launch is the one to profile
        plan.execute(send, recv)
        plan.sync()
    want = send.transpose(0, 1)
    off = ~torch.eye(n, dtype=torch.bool, device="cuda")
    ok = bool(torch.equal(recv[off], want[off]))
    plan.close()
    print(f"{a.config} m={a.m} {a.schedule}: recv ok={ok}", flush=True)
    if not ok:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
