"""Summarise sweep / bench JSON lines into a markdown table.

  python tools/report.py profiles/r01_final_scaling_G124.jsonl [more.jsonl ...]
"""
from __future__ import annotations

import json
import sys


def rows(paths):
    for p in paths:
        with open(p) as fh:
            for line in fh:
                line = line.strip()
                if line.startswith("{"):
                    yield p, json.loads(line)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    print("| config | m | GPUs | ms / all-to-all | algBW/GPU GB/s | bound frac | roofline frac (bound) "
          "| NCCL algBW/GPU | ours / NCCL | recv ok |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for _, r in rows(argv):
        if "skipped" in r:
            print(f"| {r['config']} | {r['m_bytes']} | {r['n_gpus']} | skipped: {r['skipped']} "
                  "| | | | | | |")
            continue
        n = r.get("nccl") or {}
        ratio = (f"{r['algbw_per_gpu_gbs'] / n['per_gpu']:.2f}" if n.get("per_gpu") else "")
        m = r["m_bytes"]
        ms = f"{m >> 20} MiB" if m >= 1 << 20 else f"{m >> 10} KiB"
        roof = r["roofline"]
        print(f"| {r['config']} | {ms} | {r['n_gpus']} | {r['ms']:.4f} | {r['algbw_per_gpu_gbs']:.1f} "
              f"| {r['bound_frac']:.3f} | {roof['frac']:.3f} ({roof['bound']}) "
              f"| {n.get('per_gpu', '')} | {ratio} | {r['recv_ok']} |")


if __name__ == "__main__":
    main()
