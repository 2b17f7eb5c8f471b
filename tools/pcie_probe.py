"""PCIe probe for the e2e leg: pinned host <-> device copies of 0.94 GB (the
s != d shards of GK(8,2) at 16 MiB), H2D alone, D2H alone, and both at once,
with 1, 2 or 4 streams per direction.  One JSON line."""
from __future__ import annotations

import json

import torch


def main():
    n = 939524096
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}

    def run(h2d, d2h, k, reps=5):
        ss = [torch.cuda.Stream() for _ in range(2 * k)]
        ts = []
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for s in ss:
                s.wait_event(e0)
            step = n // k
            for i in range(k):
                if h2d:
                    with torch.cuda.stream(ss[i]):
                        d_in[i * step:(i + 1) * step].copy_(h_in[i * step:(i + 1) * step], non_blocking=True)
                if d2h:
                    with torch.cuda.stream(ss[k + i]):
                        h_out[i * step:(i + 1) * step].copy_(d_out[i * step:(i + 1) * step], non_blocking=True)
            cur = torch.cuda.current_stream()
            for s in ss:
                cur.wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = sorted(ts[1:])[len(ts[1:]) // 2]
        return round(n / t / 1e9, 1)

    for k in (1, 2, 4):
        out[f"h2d_k{k}"] = run(True, False, k)
        out[f"d2h_k{k}"] = run(False, True, k)
        out[f"both_k{k}_per_direction"] = run(True, True, k)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
