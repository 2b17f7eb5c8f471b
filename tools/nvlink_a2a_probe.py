"""NVLink ceiling of an all-to-all-shaped push pattern, one process, G GPUs.

The executor's multi-GPU roofline is NVLink bytes of the busiest GPU per
direction.  tools/nvlink_pull_probe.py measures one peer; here every GPU
pushes to SEVERAL peers at once with the same TMA bulk-copy loop, CTAs split
over the peers in proportion to the bytes, as an all-to-all does:

  * uniform: every GPU pushes B bytes to each of its G-1 peers;
  * pairs:   a given GPU->GPU byte matrix (default: the GK(8,2) 16 MiB
             optimised-placement matrix at 4 GPUs from the frozen schedule);
  * with_hbm: the same plus a concurrent local HBM copy on each GPU (the
             local hops of the schedule).

Also reads the NVML NVLink byte counters around each run (which fields the
driver supports) -- the bench's live NVLink traffic evidence.

  python tools/nvlink_a2a_probe.py [--gpus 4]      # one JSON line
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch
from torch.utils.cpp_extension import load_inline

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from nvlink_pull_probe import SRC  # noqa: E402  (same TMA push loop)

CPP = ("void launch(torch::Tensor dst, torch::Tensor src, int64_t dev, int64_t engine, int64_t stream, int64_t ctas);\n"
       "void enable_peer(int64_t dev, int64_t peer);")


def nvml_fields(G):
    """{field name: [per GPU value]} for the NVLink byte counters NVML serves."""
    try:
        import pynvml as n
        n.nvmlInit()
    except Exception as ex:  # noqa: BLE001
        return {"error": repr(ex)}
    out = {}
    for g in range(G):
        pr = torch.cuda.get_device_properties(g)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        h = n.nvmlDeviceGetHandleByPciBusId(bus.encode())
        for name, fid in (("data_tx", 138), ("data_rx", 139), ("raw_tx", 140), ("raw_rx", 141),
                          ("xmit_bytes", 202), ("rcv_bytes", 204)):
            for scope, label in ((0xFFFFFFFF, "all"), (0, "l0"), (1, "l1")):
                key = f"{name}_{label}"
                try:
                    v = n.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
                    val = int(v.value.ullVal) if v.nvmlReturn == 0 else f"ret{v.nvmlReturn}"
                except Exception as ex:  # noqa: BLE001
                    val = repr(ex)[:60]
                out.setdefault(key, []).append(val)
        try:   # per-link utilization counters (older API)
            c = n.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0)
            out.setdefault("util_counter_l0_c0", []).append([int(c[0]), int(c[1])])
        except Exception as ex:  # noqa: BLE001
            out.setdefault("util_counter_l0_c0", []).append(repr(ex)[:60])
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--mib", type=int, default=512, help="bytes per (src, dst) pair, uniform case")
    a = ap.parse_args()
    G = a.gpus
    mod = load_inline("nvlink_pull_probe", cpp_sources=CPP, cuda_sources=SRC,
                      functions=["launch", "enable_peer"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                      build_directory=os.environ.get("PROBE_BUILD", None), verbose=False)
    for d in range(G):
        for q in range(G):
            if d != q:
                mod.enable_peer(d, q)
    B = a.mib << 20
    # per GPU: one src buffer per peer, one landing buffer per peer; local copy buffers
    src = {d: torch.empty(G * B, dtype=torch.uint8, device=f"cuda:{d}") for d in range(G)}
    dst = {d: torch.empty(G * B, dtype=torch.uint8, device=f"cuda:{d}") for d in range(G)}
    hb = {d: (torch.empty(4 * B, dtype=torch.uint8, device=f"cuda:{d}"),
              torch.empty(4 * B, dtype=torch.uint8, device=f"cuda:{d}")) for d in range(G)}
    streams = {d: [torch.cuda.Stream(d) for _ in range(G + 1)] for d in range(G)}

    def run(pairs, hbm_bytes=0, ctas_total=148, reps=5):
        """pairs[d][q] bytes d pushes to q; CTAs of GPU d split over its peers by bytes
        (one kernel per peer on its own stream, concurrently)."""
        def once():
            for d in range(G):
                tot = sum(pairs[d][q] for q in range(G) if q != d) + (hbm_bytes // 8 if hbm_bytes else 0)
                for q in range(G):
                    if q == d or pairs[d][q] == 0:
                        continue
                    c = max(1, round(ctas_total * pairs[d][q] / max(tot, 1)))
                    n = pairs[d][q]
                    mod.launch(dst[q][d * B: d * B + n], src[d][q * B: q * B + n], d, 1,
                               streams[d][q].cuda_stream, c)
                if hbm_bytes:
                    c = max(1, round(ctas_total * (hbm_bytes // 8) / max(tot, 1)))
                    mod.launch(hb[d][1][:hbm_bytes], hb[d][0][:hbm_bytes], d, 1,
                               streams[d][G].cuda_stream, c)
        once()
        for d in range(G):
            torch.cuda.synchronize(d)
        f0 = nvml_fields(G)
        ts = []
        for _ in range(reps):
            e0 = {d: torch.cuda.Event(enable_timing=True) for d in range(G)}
            e1 = {d: torch.cuda.Event(enable_timing=True) for d in range(G)}
            for d in range(G):
                e0[d].record(streams[d][0])
                for s in streams[d][1:]:
                    s.wait_stream(streams[d][0])
            once()
            for d in range(G):
                for s in streams[d][1:]:
                    streams[d][0].wait_stream(s)
                e1[d].record(streams[d][0])
            for d in range(G):
                torch.cuda.synchronize(d)
            ts.append(max(e0[d].elapsed_time(e1[d]) for d in range(G)) / 1e3)
        import time
        time.sleep(0.5)
        f1 = nvml_fields(G)
        t = sorted(ts)[len(ts) // 2]
        eg = [sum(pairs[d][q] for q in range(G) if q != d) for d in range(G)]
        ing = [sum(pairs[q][d] for q in range(G) if q != d) for d in range(G)]
        busiest = max(max(eg), max(ing))
        delta = {}
        for k in f0:
            if isinstance(f0[k], list):
                delta[k] = [(b - a) if isinstance(a, int) and isinstance(b, int) else b
                            for a, b in zip(f0[k], f1[k])]
        return {"ms": round(t * 1e3, 4), "busiest_gbs_per_direction": round(busiest / t / 1e9, 1),
                "egress_mib": [x >> 20 for x in eg], "ingress_mib": [x >> 20 for x in ing],
                "nvml_delta_over_run": delta, "runs_counted": reps + 0}

    out = {"gpus": G}
    uni = [[0 if d == q else B for q in range(G)] for d in range(G)]
    out["uniform"] = run(uni)
    out["uniform_with_hbm"] = run(uni, hbm_bytes=2 * B)
    for c in (74, 296):
        out[f"uniform_{c}ctas"] = run(uni, ctas_total=c)
    if G == 4:
        M = 1 << 20   # GK(8,2) 16 MiB, optimised placement [0,1,2,0,3,1,2,3]: MiB per pair
        gk = [[0, 144, 144, 112], [0, 0, 0, 288], [288, 0, 0, 0], [112, 144, 144, 0]]
        out["gk8_2_pairs"] = run([[x * M for x in r] for r in gk])
        out["gk8_2_pairs_with_hbm"] = run([[x * M for x in r] for r in gk], hbm_bytes=2 * B)
    if G >= 2:
        one = [[0] * G for _ in range(G)]
        one[0][1] = one[1][0] = B
        out["one_pair_bidir"] = run(one)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
