"""Launch overhead as bench.py times it: L2 flush (512 MiB memset), then an
event, one kernel, an event.  Empty kernels of the executor's shapes (148 x
1024 threads cooperative, 16 x 1024 plain) against the LL all-to-all of the
hypercube at 4 KiB on one GPU; back-to-back too.  One JSON line."""
from __future__ import annotations

import json
import os
import sys

import torch
from torch.utils.cpp_extension import load_inline

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SRC = r"""
#include <cuda_runtime.h>
#include <torch/extension.h>
__global__ void __launch_bounds__(1024, 1) empty_kernel(int* p) { if (threadIdx.x == 0 && blockIdx.x == 0 && p) p[0] = 1; }
void launch(int64_t ctas, int64_t coop, int64_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ctas); cfg.blockDim = dim3(1024); cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeCooperative; attr[0].val.cooperative = 1;
  cfg.attrs = attr; cfg.numAttrs = coop ? 1 : 0;
  int* p = nullptr;
  void* args[] = {&p};
  cudaLaunchKernelExC(&cfg, (const void*)empty_kernel, args);
}
"""


def main():
    mod = load_inline("launch_probe", cpp_sources="void launch(int64_t ctas, int64_t coop, int64_t stream);",
                      cuda_sources=SRC, functions=["launch"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"])
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    out = {}

    def timed(fn, flushing, reps=50):
        ts = []
        for _ in range(reps + 5):
            if flushing:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        v = sorted(x.elapsed_time(y) * 1e3 for x, y in ts[5:])
        return round(v[len(v) // 2], 2)

    for flushing in (True, False):
        tag = "flushed" if flushing else "back_to_back"
        out[f"empty_148x1024_coop_{tag}_us"] = timed(lambda: mod.launch(148, 1, st.cuda_stream), flushing)
        out[f"empty_16x1024_plain_{tag}_us"] = timed(lambda: mod.launch(16, 0, st.cuda_stream), flushing)
    import bench
    from paper_2309_13541_b200.artifacts import load_artifact
    a = load_artifact("hypercube3")
    for spec in ("ll", "ll@16", "ll128"):
        plan = bench.make_plan(a, 4096, 1, "optimized", spec)
        plan.bind(0, num_ctas=bench.spec_ctas(spec)[1])
        s = torch.zeros((8, 8, 4096), dtype=torch.uint8, device="cuda")
        r = torch.zeros_like(s)
        for flushing in (True, False):
            tag = "flushed" if flushing else "back_to_back"
            out[f"a2a_{spec}_4KiB_{tag}_us"] = timed(lambda: plan.execute(s, r, stream=st), flushing)
        plan.sync()
        plan.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
