"""NVLink SM-driven bandwidth: push (stores into peer memory) vs pull (loads
from peer memory), one direction and both directions at once, TMA bulk copies
(global -> smem -> global) and 128-bit LSU copies.  One process, two GPUs.

  python tools/nvlink_pull_probe.py        # prints one JSON line

Each variant launches one kernel per GPU (148 CTAs unless noted) that moves `bytes` through
a per-CTA slice; push: src local, dst peer; pull: src peer, dst local.
"""
from __future__ import annotations

import json
import os

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <cuda_runtime.h>
#include <cstdint>
#include <torch/extension.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int CH>
__global__ void __launch_bounds__(32, 1) tma_copy(char* dst, const char* src, long long n) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bars[S];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < S; ++i)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long long per = (n / gridDim.x) & ~(long long)(CH - 1);
  const long long lo = per * blockIdx.x, hi = lo + per;
  long long nl = 0, ns = 0;
  const long long nch = (hi - lo) / CH;
  auto issue = [&](long long k) {
    const int st = (int)(k % S);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[st])), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(sm + (size_t)st * CH)), "l"(src + lo + k * CH), "r"(CH), "r"(smem_u32(&bars[st])) : "memory");
  };
  while (nl < nch && nl < S - 1) issue(nl++);   // stage (k % S) is reused by chunk k + S
  while (ns < nch) {
    const int st = (int)(ns % S);
    const uint32_t par = (uint32_t)((ns / S) & 1);
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
                 ::"r"(smem_u32(&bars[st])), "r"(par) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + lo + ns * CH), "r"(smem_u32(sm + (size_t)st * CH)), "r"(CH) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++ns;
    if (nl < nch) {   // chunk nl = ns + S - 2 reuses the stage of chunk ns - 2: its store has read smem
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(nl++);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(1024, 1) lsu_copy(int4* dst, const int4* src, long long n16) {
  const long long per = n16 / gridDim.x, lo = per * blockIdx.x;
  for (long long i = threadIdx.x; i < per; i += 4 * blockDim.x) {
    int4 r[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) if (i + j * blockDim.x < per) r[j] = src[lo + i + j * blockDim.x];
#pragma unroll
    for (int j = 0; j < 4; ++j) if (i + j * blockDim.x < per) dst[lo + i + j * blockDim.x] = r[j];
  }
}

void enable_peer(int64_t dev, int64_t peer) {
  cudaSetDevice((int)dev);
  if (cudaDeviceEnablePeerAccess((int)peer, 0) != cudaSuccess) cudaGetLastError();
}

void launch(torch::Tensor dst, torch::Tensor src, int64_t dev, int64_t engine, int64_t stream, int64_t ctas) {
  cudaSetDevice((int)dev);
  cudaStream_t s = (cudaStream_t)stream;
  const long long n = src.numel();
  if (engine == 1) {
    constexpr int S = 6, CH = 32768;
    cudaFuncSetAttribute(tma_copy<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH);
    tma_copy<S, CH><<<(int)ctas, 32, S * CH, s>>>((char*)dst.data_ptr(), (const char*)src.data_ptr(), n);
  } else {
    lsu_copy<<<(int)ctas, 1024, 0, s>>>((int4*)dst.data_ptr(), (const int4*)src.data_ptr(), n / 16);
  }
}
"""

CPP = ("void launch(torch::Tensor dst, torch::Tensor src, int64_t dev, int64_t engine, int64_t stream, int64_t ctas);\n"
       "void enable_peer(int64_t dev, int64_t peer);")


def main():
    mod = load_inline("nvlink_pull_probe", cpp_sources=CPP, cuda_sources=SRC, functions=["launch", "enable_peer"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                      build_directory=os.environ.get("PROBE_BUILD", None), verbose=False)
    n = 1 << 30
    buf = {d: (torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}"),
               torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}")) for d in (0, 1)}
    mod.enable_peer(0, 1)
    mod.enable_peer(1, 0)
    streams = {d: torch.cuda.Stream(d) for d in (0, 1)}
    out = {}

    def run(kind, engine, both, ctas=148):
        # kind push: GPU d copies its own src -> peer dst; pull: peer src -> own dst
        def once():
            for d in ((0, 1) if both else (0,)):
                q = 1 - d
                if kind == "push":
                    dst, src = buf[q][1], buf[d][0]
                else:
                    dst, src = buf[d][1], buf[q][0]
                mod.launch(dst, src, d, engine, streams[d].cuda_stream, ctas)
        once()
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ts = []
        for _ in range(5):
            e0 = [torch.cuda.Event(enable_timing=True) for _ in (0, 1)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in (0, 1)]
            for d in (0, 1):
                e0[d].record(streams[d])
            once()
            for d in (0, 1):
                e1[d].record(streams[d])
            for d in (0, 1):
                torch.cuda.synchronize(d)
            ts.append(max(e0[d].elapsed_time(e1[d]) for d in ((0, 1) if both else (0,))))
        t = sorted(ts)[len(ts) // 2] / 1e3
        return round(n / t / 1e9, 1)

    for engine, en in ((1, "tma"), (0, "lsu")):
        for kind in ("push", "pull"):
            out[f"{en}_{kind}_oneway_gbs"] = run(kind, engine, False)
            out[f"{en}_{kind}_bidir_gbs_per_direction"] = run(kind, engine, True)
    for ctas in (16, 32, 48, 74, 111):   # how many pushing SMs saturate NVLink
        out[f"tma_push_bidir_{ctas}ctas_gbs_per_direction"] = run("push", 1, True, ctas)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
