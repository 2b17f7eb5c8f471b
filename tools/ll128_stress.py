"""LL128 line-atomicity stress test (validation campaign for A2A_PROTO_LL128).

The LL128 transport stores each 128-byte line {120 payload bytes, 8-byte
epoch flag} as ONE warp instruction (8 lanes x 16 bytes, st.volatile.v2.u64)
and the reader loads the line the same way and trusts the payload when the
flag carries the epoch -- the protocol NCCL uses over NVLink.  It relies on a
warp's 128-byte line store reaching the reader as a unit.  This tool hammers
exactly that: producer warps write epochs of lines whose payload words are a
hash of (epoch, line, word); consumer warps poll the lines while they are
being written and check every payload word of every line whose flag matches.
A torn line (flag new, payload old) is counted.

  python tools/ll128_stress.py [--epochs 4000] [--lines 65536]   # one JSON line

Cases: remote (producer on GPU 0 stores over NVLink into GPU 1, consumer on
GPU 1) and local (producer and consumer CTAs on the same GPU).
"""
from __future__ import annotations

import argparse
import json
import os
import time

# kernels that wait on each other must be loaded before either runs (lazy
# module loading can block a launch until the running kernel finishes)
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <cuda_runtime.h>
#include <cstdint>
#include <torch/extension.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL; return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t word(uint64_t e, uint64_t line, int k) { return mix((e << 40) ^ (line << 4) ^ k); }
__device__ __forceinline__ void st16(uint64_t* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld16(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
constexpr uint64_t kTimeout = 10000000000ULL;   // 10 s: a stuck spin bails out (never a hang)
__device__ __forceinline__ unsigned long long ldv(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}

// lines: [2 parities][nl][16 u64]; done: consumer CTAs finished per epoch (cumulative)
__device__ void producer_body(uint64_t* lines, const unsigned long long* done, long long nl, int epochs,
                              int ncons, int bid, int nblk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j = lane & 7;
  __shared__ int s_abort;
  if (threadIdx.x == 0) s_abort = 0;
  for (int e = 1; e <= epochs; ++e) {
    if (e > 2) {  // parity buffer of epoch e-2 fully consumed
      if (threadIdx.x == 0) {
        const uint64_t t0 = gtime();
        while (ldv(done) < (unsigned long long)ncons * (e - 2)) {
          __nanosleep(100);
          if (gtime() - t0 > kTimeout) { s_abort = 1; break; }
        }
      }
      __syncthreads();
      if (s_abort) return;
    }
    uint64_t* buf = lines + (size_t)(e & 1) * nl * 16;
    for (long long L0 = ((long long)bid * nw + warp) * 4; L0 < nl; L0 += (long long)nblk * nw * 4) {
      const long long L = L0 + (lane >> 3);
      if (L >= nl) continue;
      const uint64_t a = word(e, L, 2 * j);
      const uint64_t b = j == 7 ? (uint64_t)e : word(e, L, 2 * j + 1);
      st16(buf + L * 16 + 2 * j, a, b);
    }
  }
}

__device__ void consumer_body(const uint64_t* lines, unsigned long long* done, unsigned long long* bad,
                              unsigned long long* checked, long long nl, int epochs, int bid, int nblk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j = lane & 7;
  unsigned long long nbad = 0, nchk = 0;
  if ((long long)bid * nw * 4 >= nl) return;   // no lines: not counted in `done`
  for (int e = 1; e <= epochs; ++e) {
    const uint64_t* buf = lines + (size_t)(e & 1) * nl * 16;
    for (long long L0 = ((long long)bid * nw + warp) * 4; L0 < nl; L0 += (long long)nblk * nw * 4) {
      const long long L = L0 + (lane >> 3);
      const bool live = L < nl;
      uint64_t a = 0, b = 0;
      const uint64_t t0 = gtime();
      for (;;) {
        if (gtime() - t0 > kTimeout) { atomicAdd(bad, 1ull << 40); return; }
        if (live) ld16(buf + L * 16 + 2 * j, a, b);
        const uint64_t flag = __shfl_sync(0xffffffffu, b, (lane & ~7) | 7);
        const bool ok = !live || flag == (uint64_t)e;
        if (__all_sync(0xffffffffu, ok)) break;
      }
      if (live) {
        bool good = a == word(e, L, 2 * j) && (j == 7 || b == word(e, L, 2 * j + 1));
        nbad += !good;
        nchk += 1;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) { __threadfence_system(); atomicAdd(done, 1ull); }
  }
  atomicAdd(bad, nbad);
  atomicAdd(checked, nchk);
}

__global__ void producer(uint64_t* lines, const unsigned long long* done, long long nl, int epochs, int ncons) {
  producer_body(lines, done, nl, epochs, ncons, blockIdx.x, gridDim.x);
}
__global__ void consumer(const uint64_t* lines, unsigned long long* done, unsigned long long* bad,
                         unsigned long long* checked, long long nl, int epochs) {
  consumer_body(lines, done, bad, checked, nl, epochs, blockIdx.x, gridDim.x);
}
// local case: one launch, CTAs [0, np) produce, the rest consume (co-resident by construction)
__global__ void both(uint64_t* lines, unsigned long long* done, unsigned long long* bad,
                     unsigned long long* checked, long long nl, int epochs, int np, int ncons) {
  if ((int)blockIdx.x < np) producer_body(lines, done, nl, epochs, ncons, blockIdx.x, np);
  else consumer_body(lines, done, bad, checked, nl, epochs, blockIdx.x - np, gridDim.x - np);
}
void run_both(torch::Tensor lines, torch::Tensor done, torch::Tensor bad, torch::Tensor chk,
              int64_t nl, int64_t epochs, int64_t np, int64_t nc, int64_t ncons, int64_t dev, int64_t stream) {
  cudaSetDevice((int)dev);
  both<<<(int)(np + nc), 256, 0, (cudaStream_t)stream>>>((uint64_t*)lines.data_ptr(),
      (unsigned long long*)done.data_ptr(), (unsigned long long*)bad.data_ptr(),
      (unsigned long long*)chk.data_ptr(), nl, (int)epochs, (int)np, (int)ncons);
}
void enable_peer(int64_t dev, int64_t peer) {
  cudaSetDevice((int)dev);
  if (cudaDeviceEnablePeerAccess((int)peer, 0) != cudaSuccess) cudaGetLastError();
}
void run_producer(torch::Tensor lines, torch::Tensor done, int64_t nl, int64_t epochs, int64_t ncons,
                  int64_t dev, int64_t ctas, int64_t stream) {
  cudaSetDevice((int)dev);
  producer<<<(int)ctas, 256, 0, (cudaStream_t)stream>>>((uint64_t*)lines.data_ptr(),
      (const unsigned long long*)done.data_ptr(), nl, (int)epochs, (int)ncons);
}
void run_consumer(torch::Tensor lines, torch::Tensor done, torch::Tensor bad, torch::Tensor chk,
                  int64_t nl, int64_t epochs, int64_t dev, int64_t ctas, int64_t stream) {
  cudaSetDevice((int)dev);
  consumer<<<(int)ctas, 256, 0, (cudaStream_t)stream>>>((const uint64_t*)lines.data_ptr(),
      (unsigned long long*)done.data_ptr(), (unsigned long long*)bad.data_ptr(),
      (unsigned long long*)chk.data_ptr(), nl, (int)epochs);
}
"""
CPP = ("void enable_peer(int64_t dev, int64_t peer);\n"
       "void run_both(torch::Tensor lines, torch::Tensor done, torch::Tensor bad, torch::Tensor chk, int64_t nl, int64_t epochs, int64_t np, int64_t nc, int64_t ncons, int64_t dev, int64_t stream);\n"
       "void run_producer(torch::Tensor lines, torch::Tensor done, int64_t nl, int64_t epochs, int64_t ncons, int64_t dev, int64_t ctas, int64_t stream);\n"
       "void run_consumer(torch::Tensor lines, torch::Tensor done, torch::Tensor bad, torch::Tensor chk, int64_t nl, int64_t epochs, int64_t dev, int64_t ctas, int64_t stream);")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=4000)
    ap.add_argument("--lines", type=int, default=65536)
    ap.add_argument("--local-only", action="store_true")
    a = ap.parse_args()
    mod = load_inline("ll128_stress", cpp_sources=CPP, cuda_sources=SRC,
                      functions=["enable_peer", "run_producer", "run_consumer", "run_both"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"],
                      verbose=False)
    out = {"epochs": a.epochs, "lines": a.lines}
    cases = [("local", 0, 0)]
    if torch.cuda.device_count() >= 2 and not a.local_only:
        mod.enable_peer(0, 1)
        mod.enable_peer(1, 0)
        cases.append(("remote", 0, 1))
    # warm-up: load both kernels on both devices before any pair runs concurrently
    for d in range(min(2, torch.cuda.device_count())):
        z = torch.zeros(64, dtype=torch.int64, device=f"cuda:{d}")
        st = torch.cuda.Stream(d)
        mod.run_consumer(z, z[:1], z[1:2], z[2:3], 0, 0, d, 1, st.cuda_stream)
        mod.run_producer(z, z[:1], 0, 0, 1, d, 1, st.cuda_stream)
        torch.cuda.synchronize(d)
    for name, pdev, cdev in cases:
        nl = a.lines
        lines = torch.zeros(2 * nl * 16, dtype=torch.int64, device=f"cuda:{cdev}")
        done = torch.zeros(1, dtype=torch.int64, device=f"cuda:{cdev}")
        bad = torch.zeros(1, dtype=torch.int64, device=f"cuda:{cdev}")
        chk = torch.zeros(1, dtype=torch.int64, device=f"cuda:{cdev}")
        # the zero fills above run on the default stream; the test streams do not
        # wait for it, so finish them first (a late fill would erase epoch-1 lines)
        torch.cuda.synchronize(pdev)
        torch.cuda.synchronize(cdev)
        sp, sc = torch.cuda.Stream(pdev), torch.cuda.Stream(cdev)
        pc, cc = (64, 64) if pdev == cdev else (132, 132)
        cc = min(cc, (nl + 31) // 32)             # consumer CTAs that own lines (8 warps x 4)
        t0 = time.time()
        if pdev == cdev:
            mod.run_both(lines, done, bad, chk, nl, a.epochs, pc, 64, cc, cdev, sc.cuda_stream)
        else:
            mod.run_consumer(lines, done, bad, chk, nl, a.epochs, cdev, cc, sc.cuda_stream)
            mod.run_producer(lines, done, nl, a.epochs, cc, pdev, pc, sp.cuda_stream)
        torch.cuda.synchronize(pdev)
        torch.cuda.synchronize(cdev)
        dt = time.time() - t0
        out[name] = {"torn_lines": int(bad.item()), "lines_checked": int(chk.item()),
                     "expected": a.epochs * nl, "seconds": round(dt, 2),
                     "line_gbs": round(a.epochs * nl * 128 / dt / 1e9, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
