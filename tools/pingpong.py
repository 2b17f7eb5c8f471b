"""Cross-GPU flag latency microbenchmark (diagnostic).

Two processes, one CTA each: rank 0 stores a flag into rank 1's memory
(st.release.sys through the IPC mapping), rank 1 spins (ld.acquire.sys) and
answers into rank 0's memory; K round trips timed with %globaltimer.  Gives
the floor for one cross-GPU dependency hop of a2a_exec_kernel.
Built on the fly with torch.utils.cpp_extension.load_inline (diagnostic only).
"""
from __future__ import annotations

import os
import sys

import torch
import torch.distributed as dist

SRC = r"""
#include <cstdint>
__global__ void pp(uint32_t* mine, uint32_t* peer, int rank, int iters, unsigned long long* out) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    if (rank == 0) {
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer), "r"(i) : "memory");
      uint32_t v;
      do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory"); } while (v < (uint32_t)i);
    } else {
      uint32_t v;
      do { asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory"); } while (v < (uint32_t)i);
      asm volatile("st.release.sys.global.u32 [%0], %1;" :: "l"(peer), "r"(i) : "memory");
    }
  }
  unsigned long long t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = t1 - t0;
}
void launch(int64_t mine, int64_t peer, int rank, int iters, int64_t out) {
  pp<<<1, 1>>>((uint32_t*)mine, (uint32_t*)peer, rank, iters, (unsigned long long*)out);
}
"""


def main():
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    from torch.utils.cpp_extension import load_inline
    mod = load_inline("pp_ext", cpp_sources="void launch(int64_t, int64_t, int, int, int64_t);",
                      cuda_sources=SRC, functions=["launch"],
                      extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a"],
                      verbose=False)
    import ctypes
    cudart = ctypes.CDLL("libcudart.so") if False else None  # noqa: F841
    buf = torch.zeros(1024, dtype=torch.int32, device="cuda")
    # exchange IPC handles through torch's storage sharing helpers
    h = buf.untyped_storage()._share_cuda_()
    hs = [None, None]
    dist.all_gather_object(hs, h)
    other = hs[1 - rank]
    peer_storage = torch.UntypedStorage._new_shared_cuda(*other)
    peer = torch.empty(0, dtype=torch.int32, device=peer_storage.device).set_(peer_storage)
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    iters = 1000
    dist.barrier()
    mod.launch(buf.data_ptr(), peer.data_ptr(), rank, iters, out.data_ptr())
    torch.cuda.synchronize()
    ns = out.item()
    if rank == 0:
        print(f"round trip {ns / iters / 1e3:.3f} us (one way ~{ns / iters / 2e3:.3f} us) over {iters}")
    dist.barrier()


if __name__ == "__main__":
    main()
