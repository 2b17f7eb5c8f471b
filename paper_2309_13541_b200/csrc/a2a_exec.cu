// Device side of the executor: one persistent, cooperatively launched kernel
// per GPU and all-to-all.
//
// Per step t the kernel runs this GPU's copy items (hop-ops whose source
// virtual node lives here).  Each item is a contiguous byte range; hop 0 reads
// the caller's send buffer directly (pack fused), the last hop writes the
// destination's recv buffer directly (unpack fused), intermediate hops go
// through forwarding scratch.  Destinations on other GPUs are written with
// plain 128-bit stores through CUDA-IPC-mapped peer pointers (NVLink5 via
// NVSwitch).  The step's bytes are split into one contiguous range per CTA.
//
// Ordering (store-and-forward, reference evaluate.py:93-113: a chunk received
// at step t is forwarded at t+1 at the earliest) — exact producer dependencies,
// no step barrier (chunk-pipelined execution):
//   producer CTA c of GPU g, after its step-t byte range:
//       bar.sync; fence.sc.sys; st.release.sys flag_h[t][g][c] = epoch on every
//       GPU h it wrote to in step t
//   consumer CTA c' of GPU h, before its step-t' range: warp 0 polls
//       (ld.acquire.sys, one flag per lane, __all_sync) exactly the producer
//       CTAs that wrote the bytes its pieces read (host-computed from the static
//       work split: interval overlap of source ranges with earlier writes),
//       then fence + bar.sync.  Steps therefore overlap: a CTA starts step t+1
//       as soon as its own inputs exist, not when the whole GPU finished step t.
//   entry barrier (multi-GPU): every GPU announces the epoch to all peers
//       (relaxed store) and acquires theirs before storing into peer memory, so
//       a peer's buffers are never overwritten while its previous all-to-all is
//       still live.
//   exit (multi-GPU): CTA 0 polls every producer flag of this GPU, so kernel
//       completion implies this GPU's recv buffer is final.
// Every spin is bounded by a %globaltimer timeout and reports A2A_ERR_TIMEOUT.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "a2a_internal.h"

namespace a2a {

struct KParams {
  char* base[1 + 3 * A2A_MAX_GPUS];        // send | recv[G] | scratch[G] | LL landing[G]
  uint32_t* step_flags[A2A_MAX_GPUS];      // per GPU: [T'][G][nC] u32, slot (t, producer gpu, cta)
  uint32_t* entry_flags[A2A_MAX_GPUS];     // per GPU: [G] u32
  const DevPiece* pieces;                  // this GPU's pieces, ordered by (cta, step)
  const CtaStep* prog;                     // [nC][T'] per-CTA step programs
  const int32_t* wait_idx;                 // producer flag indices in own step_flags
  const int32_t* exit_idx;                 // every producer flag of this GPU (exit wait)
  int32_t n_exit;
  unsigned long long* counters;            // [T'][E]
  int32_t* err;
  int64_t timeout_ns;
  uint32_t* ctl;                           // [nC] last completed epoch of each CTA (device memory)
  int64_t ll_half[A2A_MAX_GPUS];           // LL landing region bytes per epoch parity
  int32_t G, rank, nC, T, E, count_links;
  int32_t ll;                              // A2A_PROTO_LL: cross-GPU bytes as LL lines
  int32_t ll128, smem_ll;                  // A2A_PROTO_LL128 lines; its per-warp gather smem
  int32_t tma_chunk, tma_stages;           // TMA engine: bytes per bulk copy, ring depth
  int32_t sync_mode;                       // a2a_plan_set_sync_mode bits (include/a2a_exec.h):
                                           // 0-5 publish/poll variants, 6 perturb, 7 no waits
  int32_t smem_prog, smem_batch, batch;    // dynamic smem offsets, pieces per staged batch
  unsigned long long* timeline;            // [nC][2T'+3] %globaltimer stamps (see read_timeline)
  // dynamic mode (a2a_dyn_kernel)
  const DevUnit* units;                    // this GPU's units in grab order
  const int32_t* unit_wait;                // global unit ids to acquire
  int32_t n_units, unit_base;              // this GPU's units; global id of its first
  int32_t n_remote, remote_ctas;           // remote queue = units [0, n_remote); CTAs starting on it
  int32_t pin_queues;                      // CTAs never switch queues
  unsigned long long* grab;                // per-GPU grab counters [2] (remote, local queue)
  // ready-queue mode (sched_mode 5): per GPU its queue control words (head,
  // tail, arrived), per-unit completion counters and queue slots (arena, peer-visible)
  unsigned long long* qctl[A2A_MAX_GPUS];
  unsigned long long* qdone[A2A_MAX_GPUS];
  unsigned long long* qslot[A2A_MAX_GPUS];
  int32_t ubase[A2A_MAX_GPUS + 1];         // global unit id range of every GPU
  int32_t n_init, n_into;                  // own units ready at start; units writing into this GPU
  // chain mode (sched_mode 7): task k = units [chain_begin[k], chain_begin[k+1])
  const int32_t* chain_begin;
  int32_t n_tasks;
  int32_t chain_discard;                   // sched_mode 8: discard the chain's dead scratch lines
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p, bool sys) {
  uint32_t v;
  if (sys)
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p, bool sys) {
  uint32_t v;
  if (sys)
    asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(uint32_t* p, uint32_t v, bool sys) {
  if (sys)
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_acq_rel_sys(unsigned long long* p, unsigned long long v) {
  unsigned long long r;
  asm volatile("atom.acq_rel.sys.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}
__device__ __forceinline__ unsigned long long atom_add_relaxed_sys(unsigned long long* p, unsigned long long v) {
  unsigned long long r;
  asm volatile("atom.relaxed.sys.global.add.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(v) : "memory");
  return r;
}
__device__ __forceinline__ void red_add_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel(bool sys) {
  if (sys)
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  else
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// Whole-CTA byte copy.  Fast path when src == dst (mod 16): byte head,
// 128-bit body with kUnroll loads in flight per thread, byte tail.
template <int kUnroll>
__device__ __forceinline__ void cta_copy(char* __restrict__ dst, const char* __restrict__ src,
                                         int64_t n) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if ((((uintptr_t)src ^ (uintptr_t)dst) & 15) != 0) {
    for (int64_t i = tid; i < n; i += nt) dst[i] = src[i];
    return;
  }
  int64_t head = (16 - ((uintptr_t)dst & 15)) & 15;
  if (head > n) head = n;
  if (tid < head) dst[tid] = src[tid];
  dst += head;
  src += head;
  n -= head;
  const int64_t nv = n >> 4;
  const int4* s4 = reinterpret_cast<const int4*>(src);
  int4* d4 = reinterpret_cast<int4*>(dst);
  int64_t i = tid;
  const int64_t stride = (int64_t)nt * kUnroll;
  for (; i + (int64_t)(kUnroll - 1) * nt < nv; i += stride) {
    int4 r[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) r[j] = ld_stream(s4 + i + (int64_t)j * nt);
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) st_stream(d4 + i + (int64_t)j * nt, r[j]);
  }
  for (; i < nv; i += nt) st_stream(d4 + i, ld_stream(s4 + i));
  const int64_t tail = n & 15;
  if (tid < tail) dst[nv * 16 + tid] = src[nv * 16 + tid];
}

// ---- LL transport (A2A_PROTO_LL) ----
// A 16-byte line {payload[0..4), epoch, payload[4..8), epoch}: each 8-byte half
// is stored and loaded as one unit, so a reader that sees the epoch in both
// halves holds the payload -- no fence, no separate flag (the LL protocol).
// LL offsets are payload addresses: payload byte x of a landing region lives
// in line x/8.
__device__ __forceinline__ uint64_t plain_load8(const char* __restrict__ s, int nb) {
  if (nb == 8 && ((uintptr_t)s & 7) == 0) return *reinterpret_cast<const uint64_t*>(s);
  uint64_t v = 0;
  for (int j = 0; j < nb; ++j) v |= (uint64_t)(uint8_t)s[j] << (8 * j);
  return v;
}
__device__ __forceinline__ void plain_store8(char* __restrict__ d, uint64_t v, int nb) {
  if (nb == 8 && ((uintptr_t)d & 7) == 0) {
    *reinterpret_cast<uint64_t*>(d) = v;
    return;
  }
  for (int j = 0; j < nb; ++j) d[j] = (char)((v >> (8 * j)) & 0xff);
}
__device__ __forceinline__ void ll_store(uint4* dst, uint64_t v, uint32_t epoch) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"((uint32_t)v),
               "r"(epoch), "r"((uint32_t)(v >> 32)), "r"(epoch)
               : "memory");
}
#ifndef A2A_LL_SPIN
#define A2A_LL_SPIN 32
#endif
constexpr uint32_t kLLSpin = A2A_LL_SPIN;
// Poll one line until both halves carry `epoch`.  Polls back off (up to
// ~0.5 us) so that CTAs waiting on large landing regions do not flood L2 with
// requests while the NVLink writes are arriving.  False on timeout / error.
__device__ __forceinline__ bool ll_poll(const uint4* line, uint32_t epoch, int64_t timeout_ns,
                                        int32_t* err, uint64_t* out) {
  uint32_t a, f0, b, f1, spins = 0, nap = 0;
  uint64_t t0 = 0;
  for (;;) {
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(f0), "=r"(b), "=r"(f1)
                 : "l"(line)
                 : "memory");
    if (f0 == epoch && f1 == epoch) {
      *out = (uint64_t)a | ((uint64_t)b << 32);
      return true;
    }
    if (++spins > kLLSpin) {   // hot polling first (small shards), then back off
      nap = nap ? min(2 * nap, 1024u) : 64u;
      __nanosleep(nap);
    }
    if ((spins & 255) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      if ((int64_t)(now - t0) > timeout_ns || *(volatile int32_t*)err != 0) return false;
    }
  }
}
// One LL-mode piece, all threads: thread k produces payload bytes [8k, 8k+8)
// -- gathered from plain memory or from the one or two source lines they span
// (polled) -- and stores them as one destination line (8-aligned payload
// address) or as plain bytes.  Plain sources: 4 lines in flight per thread.
__device__ __forceinline__ bool ll_piece(const char* sbase, char* dbase, const DevPiece& q,
                                         uint32_t epoch, int64_t timeout_ns, int32_t* err) {
  const bool sll = q.kind & kLLSrc, dll = q.kind & kLLDst;
  const int64_t n = q.nbytes, L = (n + 7) >> 3, nt = blockDim.x;
  const uint4* sl = reinterpret_cast<const uint4*>(sbase);
  uint4* dl = reinterpret_cast<uint4*>(dbase) + (q.dst_off >> 3);
  char* dp = dbase + q.dst_off;
  int64_t k = threadIdx.x;
  if (!sll) {
    const char* sp = sbase + q.src_off;
    constexpr int kU = 4;
    for (; k + (kU - 1) * nt < L; k += kU * nt) {
      uint64_t v[kU];
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int64_t b = (k + j * nt) << 3;
        v[j] = plain_load8(sp + b, (int)min((int64_t)8, n - b));
      }
#pragma unroll
      for (int j = 0; j < kU; ++j) {
        const int64_t b = (k + j * nt) << 3;
        if (dll) ll_store(dl + k + j * nt, v[j], epoch);
        else plain_store8(dp + b, v[j], (int)min((int64_t)8, n - b));
      }
    }
  }
  for (; k < L; k += nt) {
    const int64_t b = k << 3;
    const int nb = (int)min((int64_t)8, n - b);
    uint64_t v;
    if (sll) {
      const int64_t pa = q.src_off + b;
      const int sh = (int)(pa & 7);
      uint64_t x;
      if (!ll_poll(sl + (pa >> 3), epoch, timeout_ns, err, &x)) return false;
      v = x >> (8 * sh);
      if (sh && sh + nb > 8) {
        uint64_t y;
        if (!ll_poll(sl + (pa >> 3) + 1, epoch, timeout_ns, err, &y)) return false;
        v |= y << (64 - 8 * sh);
      }
    } else {
      v = plain_load8(sbase + q.src_off + b, nb);
    }
    if (dll) ll_store(dl + k, v, epoch);
    else plain_store8(dp + b, v, nb);
  }
  return true;
}

// ---- LL128 transport (A2A_PROTO_LL128) ----
// A 128-byte line = 120 payload bytes + the 8-byte epoch flag (bytes 120..127).
// A warp moves 4 lines per instruction: lane = 8 * line + seg, seg j holds line
// bytes [16j, 16j + 16) (seg 7: 8 payload bytes + the flag), each lane one
// ld/st.volatile.v2.u64.  A reader trusts a line whose flag carries the epoch:
// the whole line is one warp store (NCCL's LL128 protocol over NVLink; validated
// on this hardware by tools/ll128_stress.py).  Offsets are payload addresses:
// payload byte x of a landing region lives at byte 128 * (x / 120) + x % 120.
__device__ __forceinline__ void st16v(char* p, uint64_t a, uint64_t b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld16v(const char* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// Every lane of the warp: poll its segment of `line` (when `need`) until every
// needed line of the warp carries epoch E.  Hot polling first, then back off.
// False (all lanes) on timeout / device error.
__device__ __forceinline__ bool ll128_poll(const char* line, bool need, int j, uint64_t E,
                                           uint64_t& a, uint64_t& b, int64_t timeout_ns, int32_t* err) {
  const int lane = threadIdx.x & 31;
  uint32_t spins = 0, nap = 0;
  uint64_t t0 = 0;
  for (;;) {
    if (need) ld16v(line + 16 * j, a, b);
    const uint64_t f = __shfl_sync(0xffffffffu, b, lane | 7);
    if (__all_sync(0xffffffffu, !need || f == E)) return true;
    if (++spins > kLLSpin) {
      nap = nap ? min(2 * nap, 1024u) : 64u;
      __nanosleep(nap);
    }
    if ((spins & 255) == 0) {
      const uint64_t now = globaltimer();
      if (t0 == 0) t0 = now;
      const bool out = (int64_t)(now - t0) > timeout_ns || *(volatile int32_t*)err != 0;
      if (__any_sync(0xffffffffu, out)) return false;
    }
  }
}
__device__ __forceinline__ void ld16_plain(const char* s, int nb, uint64_t& a, uint64_t& b) {
  a = plain_load8(s, min(nb, 8));
  b = nb > 8 ? plain_load8(s + 8, nb - 8) : 0;
}
// One LL128 piece, all threads of the CTA (4 output lines per warp and turn).
// Sources: plain bytes (send), LL128 lines on a line boundary (a forwarded
// arrival: a verbatim line copy), or LL128 lines at any payload offset (the
// warp gathers the source window through shared memory `wsm`, 640 B per warp).
// Destinations: LL128 lines (whole lines, flag = epoch) or plain bytes (recv).
__device__ __forceinline__ bool ll128_piece(const char* sbase, char* dbase, const DevPiece& q,
                                            uint32_t epoch, int64_t timeout_ns, int32_t* err,
                                            char* wsm) {
  const bool sll = q.kind & kLLSrc, dll = q.kind & kLLDst;
  const int64_t n = q.nbytes, NL = (n + 119) / 120, sa = q.src_off;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j = lane & 7, li = lane >> 3;
  const uint64_t E = epoch;
  const int64_t r = sll ? sa % 120 : 0;
  char* ws = wsm + warp * 640;
  if (!sll || r == 0) {
    // plain source or a line-aligned LL128 source: kU line groups (16 lines)
    // per warp and turn, all their loads in flight before the first use.
    // Per-lane base pointers and strides are set up once (no division in the
    // loop); only the piece's last line can be partial.
    constexpr int kU = 4;
    const int cap = j == 7 ? 8 : 16;
    const int64_t NLfull = n / 120;                       // lines entirely inside the piece
    const char* sp = sll ? sbase + 128 * (sa / 120) + 16 * j : sbase + sa + 16 * j;
    const int64_t ss = sll ? 128 : 120;
    const bool sal = sll || (((uintptr_t)(sbase + sa)) & 7) == 0;   // 8-byte aligned plain loads
    char* dp = dll ? dbase + 128 * (q.dst_off / 120) + 16 * j : dbase + q.dst_off + 16 * j;
    const int64_t ds = dll ? 128 : 120;
    const bool dal = dll || (((uintptr_t)(dbase + q.dst_off)) & 7) == 0;
    for (int64_t L0 = (int64_t)warp * 4 * kU; L0 < NL; L0 += (int64_t)nw * 4 * kU) {
      uint64_t a[kU], b[kU];
      int nb[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t L = L0 + 4 * u + li;
        nb[u] = L < NLfull ? cap : L < NL ? (int)max((int64_t)0, min((int64_t)cap, n - 120 * L - 16 * j)) : -1;
        a[u] = b[u] = 0;
        const char* s = sp + L * ss;
        if (sll) {
          if (nb[u] >= 0) ld16v(s, a[u], b[u]);
        } else if (nb[u] == 16 && sal) {
          a[u] = reinterpret_cast<const uint64_t*>(s)[0];
          b[u] = reinterpret_cast<const uint64_t*>(s)[1];
        } else if (nb[u] == 8 && sal) {
          a[u] = reinterpret_cast<const uint64_t*>(s)[0];
        } else if (nb[u] > 0) {
          ld16_plain(s, nb[u], a[u], b[u]);
        }
      }
      if (sll) {  // poll: reload the line groups whose flag is not yet the epoch
        uint32_t spins = 0, nap = 0;
        uint64_t t0 = 0;
        for (;;) {
          bool ok = true;
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const uint64_t f = __shfl_sync(0xffffffffu, b[u], lane | 7);
            if (nb[u] >= 0 && f != E) {
              ok = false;
              ld16v(sp + (L0 + 4 * u + li) * ss, a[u], b[u]);
            }
          }
          if (__all_sync(0xffffffffu, ok)) break;
          if (++spins > kLLSpin) {
            nap = nap ? min(2 * nap, 1024u) : 64u;
            __nanosleep(nap);
          }
          if ((spins & 255) == 0) {
            const uint64_t now = globaltimer();
            if (t0 == 0) t0 = now;
            const bool out = (int64_t)(now - t0) > timeout_ns || *(volatile int32_t*)err != 0;
            if (__any_sync(0xffffffffu, out)) return false;
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        char* d = dp + (L0 + 4 * u + li) * ds;
        if (dll) {
          if (nb[u] >= 0) st16v(d, a[u], j == 7 ? E : b[u]);
        } else if (nb[u] == 16 && dal) {
          reinterpret_cast<uint64_t*>(d)[0] = a[u];
          reinterpret_cast<uint64_t*>(d)[1] = b[u];
        } else if (nb[u] == 8 && dal) {
          reinterpret_cast<uint64_t*>(d)[0] = a[u];
        } else if (nb[u] > 0) {
          plain_store8(d, a[u], min(nb[u], 8));
          if (nb[u] > 8) plain_store8(d + 8, b[u], nb[u] - 8);
        }
      }
    }
    return true;
  }
  for (int64_t L0 = (int64_t)warp * 4; L0 < NL; L0 += (int64_t)nw * 4) {
    const int64_t L = L0 + li;
    const bool live = L < NL;
    const int64_t pb = 120 * L + 16 * j;
    const int nb = live ? (int)max((int64_t)0, min((int64_t)(j == 7 ? 8 : 16), n - pb)) : 0;
    uint64_t a = 0, b = 0;
    {  // misaligned LL128 source: gather the window through shared memory
      const int64_t A = (sa + 120 * L0) / 120;
      const int64_t Aend = (sa + min(n, 120 * (L0 + 4)) - 1) / 120;
      uint64_t x = 0, y = 0;
      bool need = A + li <= Aend;
      if (!ll128_poll(sbase + 128 * (A + li), need, j, E, x, y, timeout_ns, err)) return false;
      if (need) {
        uint64_t* w = reinterpret_cast<uint64_t*>(ws + 120 * li + 16 * j);
        w[0] = x;
        if (j < 7) w[1] = y;
      }
      need = li == 0 && A + 4 <= Aend;
      if (!ll128_poll(sbase + 128 * (A + 4), need, j, E, x, y, timeout_ns, err)) return false;
      if (need) {
        uint64_t* w = reinterpret_cast<uint64_t*>(ws + 480 + 16 * j);
        w[0] = x;
        if (j < 7) w[1] = y;
      }
      __syncwarp();
      if (nb > 0) ld16_plain(ws + r + 120 * li + 16 * j, nb, a, b);
      __syncwarp();
    }
    if (dll) {
      if (live) st16v(dbase + 128 * (q.dst_off / 120 + L) + 16 * j, a, j == 7 ? E : b);
    } else if (nb > 0) {
      char* d = dbase + q.dst_off + pb;
      plain_store8(d, a, min(nb, 8));
      if (nb > 8) plain_store8(d + 8, b, nb - 8);
    }
  }
  return true;
}

// ---- TMA bulk-copy engine helpers (cp.async.bulk + mbarrier, SASS UBLKCP) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(smem_src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Race hunting on the device (tests only).  sync_mode bit 6: before every step /
// unit / chain task the CTA naps a pseudo-random 0-16 us, one time in 16 up to
// 260 us (keyed by epoch, CTA and wait range), so producers and consumers finish
// in orders the default timing never produces.  Bit 7 (mutation self-test): the
// dependency waits are skipped, so a perturbed run must then deliver a wrong
// transpose -- proof that the check bites.  Entry/exit barriers are unaffected.
constexpr int kSyncPerturb = 64, kSyncNoWaits = 128;
__device__ __forceinline__ void perturb_nap(uint32_t epoch, uint32_t key) {
  uint32_t h = epoch * 0x9E3779B1u ^ blockIdx.x * 0x85EBCA77u ^ key * 0xC2B2AE3Du;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12; h *= 0x297A2D39u; h ^= h >> 15;
  if (h & 1) return;
  // mostly short naps; one in 16 long enough that a producer which grabbed its
  // unit early finishes after consumers queued hundreds of units later
  __nanosleep(((h >> 1) & 7) == 0 ? (h >> 8) & 262143 : (h >> 8) & 16383);
}

// Warp 0 waits until every listed flag reached `epoch`: each lane polls its
// flags with relaxed loads (optionally backing off), then every lane executes
// fence.acq_rel (the PTX acquire pattern: morally-strong read + fence).
// Returns false on timeout.
__device__ bool warp_wait_flags(const uint32_t* flags, const int32_t* idx, int32_t lo, int32_t hi,
                                uint32_t epoch, int64_t timeout_ns, int32_t* err, bool sys,
                                int mode) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  uint64_t t0 = 0;
  if (mode & kSyncPerturb) perturb_nap(epoch, (uint32_t)lo * 7919u + (uint32_t)hi);
  if (mode & kSyncNoWaits) hi = lo;
  for (int32_t i = lo + lane; i < hi; i += 32) {
    const uint32_t* f = flags + idx[i];
    uint32_t spins = 0;
    for (;;) {
      const uint32_t v = (mode & 16) ? ld_acquire(f, sys) : ld_relaxed(f, sys);
      if ((int32_t)(v - epoch) >= 0) break;
      if (mode & 8) __nanosleep(64);
      if ((++spins & 255) == 0) {
        uint64_t now = globaltimer();
        if (t0 == 0) t0 = now;
        if ((int64_t)(now - t0) > timeout_ns || *(volatile int32_t*)err != 0) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) break;
  }
  fence_acq_rel(sys);
  ok = __all_sync(0xffffffffu, ok);
  if (!ok && lane == 0) atomicCAS(err, 0, (int32_t)A2A_ERR_TIMEOUT);
  return ok;
}

// Chunk cursor over the 16-byte-aligned bodies of a staged batch of pieces
// (TMA engine).  Heads/tails and misaligned pieces are copied by threads.
// pieces at most this long are copied with 128-bit loads/stores by all threads
// even in the TMA engine: no bulk-group completion round trip before publishing
constexpr int64_t kSmallPiece = 32768;

struct BodyCursor {
  const DevPiece* pc;
  int32_t k, n;
  int64_t off;
  __device__ bool next(const KParams& p, uint32_t ch, const char** src, char** dst, uint32_t* len) {
    while (k < n) {
      const DevPiece& q = pc[k];
      if (q.nbytes <= kSmallPiece || q.kind != kCopy) { ++k; off = 0; continue; }
      const char* s0 = p.base[q.src_loc] + q.src_off;
      char* d0 = p.base[q.dst_loc] + q.dst_off;
      const int64_t L = q.nbytes;
      if ((((uintptr_t)s0 ^ (uintptr_t)d0) & 15) != 0) { ++k; off = 0; continue; }
      int64_t head = (16 - ((uintptr_t)d0 & 15)) & 15;
      if (head > L) head = L;
      const int64_t body = (L - head) & ~(int64_t)15;
      if (off >= body) { ++k; off = 0; continue; }
      const int64_t c = min((int64_t)ch, body - off);
      *src = s0 + head + off;
      *dst = d0 + head + off;
      *len = (uint32_t)c;
      off += c;
      return true;
    }
    return false;
  }
};

// ---- device-side epochs (graph-capturable executes) ----
// Every CTA keeps the epoch of its last all-to-all in its own device word: it
// reads it at kernel start (+1) and writes it back at its end.  All CTAs run
// every execute, so the words agree, no cross-CTA synchronisation is needed,
// and a replayed CUDA graph runs a fresh epoch each time without the host.
__device__ __forceinline__ uint32_t begin_epoch(const KParams& p) {
  const uint32_t e = *(volatile const uint32_t*)(p.ctl + blockIdx.x) + 1;
  return e == 0 ? 1 : e;
}
__device__ __forceinline__ void end_epoch(const KParams& p, uint32_t epoch) {
  __syncthreads();  // every thread has read the old value
  if (threadIdx.x == 0) p.ctl[blockIdx.x] = epoch;
}

template <int kEngine, int kThreads>
__device__ __forceinline__ void exec_body(const KParams& p, const uint32_t epoch) {
  __shared__ int s_abort;
  extern __shared__ __align__(128) unsigned char dsmem[];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5;
  // dynamic smem: [TMA: S mbarriers | S dst ptrs | S sizes | pad | S stages] [program] [batch]
  const int S = p.tma_stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsmem);
  char** ring_dst = reinterpret_cast<char**>(dsmem + 8 * S);
  uint32_t* ring_n = reinterpret_cast<uint32_t*>(dsmem + 16 * S);
  char* stages = reinterpret_cast<char*>(dsmem + ((20 * S + 127) & ~127));
  CtaStep* s_prog = reinterpret_cast<CtaStep*>(dsmem + p.smem_prog);
  DevPiece* s_pc = reinterpret_cast<DevPiece*>(dsmem + p.smem_batch);
  uint32_t gi = 0;  // TMA chunks consumed so far (thread 0): stage/phase bookkeeping
  unsigned long long* tl = p.timeline + (int64_t)c * (2 * p.T + 3);
  if (tid == 0) {
    tl[0] = globaltimer();
    s_abort = 0;
    if (kEngine == 1) {
      for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  // ---- LL entry: announce the epoch; a peer's landing region of this parity
  //      was last read two all-to-alls ago, so it is free once that peer has
  //      started the previous one (its entry flag >= epoch - 1).  Overlaps the
  //      program staging below (one barrier for both).
  if (p.G > 1 && p.ll) {
    if (c == 0 && tid < p.G && tid != p.rank) st_relaxed(p.entry_flags[tid] + p.rank, epoch, true);
    if (warp == 0) {
      const int lane = tid & 31;
      bool ok = true;
      if (lane < p.G && lane != p.rank) {
        const uint32_t* f = p.entry_flags[p.rank] + lane;
        uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while ((int32_t)(ld_relaxed(f, true) - (epoch - 1)) < 0) {
          if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                       *(volatile int32_t*)p.err != 0)) {
            ok = false;
            break;
          }
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (!ok && lane == 0) { atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT); s_abort = 1; }
    }
  }
  // stage this CTA's step program (one parallel load instead of per-step
  // chains); with the LL entry poll in warp 0, the other warps stage
  const int st = (p.G > 1 && p.ll) ? (tid + kThreads - 32) % kThreads : tid;
  for (int i = st; i < p.T; i += kThreads) s_prog[i] = p.prog[(int64_t)c * p.T + i];
  // if all of this CTA's pieces (every step) fit the batch buffer, stage them
  // now too: no per-step piece load on the latency path (small shards)
  const int32_t pb0 = p.prog[(int64_t)c * p.T].pb, pe1 = p.prog[(int64_t)c * p.T + p.T - 1].pe;
  const bool all_staged = pe1 - pb0 <= p.batch;
  if (all_staged)
    for (int i = st; i < pe1 - pb0; i += kThreads) s_pc[i] = p.pieces[pb0 + i];
  __syncthreads();
  if (s_abort) return;
  const uint32_t* my_flags = p.step_flags[p.rank];
  // one GPU (or LL: every step flag is GPU-local) -> .gpu scope suffices
  const bool sys = (p.G > 1 && !p.ll) || (p.sync_mode & 4);

  // ---- entry barrier: announce epoch to every peer, then wait for theirs
  if (p.G > 1 && !p.ll) {
    // relaxed: the flag orders nothing of this kernel -- the reads it vouches for
    // (the previous all-to-all's) completed at the kernel boundary
    if (c == 0 && tid < p.G && tid != p.rank) st_relaxed(p.entry_flags[tid] + p.rank, epoch, true);
    if (warp == 0) {
      const int lane = tid & 31;
      bool ok = true;
      if (lane < p.G && lane != p.rank) {
        const uint32_t* f = p.entry_flags[p.rank] + lane;
        uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
          if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                       *(volatile int32_t*)p.err != 0)) {
            ok = false;
            break;
          }
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (!ok) {
        if (lane == 0) { atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT); s_abort = 1; }
      }
    }
    __syncthreads();
    if (s_abort) return;
  }
  if (tid == 0) tl[1] = globaltimer();

  for (int t = 0; t < p.T; ++t) {
    const CtaStep cs = s_prog[t];
    if (cs.pe <= cs.pb) {
      if (tid == 0) tl[2 + t] = tl[3 + p.T + t] = 0;
      continue;
    }
    if (tid == 0 && cs.we <= cs.wb) tl[3 + p.T + t] = 0;
    bool waited = cs.we <= cs.wb && !(p.sync_mode & kSyncPerturb);
    for (int32_t base = cs.pb; base < cs.pe; base += p.batch) {
      const int n = min(p.batch, cs.pe - base);
      DevPiece* pcs = s_pc;
      if (all_staged) {
        pcs = s_pc + (base - pb0);
      } else {  // stage the batch first: independent of the flags, so it overlaps the wait
        for (int i = tid; i < n; i += kThreads) s_pc[i] = p.pieces[base + i];
      }
      if (!waited) {
        if (warp == 0) {
          bool ok = warp_wait_flags(my_flags, p.wait_idx, cs.wb, cs.we, epoch, p.timeout_ns,
                                    p.err, sys, p.sync_mode);
          if (!ok && tid == 0) s_abort = 1;
          if (tid == 0) tl[3 + p.T + t] = globaltimer();
        }
        waited = true;
      }
      __syncthreads();
      if (s_abort) return;
      // LL pieces (any size) and small copies: all threads, in program order
      // (same-step decodes are last in every CTA's step)
      for (int i = 0; i < n; ++i) {
        const DevPiece& q = pcs[i];
        if (q.kind != kCopy) {  // LL regions: this epoch's parity
          const char* sb = p.base[q.src_loc];
          char* db = p.base[q.dst_loc];
          if (q.kind & kLLSrc) sb += (epoch & 1) * p.ll_half[p.rank];
          if (q.kind & kLLDst) db += (epoch & 1) * p.ll_half[q.dst_loc - (1 + 2 * p.G)];
          bool ok;
          if constexpr (kThreads <= 512)   // LL128 plans launch the 512- or 256-thread kernels
            ok = p.ll128 ? ll128_piece(sb, db, q, epoch, p.timeout_ns, p.err,
                                       reinterpret_cast<char*>(dsmem + p.smem_ll))
                         : ll_piece(sb, db, q, epoch, p.timeout_ns, p.err);
          else
            ok = ll_piece(sb, db, q, epoch, p.timeout_ns, p.err);
          if (!ok) {
            atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
            s_abort = 1;
          }
        } else if (kEngine == 0 || q.nbytes <= kSmallPiece) {
          cta_copy<4>(p.base[q.dst_loc] + q.dst_off, p.base[q.src_loc] + q.src_off, q.nbytes);
        }
      }
      if (kEngine == 1) {
        bool any_big = false;
        for (int i = 0; i < n && !any_big; ++i) any_big = pcs[i].nbytes > kSmallPiece && pcs[i].kind == kCopy;
        if (!any_big) {
          // nothing for the TMA ring in this batch
        } else if (tid != 0) {  // threads 1..: heads, tails, misaligned big pieces
          const int nt = kThreads - 1, me = tid - 1;
          for (int i = 0; i < n; ++i) {
            const DevPiece& q = pcs[i];
            if (q.nbytes <= kSmallPiece || q.kind != kCopy) continue;
            const char* s0 = p.base[q.src_loc] + q.src_off;
            char* d0 = p.base[q.dst_loc] + q.dst_off;
            const int64_t len = q.nbytes;
            if ((((uintptr_t)s0 ^ (uintptr_t)d0) & 15) != 0) {
              for (int64_t j = me; j < len; j += nt) d0[j] = s0[j];
            } else {
              int64_t head = (16 - ((uintptr_t)d0 & 15)) & 15;
              if (head > len) head = len;
              const int64_t body = (len - head) & ~(int64_t)15, tail = len - head - body;
              if (me < head) d0[me] = s0[me];
              if (me < tail) d0[head + body + me] = s0[head + body + me];
            }
          }
        } else {  // thread 0: TMA pipeline over the batch's bodies
          fence_proxy_async();
          const uint32_t CH = (uint32_t)p.tma_chunk;
          BodyCursor cur{pcs, 0, n, 0};
          const uint32_t g0 = gi;
          uint32_t nl = 0, ns = 0;
          bool more = true;
          auto issue = [&]() -> bool {
            const char* src;
            char* dst;
            uint32_t len;
            if (!cur.next(p, CH, &src, &dst, &len)) return false;
            const uint32_t st = (g0 + nl) % S;
            ring_dst[st] = dst;
            ring_n[st] = len;
            mbar_expect_tx(&bars[st], len);
            bulk_load(stages + (size_t)st * CH, src, len, &bars[st]);
            ++nl;
            return true;
          };
          while (more && nl < (uint32_t)S) more = issue();
          while (ns < nl) {
            const uint32_t st = (g0 + ns) % S;
            mbar_wait(&bars[st], ((g0 + ns) / S) & 1);
            bulk_store(ring_dst[st], stages + (size_t)st * CH, ring_n[st]);
            ++ns;
            if (more) {
              if (S == 1) {
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                more = issue();
              } else if (ns >= 2 && nl - (uint32_t)S == ns - 2) {
                bulk_wait_read1();
                more = issue();
              }
            }
          }
          bulk_wait_all();
          fence_proxy_async();
          gi = g0 + nl;
        }
      }
      if (p.count_links && tid == 0)
        for (int i = 0; i < n; ++i)
          if (pcs[i].edge >= 0)
            atomicAdd(p.counters + (int64_t)t * p.E + pcs[i].edge, (unsigned long long)pcs[i].nbytes);
      __syncthreads();
    }
    if (s_abort) return;
    if (tid == 0) {
      const int64_t slot = ((int64_t)t * p.G + p.rank) * p.nC + c;
      if (p.sync_mode & 32) {
        // release pattern: one fence, then relaxed flag stores, peers first
        fence_acq_rel(sys);
        const uint32_t own = 1u << p.rank;
        uint32_t mask = cs.mask & ~own;
        while (mask) {
          const int h = __ffs(mask) - 1;
          mask &= mask - 1;
          st_relaxed(p.step_flags[h] + slot, epoch, sys);
        }
        if (cs.mask & own) st_relaxed(p.step_flags[p.rank] + slot, epoch, sys);
      } else {
        if (!(p.sync_mode & 2)) {
          if (p.sync_mode & 1) fence_acq_rel(sys);
          else if (sys) __threadfence_system();
          else __threadfence();
        }
        uint32_t mask = cs.mask;
        while (mask) {
          const int h = __ffs(mask) - 1;
          mask &= mask - 1;
          st_release(p.step_flags[h] + slot, epoch, sys);
        }
      }
      tl[2 + t] = globaltimer();
    }
  }
  // ---- LL exit: every peer's entry flag for this epoch has landed here, so
  //      once the kernel completes no peer store into this arena is in flight
  //      (the lines were all polled; the flags are stored at peer kernel start)
  if (c == 0 && p.G > 1 && p.ll && warp == 0) {
    const int lane = tid & 31;
    bool ok = true;
    if (lane < p.G && lane != p.rank) {
      const uint32_t* f = p.entry_flags[p.rank] + lane;
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while ((int32_t)(ld_relaxed(f, true) - epoch) < 0) {
        if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                     *(volatile int32_t*)p.err != 0)) {
          ok = false;
          break;
        }
      }
    }
    if (!__all_sync(0xffffffffu, ok) && lane == 0) atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
  }
  // ---- exit: all incoming stores of every step have landed (multi-GPU)
  if (c == 0 && p.G > 1 && !p.ll) {
    bool ok = true;
    for (int32_t i = tid; i < p.n_exit && ok; i += kThreads) {
      const uint32_t* f = my_flags + p.exit_idx[i];
      uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
        if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                     *(volatile int32_t*)p.err != 0)) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
    __syncthreads();
  }
  if (tid == 0) tl[2 + p.T] = globaltimer();
}

template <int kEngine, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) a2a_exec_kernel(const KParams p) {
  const uint32_t epoch = begin_epoch(p);
  exec_body<kEngine, kThreads>(p, epoch);
  end_epoch(p, epoch);
}

// ---- dynamic mode: CTAs grab units from a per-GPU counter ----
// Ready-queue mode (kReady): units are enqueued on their GPU's queue when
// their last producer finishes (per-unit completion counters, counted down
// with acq_rel system-scope atomics over NVLink); a CTA claims the next queue
// position while it copies its current unit and waits for that position only
// after publishing, so CTAs never wait on a unit whose inputs are missing
// while ready work exists (csrc/a2a_plan.cpp build_dyn, emulate_ready).
__device__ __forceinline__ void ready_push(const KParams& p, int h, int32_t li, uint32_t epoch) {
  const int32_t nu = p.ubase[h + 1] - p.ubase[h];
  const unsigned long long pos =
      atom_add_relaxed_sys(p.qctl[h] + 1, 1ull) - (unsigned long long)(epoch - 1) * (unsigned long long)nu;
  if (pos >= (unsigned long long)nu) {  // more pushes than units: a broken epoch; never write past the queue
    atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
    return;
  }
  st_release_sys_u64(p.qslot[h] + pos, ((unsigned long long)epoch << 32) | (uint32_t)li);
}

template <int kEngine, int kThreads, bool kReady>
__device__ __forceinline__ void dyn_body(const KParams& p, const uint32_t epoch) {
  __shared__ int s_abort;
  __shared__ long long s_idx[2];
  __shared__ DevUnit s_u[2];
  __shared__ DevPiece s_pc[2];
  extern __shared__ __align__(128) unsigned char dsmem[];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5;
  const int S = p.tma_stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsmem);
  char** ring_dst = reinterpret_cast<char**>(dsmem + 8 * S);
  uint32_t* ring_n = reinterpret_cast<uint32_t*>(dsmem + 16 * S);
  char* stages = reinterpret_cast<char*>(dsmem + ((20 * S + 127) & ~127));
  uint32_t gi = 0;
  unsigned long long* tl = p.timeline + (int64_t)c * (2 * p.T + 3);
  if (tid == 0) {
    tl[0] = globaltimer();
    s_abort = 0;
    if (kEngine == 1) {
      for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const uint32_t* my_flags = p.step_flags[p.rank];
  const bool sys = p.G > 1 || (p.sync_mode & 4);
  if (p.G > 1) {  // entry barrier (same protocol as the static kernel)
    // relaxed: the flag orders nothing of this kernel -- the reads it vouches for
    // (the previous all-to-all's) completed at the kernel boundary
    if (c == 0 && tid < p.G && tid != p.rank) st_relaxed(p.entry_flags[tid] + p.rank, epoch, true);
    if (warp == 0) {
      const int lane = tid & 31;
      bool ok = true;
      if (lane < p.G && lane != p.rank) {
        const uint32_t* f = p.entry_flags[p.rank] + lane;
        uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
          if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                       *(volatile int32_t*)p.err != 0)) {
            ok = false;
            break;
          }
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (!ok && lane == 0) { atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT); s_abort = 1; }
    }
    __syncthreads();
    if (s_abort) return;
  }
  if (tid == 0) tl[1] = globaltimer();
  if (kReady && c == 0)  // seed this GPU's queue with its dependency-free units
    for (int32_t i = tid; i < p.n_init; i += kThreads) ready_push(p, p.rank, i, epoch);
  unsigned long long waited_ns = 0, done = 0;
  int q = c < p.remote_ctas ? 0 : 1, visited = 0;  // queue state, owned by the fetching thread
  // fetch (grab + descriptor) of the next unit into slot `sl`; thread `fetcher`
  // (ready mode: claim the next queue position only -- it is waited for in acquire)
  auto fetch = [&](int sl) {
    if (kReady) {
      const long long n = p.n_units;
      const long long j = (long long)(atomicAdd(p.grab, 1ull) -
                                      (unsigned long long)(epoch - 1) * (unsigned long long)(n + p.nC));
      s_idx[sl] = j < n ? j : -1;
      return;
    }
    long long idx = -1;
    for (;;) {  // own queue first, then the other; one failing grab per queue
      // per execute a queue's counter advances by its units plus one failing
      // grab per CTA that visits it: every CTA, or (pinned) the CTAs on it
      const long long qn = q == 0 ? p.n_remote : (long long)p.n_units - p.n_remote;
      const long long visitors = !p.pin_queues ? p.nC : q == 0 ? p.remote_ctas : p.nC - p.remote_ctas;
      const long long j = (long long)(atomicAdd(p.grab + q, 1ull) -
                                      (unsigned long long)(epoch - 1) * (unsigned long long)(qn + visitors));
      if (j < qn) { idx = (q == 0 ? 0 : p.n_remote) + j; break; }
      if (++visited == 2 || p.pin_queues) break;
      q ^= 1;
    }
    s_idx[sl] = idx;
    if (idx >= 0) {
      const DevUnit u = p.units[idx];
      s_u[sl] = u;
      s_pc[sl] = DevPiece{u.src_off, u.dst_off, u.nbytes, u.edge, u.src_loc, u.dst_loc, 0};
    }
  };
  // acquire the producers of the unit in slot `sl` (one warp); ready mode:
  // wait until the claimed queue position is filled, then load the unit
  auto acquire = [&](int sl) -> bool {
    if (kReady) {
      if (s_idx[sl] < 0) return true;
      bool ok = true;
      if ((tid & 31) == 0) {
        const unsigned long long* slot = p.qslot[p.rank] + s_idx[sl];
        const uint64_t w0 = globaltimer();
        uint32_t spins = 0;
        unsigned long long v;
        while ((uint32_t)((v = ld_acquire_sys_u64(slot)) >> 32) != epoch) {
          if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - w0) > p.timeout_ns ||
                                       *(volatile int32_t*)p.err != 0)) {
            ok = false;
            break;
          }
        }
        waited_ns += globaltimer() - w0;
        if (ok) {
          const long long li = (long long)(uint32_t)v;
          const DevUnit u = p.units[li];
          s_idx[sl] = li;
          s_u[sl] = u;
          s_pc[sl] = DevPiece{u.src_off, u.dst_off, u.nbytes, u.edge, u.src_loc, u.dst_loc, 0};
        } else {
          atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
        }
      }
      return __shfl_sync(0xffffffffu, ok, 0);
    }
    const DevUnit& u = s_u[sl];
    if (s_idx[sl] < 0 || (u.we <= u.wb && !(p.sync_mode & kSyncPerturb))) return true;
    const uint64_t w0 = globaltimer();
    bool ok = warp_wait_flags(my_flags, p.unit_wait, u.wb, u.we, epoch, p.timeout_ns, p.err,
                              sys, p.sync_mode);
    if ((tid & 31) == 0) waited_ns += globaltimer() - w0;
    return ok;
  };
  // TMA engine: warp 1 prefetches unit k+1 (grab, descriptor, dependency wait)
  // while thread 0 streams unit k and threads 64.. copy its heads/tails.
  const int fw = kEngine == 1 ? 1 : 0;  // fetching warp
  if (warp == fw) {
    if ((tid & 31) == 0) fetch(0);
    __syncwarp();
    if (!acquire(0) && (tid & 31) == 0) s_abort = 1;
  }
  __syncthreads();
  if (s_abort) return;
  int cur = 0;
  for (;;) {
    const long long idx = s_idx[cur];
    if (idx < 0) break;
    const DevUnit u = s_u[cur];
    const char* s0 = p.base[u.src_loc] + u.src_off;
    char* d0 = p.base[u.dst_loc] + u.dst_off;
    // the next unit is only grabbed here; its dependency wait comes after this
    // unit's flag is published, so a CTA never withholds a finished unit
    if (kEngine == 0) {
      cta_copy<4>(d0, s0, u.nbytes);
      if (tid == 0) fetch(cur ^ 1);
    } else if (u.nbytes <= kSmallPiece) {  // small unit: all threads, no bulk round trip
      cta_copy<4>(d0, s0, u.nbytes);
      if (warp == fw && (tid & 31) == 0) fetch(cur ^ 1);
    } else if (warp == fw) {
      if ((tid & 31) == 0) fetch(cur ^ 1);
    } else if (tid >= 64) {
      const int nt = kThreads - 64, me = tid - 64;
      const int64_t len = u.nbytes;
      if ((((uintptr_t)s0 ^ (uintptr_t)d0) & 15) != 0) {
        for (int64_t j = me; j < len; j += nt) d0[j] = s0[j];
      } else {
        int64_t head = (16 - ((uintptr_t)d0 & 15)) & 15;
        if (head > len) head = len;
        const int64_t body = (len - head) & ~(int64_t)15, tail = len - head - body;
        if (me < head) d0[me] = s0[me];
        if (me < tail) d0[head + body + me] = s0[head + body + me];
      }
    } else if (tid == 0) {
      fence_proxy_async();
      const uint32_t CH = (uint32_t)p.tma_chunk;
      BodyCursor bc{&s_pc[cur], 0, 1, 0};
      const uint32_t g0 = gi;
      uint32_t nl = 0, ns = 0;
      bool more = true;
      auto issue = [&]() -> bool {
        const char* src;
        char* dst;
        uint32_t len;
        if (!bc.next(p, CH, &src, &dst, &len)) return false;
        const uint32_t st = (g0 + nl) % S;
        ring_dst[st] = dst;
        ring_n[st] = len;
        mbar_expect_tx(&bars[st], len);
        bulk_load(stages + (size_t)st * CH, src, len, &bars[st]);
        ++nl;
        return true;
      };
      while (more && nl < (uint32_t)S) more = issue();
      while (ns < nl) {
        const uint32_t st = (g0 + ns) % S;
        mbar_wait(&bars[st], ((g0 + ns) / S) & 1);
        bulk_store(ring_dst[st], stages + (size_t)st * CH, ring_n[st]);
        ++ns;
        if (more) {
          if (S == 1) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            more = issue();
          } else if (ns >= 2 && nl - (uint32_t)S == ns - 2) {
            bulk_wait_read1();
            more = issue();
          }
        }
      }
      bulk_wait_all();
      fence_proxy_async();
      gi = g0 + nl;
    }
    if (p.count_links && tid == 0 && u.edge >= 0)
      atomicAdd(p.counters + (int64_t)u.step * p.E + u.edge, (unsigned long long)u.nbytes);
    __syncthreads();
    if (kReady && warp == 0) {
      // count down the dependents, one lane each (acq_rel at system scope:
      // releases this CTA's stores, which bar.sync made cumulative, and chains
      // the earlier producers' releases); the lane that completes a dependent
      // enqueues it on its GPU; lane 31 counts the unit into its destination
      const int lane = tid & 31;
      for (int32_t k = u.wb + lane; k < u.we; k += 31) {
        if (lane == 31) break;
        const int32_t gid = p.unit_wait[2 * k], deg = p.unit_wait[2 * k + 1];
        int h = 0;
        while (gid >= p.ubase[h + 1]) ++h;
        const int32_t lj = gid - p.ubase[h];
        const unsigned long long old = atom_add_acq_rel_sys(p.qdone[h] + lj, 1ull);
        if (old + 1 == (unsigned long long)epoch * (unsigned long long)deg) ready_push(p, h, lj, epoch);
      }
      if (lane == 31) {
        const int hd = u.dst_loc >= 1 && u.dst_loc < 1 + p.G ? u.dst_loc - 1 : u.dst_loc - 1 - p.G;
        red_add_release_sys(p.qctl[hd] + 2, 1ull);
      }
      if (lane == 0) ++done;
    } else if (!kReady && tid == 0) {
      const int64_t slot = (int64_t)p.unit_base + idx;
      uint32_t mask = u.mask;
      while (mask) {
        const int h = __ffs(mask) - 1;
        mask &= mask - 1;
        st_release(p.step_flags[h] + slot, epoch, sys);
      }
      ++done;
    }
    if (warp == fw && !acquire(cur ^ 1) && (tid & 31) == 0) s_abort = 1;
    __syncthreads();
    if (s_abort) return;
    cur ^= 1;
  }
  if (kReady && c == 0 && tid == 0) {  // exit: every unit writing into this GPU has finished
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    const unsigned long long want = (unsigned long long)epoch * (unsigned long long)p.n_into;
    while (ld_acquire_sys_u64(p.qctl[p.rank] + 2) < want) {
      if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                   *(volatile int32_t*)p.err != 0)) {
        atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
        break;
      }
    }
  }
  if (!kReady && c == 0 && p.G > 1) {  // exit: every unit flagged into this GPU has landed
    bool ok = true;
    for (int32_t i = tid; i < p.n_exit && ok; i += kThreads) {
      const uint32_t* f = my_flags + p.exit_idx[i];
      uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
        if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                     *(volatile int32_t*)p.err != 0)) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
    __syncthreads();
  }
  if (tid == 0) {
    tl[2] = done;
    tl[2 + p.T] = globaltimer();
  }
  if (tid == (kEngine == 1 ? 32 : 0)) tl[3] = waited_ns;
}

template <int kEngine, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) a2a_dyn_kernel(const KParams p) {
  const uint32_t epoch = begin_epoch(p);
  dyn_body<kEngine, kThreads, false>(p, epoch);
  end_epoch(p, epoch);
}

template <int kEngine, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) a2a_ready_kernel(const KParams p) {
  const uint32_t epoch = begin_epoch(p);
  dyn_body<kEngine, kThreads, true>(p, epoch);
  end_epoch(p, epoch);
}


// ---- chain mode (sched_mode 7): a route's consecutive local hops stream through L2 ----
// A task is a chain of units (build_dyn): the head waits on its producers' flags;
// every later unit reads exactly the bytes the previous one stored, on the same
// CTA.  Thread 0 streams the whole chain through one TMA ring: chunk c of hop
// u+1 is loaded K chunks after chunk c of hop u was stored (K = chunks per unit
// >= ring depth), once `cp.async.bulk.wait_group` says that store completed, so
// the forwarded bytes are read back while they still sit in L2 and the ring
// never drains between hops.  Tasks whose units are not 16-byte clean at run
// time (odd shard sizes, user buffers) copy unit by unit with all threads.
__device__ __forceinline__ void bulk_wait_n(uint32_t n) {
  switch (n) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 7;" ::: "memory"); break;
  }
}

template <int kEngine, int kThreads>
__device__ __forceinline__ void chain_body(const KParams& p, const uint32_t epoch) {
  __shared__ int s_abort, s_cleans[2];
  __shared__ long long s_tasks[2];
  extern __shared__ __align__(128) unsigned char dsmem[];
  const int c = blockIdx.x, tid = threadIdx.x, warp = tid >> 5;
  const int S = p.tma_stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsmem);
  char** ring_dst = reinterpret_cast<char**>(dsmem + 8 * S);
  uint32_t* ring_n = reinterpret_cast<uint32_t*>(dsmem + 16 * S);
  char* stages = reinterpret_cast<char*>(dsmem + ((20 * S + 127) & ~127));
  uint32_t gi = 0;
  unsigned long long* tl = p.timeline + (int64_t)c * (2 * p.T + 3);
  if (tid == 0) {
    tl[0] = globaltimer();
    s_abort = 0;
    if (kEngine == 1) {
      for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  const uint32_t* my_flags = p.step_flags[p.rank];
  const bool sys = p.G > 1 || (p.sync_mode & 4);
  if (p.G > 1) {  // entry barrier (same protocol as the other kernels)
    if (c == 0 && tid < p.G && tid != p.rank) st_relaxed(p.entry_flags[tid] + p.rank, epoch, true);
    if (warp == 0) {
      const int lane = tid & 31;
      bool ok = true;
      if (lane < p.G && lane != p.rank) {
        const uint32_t* f = p.entry_flags[p.rank] + lane;
        uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
          if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                       *(volatile int32_t*)p.err != 0)) {
            ok = false;
            break;
          }
        }
      }
      ok = __all_sync(0xffffffffu, ok);
      if (!ok && lane == 0) { atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT); s_abort = 1; }
    }
    __syncthreads();
    if (s_abort) return;
  }
  if (tid == 0) tl[1] = globaltimer();
  unsigned long long waited_ns = 0, done = 0;
  // warp 1 grabs the next task and reads its head while thread 0 streams the
  // current one; the head's dependency wait comes only after the current
  // task has published (it may depend on it), as in dyn_body
  auto grab = [&](int sl) {
    const long long nt = p.n_tasks;
    const long long j = (long long)(atomicAdd(p.grab, 1ull) -
                                    (unsigned long long)(epoch - 1) * (unsigned long long)(nt + p.nC));
    s_tasks[sl] = j < nt ? j : -1;
    if (j < nt) {
      const int32_t ub = p.chain_begin[j], ue = p.chain_begin[j + 1];
      const DevUnit head = p.units[ub];
      // TMA streaming needs every unit 16-byte clean, larger than a small piece,
      // and (several hops) a later hop's chunk loaded >= S chunks after its store
      int clean = kEngine == 1;
      for (int32_t k = ub; k < ue && clean; ++k) {
        const DevUnit u = p.units[k];
        const uintptr_t a = (uintptr_t)(p.base[u.src_loc] + u.src_off) | (uintptr_t)(p.base[u.dst_loc] + u.dst_off);
        clean = ((a | (uintptr_t)u.nbytes) & 15) == 0 && u.nbytes > kSmallPiece && u.nbytes == head.nbytes;
      }
      if (ue - ub > 1 && (head.nbytes + p.tma_chunk - 1) / p.tma_chunk < S) clean = 0;
      s_cleans[sl] = clean;
    }
  };
  if (tid == 32) grab(0);
  __syncthreads();
  int cur = 0;
  for (;;) {
    const long long task = s_tasks[cur];
    if (task < 0) break;
    const int32_t ub = p.chain_begin[task], ue = p.chain_begin[task + 1];
    const DevUnit head = p.units[ub];
    if (warp == 0 && (head.we > head.wb || (p.sync_mode & kSyncPerturb))) {
      const uint64_t w0 = globaltimer();
      if (!warp_wait_flags(my_flags, p.unit_wait, head.wb, head.we, epoch, p.timeout_ns, p.err, sys,
                           p.sync_mode) && tid == 0)
        s_abort = 1;
      if (tid == 0) waited_ns += globaltimer() - w0;
    }
    __syncthreads();
    if (s_abort) return;
    const int clean_now = s_cleans[cur];
    if (tid == 32 && (kEngine == 1 && clean_now)) grab(cur ^ 1);   // overlaps thread 0's stream
    if (kEngine == 1 && clean_now) {
      if (tid == 0) {
        fence_proxy_async();
        const uint32_t CH = (uint32_t)p.tma_chunk;
        const int64_t n = head.nbytes;
        const uint32_t K = (uint32_t)((n + CH - 1) / CH), total = K * (uint32_t)(ue - ub);
        const uint32_t g0 = gi;
        uint32_t nl = 0, ns = 0;
        auto issue = [&]() -> bool {
          if (nl >= total) return false;
          const int32_t k = ub + (int32_t)(nl / K);
          const int64_t off = (int64_t)(nl % K) * CH;
          const uint32_t len = (uint32_t)min((int64_t)CH, n - off);
          if (nl >= K) bulk_wait_n(ns - 1 - (nl - K));   // the previous hop's store of these bytes
          const DevUnit& u = p.units[k];
          const uint32_t st = (g0 + nl) % S;
          ring_dst[st] = p.base[u.dst_loc] + u.dst_off + off;
          ring_n[st] = len;
          mbar_expect_tx(&bars[st], len);
          bulk_load(stages + (size_t)st * CH, p.base[u.src_loc] + u.src_off + off, len, &bars[st]);
          ++nl;
          return true;
        };
        bool more = true;
        while (more && nl < (uint32_t)S) more = issue();
        while (ns < nl) {
          const uint32_t st = (g0 + ns) % S;
          mbar_wait(&bars[st], ((g0 + ns) / S) & 1);
          bulk_store(ring_dst[st], stages + (size_t)st * CH, ring_n[st]);
          ++ns;
          if (more) {
            if (S == 1) {
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              more = issue();
            } else if (ns >= 2 && nl - (uint32_t)S == ns - 2) {
              bulk_wait_read1();
              more = issue();
            }
          }
        }
        bulk_wait_all();
        fence_proxy_async();
        gi = g0 + nl;
      }
    } else {
      for (int32_t k = ub; k < ue; ++k) {   // unit by unit, every thread
        const DevUnit u = p.units[k];
        cta_copy<4>(p.base[u.dst_loc] + u.dst_off, p.base[u.src_loc] + u.src_off, u.nbytes);
        __syncthreads();                    // the next unit reads these bytes
      }
      if (tid == 32) grab(cur ^ 1);
    }
    __syncthreads();
    if (p.chain_discard && ue - ub > 1) {
      // every hop but the last stored into scratch that only the next hop of
      // this task reads (build_dyn links a unit only to its sole consumer), and
      // that read has completed: drop those dirty L2 lines instead of writing
      // dead bytes back to HBM.  Only 128-byte lines entirely inside a unit's
      // range are discarded (a partial line may hold a neighbour's live bytes).
      for (int32_t k = ub; k + 1 < ue; ++k) {
        const DevUnit u = p.units[k];
        const uintptr_t a = (uintptr_t)(p.base[u.dst_loc] + u.dst_off);
        const uintptr_t lo = (a + 127) & ~(uintptr_t)127, hi = (a + u.nbytes) & ~(uintptr_t)127;
        for (uintptr_t x = lo + (uintptr_t)tid * 128; x < hi; x += (uintptr_t)kThreads * 128)
          asm volatile("discard.global.L2 [%0], 128;" ::"l"(x) : "memory");
      }
    }
    if (tid == 0) {   // every unit of the task: link counters, then its flag on each GPU of its mask
      for (int32_t k = ub; k < ue; ++k) {
        const DevUnit u = p.units[k];
        if (p.count_links && u.edge >= 0)
          atomicAdd(p.counters + (int64_t)u.step * p.E + u.edge, (unsigned long long)u.nbytes);
        const int64_t slot = (int64_t)p.unit_base + k;
        uint32_t mask = u.mask;
        while (mask) {
          const int h = __ffs(mask) - 1;
          mask &= mask - 1;
          st_release(p.step_flags[h] + slot, epoch, sys);
        }
        ++done;
      }
    }
    __syncthreads();   // the next task's slot is filled; this task is published
    cur ^= 1;
  }
  if (c == 0 && p.G > 1) {  // exit: every unit flagged into this GPU has landed
    bool ok = true;
    for (int32_t i = tid; i < p.n_exit && ok; i += kThreads) {
      const uint32_t* f = my_flags + p.exit_idx[i];
      uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while ((int32_t)(ld_acquire_sys(f) - epoch) < 0) {
        if ((++spins & 255) == 0 && ((int64_t)(globaltimer() - t0) > p.timeout_ns ||
                                     *(volatile int32_t*)p.err != 0)) {
          ok = false;
          break;
        }
      }
    }
    if (!ok) atomicCAS(p.err, 0, (int32_t)A2A_ERR_TIMEOUT);
    __syncthreads();
  }
  if (tid == 0) {
    tl[2] = done;
    tl[3] = waited_ns;
    tl[2 + p.T] = globaltimer();
  }
}

template <int kEngine, int kThreads>
__global__ void __launch_bounds__(kThreads, 1) a2a_chain_kernel(const KParams p) {
  const uint32_t epoch = begin_epoch(p);
  chain_body<kEngine, kThreads>(p, epoch);
  end_epoch(p, epoch);
}

static int cuda_fail(cudaError_t e, const char* what) {
  char buf[256];
  snprintf(buf, sizeof buf, "%s: %s", what, cudaGetErrorString(e));
  return fail(A2A_ERR_CUDA, buf);
}

#define CK(call)                                   \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// copy engines: 0 = SM load/store (LDG.128/STG.128), 1 = TMA bulk copies (UBLKCP)
struct EngineCfg {
  const void* fn;
  int threads;
  size_t smem;
  int stages, prog_off, batch_off, batch;
  int ll_off = 0;   // LL128 per-warp gather buffers
};
static EngineCfg engine_cfg(const Plan& P) {
  const int TE = P.T_exec;
  if (P.sched_mode >= 1) {
    const bool rq = P.sched_mode == 5, ch = P.sched_mode >= 7;
    if (P.engine == 1) {
      int S = P.tma_stages;
      while (S > 1 && ((20 * (size_t)S + 127) & ~(size_t)127) + (size_t)S * P.tma_chunk > 220 * 1024) --S;
      const size_t ring = ((20 * (size_t)S + 127) & ~(size_t)127) + (size_t)S * P.tma_chunk;
      return {ch ? (const void*)a2a_chain_kernel<1, 256>
                 : rq ? (const void*)a2a_ready_kernel<1, 256> : (const void*)a2a_dyn_kernel<1, 256>,
              256, ring, S, 0, 0, 0};
    }
    return {ch ? (const void*)a2a_chain_kernel<0, 1024>
               : rq ? (const void*)a2a_ready_kernel<0, 1024> : (const void*)a2a_dyn_kernel<0, 1024>,
            1024, 0, 0, 0, 0, 0};
  }
  const size_t prog = ((size_t)TE * sizeof(CtaStep) + 127) & ~(size_t)127;
  if (P.engine == 1) {
    const int batch = 64;
    const size_t fixed = prog + batch * sizeof(DevPiece) + 1024 + (P.ll128 ? 8 * 640 : 0);
    int S = P.tma_stages;
    while (S > 1 && ((20 * (size_t)S + 127) & ~(size_t)127) + (size_t)S * P.tma_chunk + fixed >
                        227 * 1024)
      --S;
    const size_t ring = ((20 * (size_t)S + 127) & ~(size_t)127) + (size_t)S * P.tma_chunk;
    const size_t po = (ring + 127) & ~(size_t)127;
    const size_t ll = P.ll128 ? (256 / 32) * 640 : 0;
    return {(const void*)a2a_exec_kernel<1, 256>, 256, po + prog + batch * sizeof(DevPiece) + ll, S,
            (int)po, (int)(po + prog), batch, (int)(po + prog + batch * sizeof(DevPiece))};
  }
  const int batch = 128;
  if (P.ll128) {  // LL128: 512 threads with 128 registers each keep 16 lines per warp in flight
    const size_t ll = (512 / 32) * 640;
    return {(const void*)a2a_exec_kernel<0, 512>, 512, prog + batch * sizeof(DevPiece) + ll, 0, 0,
            (int)prog, batch, (int)(prog + batch * sizeof(DevPiece))};
  }
  return {(const void*)a2a_exec_kernel<0, 1024>, 1024, prog + batch * sizeof(DevPiece), 0, 0,
          (int)prog, batch, 0};
}

// arena flag region: entry[G] u32 | grab counters u64 @128 | flags @256:
//   static: [T'][G][nC] u32 (slot (t, gpu, cta)); dynamic: [total units] u32
static inline int64_t entry_flags_off() { return 0; }
static inline int64_t grab_off() { return 128; }
static inline int64_t step_flags_off() { return 256; }
static inline int64_t flag_region_bytes(int64_t n_flags) {
  return (step_flags_off() + n_flags * 4 + 65535) & ~65535LL;
}

static inline int64_t recv_stride(const Plan& P, int g) {
  return (P.info[g].recv_bytes + 4095) & ~4095LL;
}

static void free_device(Plan& P) {
  if (P.device < 0) return;
  DeviceGuard dg(P.device);
  for (int g = 0; g < A2A_MAX_GPUS; ++g) {
    if (P.peer_opened[g] && P.peer_arena[g]) cudaIpcCloseMemHandle(P.peer_arena[g]);
    P.peer_opened[g] = false;
    P.peer_arena[g] = nullptr;
  }
  void** bufs[] = {&P.arena, &P.d_items, &P.d_step_begin, &P.d_step_bytes, &P.d_dst_mask, &P.d_exit_idx,
                   &P.d_wait_off, &P.d_wait_idx, &P.d_counters, &P.d_timeline, &P.d_ctl};
  for (void** b : bufs) {
    if (*b) cudaFree(*b);
    *b = nullptr;
  }
  if (P.h_err) cudaFreeHost(P.h_err);
  P.h_err = nullptr;
  P.d_err = nullptr;
  P.bound = P.imported = false;
}

template <typename T>
static int upload(void** dst, const std::vector<T>& v) {
  size_t bytes = std::max<size_t>(v.size() * sizeof(T), 16);
  CK(cudaMalloc(dst, bytes));
  if (!v.empty()) CK(cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return A2A_OK;
}

static int bind_plan(Plan& P, int gpu, int dev, int nC) {
  if (gpu < 0 || gpu >= P.G) return fail(A2A_ERR_INVALID, "gpu rank out of range");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (dev < 0 || dev >= ndev) return fail(A2A_ERR_INVALID, "device ordinal out of range");
  DeviceGuard dg(dev);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major < 10) return fail(A2A_ERR_CUDA, "this library is built for sm_100a (B200) only");
  int coop = 0;
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) return fail(A2A_ERR_CUDA, "device does not support cooperative launch");
  const EngineCfg ec = engine_cfg(P);
  P.nT = ec.threads;
  if (ec.smem > 48 * 1024)
    CK(cudaFuncSetAttribute(ec.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ec.smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ec.fn, P.nT, ec.smem));
  const int max_ctas = per_sm * prop.multiProcessorCount;
  if (nC <= 0) nC = prop.multiProcessorCount;
  if (nC > max_ctas) return fail(A2A_ERR_INVALID, "num_ctas exceeds co-resident capacity");
  P.rank = gpu;
  P.device = dev;
  P.nC = nC;
  {  // experiments only: plain launch (co-residency then rests on 1 CTA/SM and an idle GPU)
    const char* nc = getenv("A2A_NONCOOP");
    P.coop = !(nc && nc[0] == '1');
  }
  const int G = P.G, TE = P.T_exec;

  // ---- CTA split + producer dependency lists (host, identical on all ranks)
  int rc = P.sched_mode >= 1 ? build_dyn(P, nC, P.dyn_unit_bytes) : build_sync(P, nC);
  if (rc != A2A_OK) return rc;
  const SyncTables& S = P.sync;
  const DynTables& Dy = P.dyn;

  // ---- arena layout, identical on every rank: flags | recv | scratch
  // ready mode: per-unit u64 completion counters + u64 queue slots (4 u32 each)
  P.flags_bytes = flag_region_bytes(P.sched_mode == 5  ? 4 * (int64_t)Dy.max_units
                                    : P.sched_mode >= 1 ? (int64_t)Dy.unit_base[G]
                                                        : (int64_t)TE * G * nC);
  P.recv_off.assign(G, 0);
  P.scratch_off.assign(G, 0);
  P.arena_bytes.assign(G, 0);
  for (int g = 0; g < G; ++g) {
    P.recv_off[g] = P.flags_bytes;
    P.scratch_off[g] = P.recv_off[g] + (int64_t)P.n_recv * recv_stride(P, g);
    P.arena_bytes[g] = P.scratch_off[g] + P.info[g].scratch_bytes;
  }
  cudaError_t e = cudaMalloc(&P.arena, (size_t)P.arena_bytes[gpu]);
  if (e != cudaSuccess) {
    P.arena = nullptr;
    char buf[200];
    snprintf(buf, sizeof buf, "cannot allocate %.3f GiB device arena: %s",
             P.arena_bytes[gpu] / 1073741824.0, cudaGetErrorString(e));
    return fail(A2A_ERR_NOMEM, buf);
  }
  CK(cudaMemset(P.arena, 0, (size_t)P.flags_bytes));
  if (P.ll && P.ll_half[gpu] > 0)  // LL lines: epoch 0 never matches
    CK(cudaMemset((char*)P.arena + P.scratch_off[gpu] + P.ll_off[gpu], 0, (size_t)(2 * P.ll_half[gpu])));
  if (P.sched_mode >= 1) {
    if ((rc = upload(&P.d_items, Dy.units[gpu])) != A2A_OK) return rc;
    if (P.sched_mode >= 7 && (rc = upload(&P.d_step_begin, Dy.chain_begin[gpu])) != A2A_OK) return rc;
    if ((rc = upload(&P.d_wait_idx, P.sched_mode == 5 ? Dy.deps_out[gpu] : Dy.wait_idx[gpu])) != A2A_OK)
      return rc;
    if ((rc = upload(&P.d_exit_idx, Dy.exit_idx[gpu])) != A2A_OK) return rc;
  } else {
    if ((rc = upload(&P.d_items, S.pieces[gpu])) != A2A_OK) return rc;
    if ((rc = upload(&P.d_step_begin, S.prog[gpu])) != A2A_OK) return rc;
    if ((rc = upload(&P.d_wait_idx, S.wait_idx[gpu])) != A2A_OK) return rc;
    if ((rc = upload(&P.d_exit_idx, S.exit_idx[gpu])) != A2A_OK) return rc;
  }
  CK(cudaMalloc(&P.d_ctl, (size_t)nC * 4));
  CK(cudaMemset(P.d_ctl, 0, (size_t)nC * 4));
  CK(cudaMalloc(&P.d_timeline, (size_t)nC * (2 * TE + 3) * 8));
  CK(cudaMemset(P.d_timeline, 0, (size_t)nC * (2 * TE + 3) * 8));
  size_t cbytes = std::max<size_t>((size_t)TE * std::max(P.E, 1) * 8, 16);
  CK(cudaMalloc(&P.d_counters, cbytes));
  CK(cudaMemset(P.d_counters, 0, cbytes));
  CK(cudaHostAlloc((void**)&P.h_err, 64, cudaHostAllocMapped | cudaHostAllocPortable));
  *P.h_err = 0;
  CK(cudaHostGetDevicePointer((void**)&P.d_err, P.h_err, 0));
  P.peer_arena[gpu] = P.arena;
  P.bound = true;
  P.imported = (G == 1);
  return A2A_OK;
}

}  // namespace a2a

using namespace a2a;

extern "C" {

int a2a_plan_destroy(a2a_plan* plan) {
  return guard([&]() -> int {
    if (!plan) return A2A_OK;
    if (plan->p.launched && plan->p.device >= 0) {
      DeviceGuard dg(plan->p.device);
      cudaDeviceSynchronize();
    }
    free_device(plan->p);
    delete plan;
    return A2A_OK;
  });
}

int a2a_plan_bind(a2a_plan* plan, int32_t gpu, int32_t device_ordinal, int32_t num_ctas) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "plan already bound");
    int rc = bind_plan(plan->p, gpu, device_ordinal, num_ctas);
    if (rc != A2A_OK) {
      std::string msg = a2a_last_error();
      free_device(plan->p);
      set_error(msg);
    }
    return rc;
  });
}

int a2a_plan_export_handle(const a2a_plan* plan, void* out_handle64) {
  return guard([&]() -> int {
    if (!plan || !out_handle64) return fail(A2A_ERR_INVALID, "null argument");
    if (!plan->p.bound) return fail(A2A_ERR_STATE, "plan not bound");
    DeviceGuard dg(plan->p.device);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, plan->p.arena));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
    std::memcpy(out_handle64, &h, 64);
    return A2A_OK;
  });
}

int a2a_plan_import_handles(a2a_plan* plan, const void* handles) {
  return guard([&]() -> int {
    if (!plan || !handles) return fail(A2A_ERR_INVALID, "null argument");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    if (P.imported && P.G > 1) return fail(A2A_ERR_STATE, "peer handles already imported");
    DeviceGuard dg(P.device);
    for (int g = 0; g < P.G; ++g) {
      if (g == P.rank) continue;
      cudaIpcMemHandle_t h;
      std::memcpy(&h, (const char*)handles + 64 * g, 64);
      void* ptr = nullptr;
      CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      P.peer_arena[g] = ptr;
      P.peer_opened[g] = true;
    }
    P.imported = true;
    return A2A_OK;
  });
}

// single-process multi-GPU: peers' arenas given directly (peer access is enabled here)
int a2a_plan_import_pointers(a2a_plan* plan, void* const* arenas) {
  return guard([&]() -> int {
    if (!plan || !arenas) return fail(A2A_ERR_INVALID, "null argument");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    DeviceGuard dg(P.device);
    for (int g = 0; g < P.G; ++g) {
      if (g == P.rank) continue;
      cudaPointerAttributes attr;
      CK(cudaPointerGetAttributes(&attr, arenas[g]));
      if (attr.device != P.device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(attr.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
      P.peer_arena[g] = arenas[g];
      P.peer_opened[g] = false;
    }
    P.imported = true;
    return A2A_OK;
  });
}

int a2a_plan_close_peers(a2a_plan* plan) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    Plan& P = plan->p;
    if (!P.bound) return A2A_OK;
    DeviceGuard dg(P.device);
    if (P.launched) CK(cudaDeviceSynchronize());
    for (int g = 0; g < A2A_MAX_GPUS; ++g) {
      if (g == P.rank) continue;
      if (P.peer_opened[g] && P.peer_arena[g]) CK(cudaIpcCloseMemHandle(P.peer_arena[g]));
      P.peer_opened[g] = false;
      P.peer_arena[g] = nullptr;
    }
    P.imported = (P.G == 1);
    return A2A_OK;
  });
}

int a2a_plan_layout(const a2a_plan* plan, int64_t* out8) {
  return guard([&]() -> int {
    if (!plan || !out8) return fail(A2A_ERR_INVALID, "null argument");
    const Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    int64_t arena = 0;
    for (int64_t b : P.arena_bytes) arena += b;
    const int64_t v[8] = {P.nC, P.sched_mode, P.dyn_unit_bytes, P.n_recv, P.flags_bytes, arena,
                          P.engine, P.ll ? 1 : 0};
    std::memcpy(out8, v, sizeof v);
    return A2A_OK;
  });
}

int a2a_plan_arena(const a2a_plan* plan, void** out_ptr) {
  return guard([&]() -> int {
    if (!plan || !out_ptr) return fail(A2A_ERR_INVALID, "null argument");
    if (!plan->p.bound) return fail(A2A_ERR_STATE, "plan not bound");
    *out_ptr = plan->p.arena;
    return A2A_OK;
  });
}

int a2a_plan_recv_buffer(const a2a_plan* plan, void** out_ptr) {
  return guard([&]() -> int {
    if (!plan || !out_ptr) return fail(A2A_ERR_INVALID, "null argument");
    if (!plan->p.bound) return fail(A2A_ERR_STATE, "plan not bound");
    *out_ptr = (char*)plan->p.arena + plan->p.recv_off[plan->p.rank];
    return A2A_OK;
  });
}

int a2a_plan_recv_buffer_at(const a2a_plan* plan, int32_t index, void** out_ptr) {
  return guard([&]() -> int {
    if (!plan || !out_ptr) return fail(A2A_ERR_INVALID, "null argument");
    const Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    if (index < 0 || index >= P.n_recv) return fail(A2A_ERR_INVALID, "recv buffer index out of range");
    *out_ptr = (char*)P.arena + P.recv_off[P.rank] + (int64_t)index * recv_stride(P, P.rank);
    return A2A_OK;
  });
}

int a2a_plan_set_engine(a2a_plan* plan, int32_t engine, int32_t tma_chunk, int32_t tma_stages) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "set the copy engine before a2a_plan_bind");
    if (engine != 0 && engine != 1) return fail(A2A_ERR_INVALID, "engine must be 0 (LSU) or 1 (TMA)");
    if (engine == 1) {
      if (tma_chunk <= 0) tma_chunk = 32768;
      if (tma_stages <= 0) tma_stages = 6;
      if (tma_chunk % 16 || tma_chunk > (1 << 19) || tma_stages > 32 ||
          (size_t)tma_chunk * tma_stages > 220 * 1024)
        return fail(A2A_ERR_INVALID, "bad TMA ring (chunk % 16, chunk*stages <= 220 KiB)");
      plan->p.tma_chunk = tma_chunk;
      plan->p.tma_stages = tma_stages;
    }
    plan->p.engine = engine;
    plan->p.dyn = DynTables{};   // chain links depend on the TMA ring size
    return A2A_OK;
  });
}

int a2a_plan_set_recv_buffers(a2a_plan* plan, int32_t count) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "set the recv buffer count before a2a_plan_bind");
    if (count < 1 || count > 4) return fail(A2A_ERR_INVALID, "recv buffer count must be 1..4");
    plan->p.n_recv = count;
    return A2A_OK;
  });
}

int a2a_plan_set_sync_mode(a2a_plan* plan, int32_t mode) {
  return guard([&]() -> int {
    if (!plan || mode < 0 || mode > 255) return fail(A2A_ERR_INVALID, "bad sync mode");
    // bit 7 breaks the all-to-all on purpose (mutation self-test): tests only
    const char* mut = getenv("A2A_ALLOW_MUTATION");
    if ((mode & kSyncNoWaits) && !(mut && mut[0] == '1'))
      return fail(A2A_ERR_INVALID, "bad sync mode: bit 7 (skipped waits) needs A2A_ALLOW_MUTATION=1");
    plan->p.sync_mode = mode;
    return A2A_OK;
  });
}

int a2a_plan_set_timeout(a2a_plan* plan, int64_t timeout_ns) {
  return guard([&]() -> int {
    if (!plan || timeout_ns <= 0) return fail(A2A_ERR_INVALID, "bad argument");
    plan->p.timeout_ns = timeout_ns;
    return A2A_OK;
  });
}

int a2a_plan_execute(a2a_plan* plan, const void* send, void* recv, void* stream, int32_t options) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound to a device");
    if (!P.imported) return fail(A2A_ERR_STATE, "peer arenas not imported");
    if (*P.h_err != 0) return fail(*P.h_err, "a previous execute failed on the device (timeout)");
    char* own_recv = (char*)P.arena + P.recv_off[P.rank];
    if (!recv) recv = own_recv;
    int32_t ridx = 0;
    if (P.G > 1 && !P.ll) {
      const int64_t st = recv_stride(P, P.rank);
      ridx = -1;
      for (int i = 0; i < P.n_recv; ++i)
        if ((char*)recv == own_recv + i * st) ridx = i;
      if (ridx < 0)
        return fail(A2A_ERR_INVALID, "multi-GPU plans must receive into an arena recv buffer");
    }
    if (!send && P.info[P.rank].send_bytes > 0) return fail(A2A_ERR_INVALID, "null send buffer");
    DeviceGuard dg(P.device);
    KParams kp;
    std::memset(&kp, 0, sizeof kp);
    kp.base[loc_send()] = (char*)send;
    for (int g = 0; g < P.G; ++g) {
      char* ar = (char*)P.peer_arena[g];
      kp.base[loc_recv(g)] =
          (g == P.rank) ? (char*)recv : ar + P.recv_off[g] + (int64_t)ridx * recv_stride(P, g);
      kp.base[loc_scratch(g, P.G)] = ar + P.scratch_off[g];
      if (P.ll) {  // parity 0; the kernel adds (epoch & 1) * ll_half
        kp.base[loc_ll(g, P.G)] = ar + P.scratch_off[g] + P.ll_off[g];
        kp.ll_half[g] = P.ll_half[g];
      }
      kp.entry_flags[g] = (uint32_t*)(ar + entry_flags_off());
      kp.step_flags[g] = (uint32_t*)(ar + step_flags_off());
    }
    kp.pieces = (const DevPiece*)P.d_items;
    kp.prog = (const CtaStep*)P.d_step_begin;
    kp.exit_idx = (const int32_t*)P.d_exit_idx;
    if (P.sched_mode >= 1) {
      const DynTables& Dy = P.dyn;
      kp.n_exit = (int32_t)Dy.exit_idx[P.rank].size();
      kp.units = (const DevUnit*)P.d_items;
      kp.unit_wait = (const int32_t*)P.d_wait_idx;
      kp.n_units = (int32_t)Dy.units[P.rank].size();
      kp.unit_base = Dy.unit_base[P.rank];
      kp.grab = (unsigned long long*)((char*)P.arena + grab_off());
      if (P.sched_mode == 5) {
        for (int g = 0; g < P.G; ++g) {
          char* ar = (char*)P.peer_arena[g];
          kp.qctl[g] = (unsigned long long*)(ar + grab_off());
          kp.qdone[g] = (unsigned long long*)(ar + step_flags_off());
          kp.qslot[g] = (unsigned long long*)(ar + step_flags_off() + 8 * (int64_t)Dy.max_units);
        }
        for (int g = 0; g <= P.G; ++g) kp.ubase[g] = Dy.unit_base[g];
        kp.n_init = Dy.n_init[P.rank];
        kp.n_into = Dy.n_into[P.rank];
      }
      if (P.sched_mode >= 7) {
        kp.chain_begin = (const int32_t*)P.d_step_begin;
        kp.n_tasks = (int32_t)Dy.chain_begin[P.rank].size() - 1;
        kp.chain_discard = P.sched_mode == 8 ? 1 : 0;
      }
      kp.n_remote = Dy.n_remote[P.rank];
      kp.remote_ctas = Dy.remote_ctas[P.rank];
      kp.pin_queues = Dy.pin;
    } else {
      kp.n_exit = (int32_t)P.sync.exit_idx[P.rank].size();
    }
    kp.wait_idx = (const int32_t*)P.d_wait_idx;
    kp.counters = (unsigned long long*)P.d_counters;
    kp.err = P.d_err;
    kp.timeout_ns = P.timeout_ns;
    kp.ctl = (uint32_t*)P.d_ctl;
    kp.ll = P.ll ? 1 : 0;
    kp.ll128 = P.ll128 ? 1 : 0;
    kp.G = P.G;
    kp.rank = P.rank;
    kp.nC = P.nC;
    kp.T = P.T_exec;
    kp.E = P.E;
    kp.count_links = (options & A2A_EXEC_COUNT_LINKS) ? 1 : 0;
    void* args[] = {&kp};
    kp.timeline = (unsigned long long*)P.d_timeline;
    kp.sync_mode = P.sync_mode;
    const EngineCfg ec = engine_cfg(P);
    kp.tma_chunk = P.tma_chunk;
    kp.tma_stages = ec.stages;
    kp.smem_prog = ec.prog_off;
    kp.smem_batch = ec.batch_off;
    kp.batch = ec.batch;
    kp.smem_ll = ec.ll_off;
    // cooperative launch (all CTAs co-resident: CTAs spin on each other's flags);
    // cudaLaunchKernelExC with the cooperative attribute is stream-capturable
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.nC);
    cfg.blockDim = dim3(ec.threads);
    cfg.dynamicSmemBytes = ec.smem;
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = P.coop ? 1 : 0;
    cudaError_t e = cudaLaunchKernelExC(&cfg, ec.fn, args);
    if (e != cudaSuccess) return cuda_fail(e, "cudaLaunchKernelExC (cooperative)");
    P.last_stream = stream;
    P.launched = true;
    return A2A_OK;
  });
}

int a2a_plan_sync(a2a_plan* plan) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    DeviceGuard dg(P.device);
    CK(cudaStreamSynchronize((cudaStream_t)P.last_stream));
    if (*P.h_err != 0) {
      return fail(*P.h_err, "device-side flag wait timed out (a peer did not arrive)");
    }
    return A2A_OK;
  });
}

int a2a_plan_read_timeline(a2a_plan* plan, uint64_t* out, int32_t* out_cols) {
  return guard([&]() -> int {
    if (!plan || !out_cols) return fail(A2A_ERR_INVALID, "null argument");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    *out_cols = 2 * P.T_exec + 3;
    if (!out) return A2A_OK;
    DeviceGuard dg(P.device);
    CK(cudaStreamSynchronize((cudaStream_t)P.last_stream));
    CK(cudaMemcpy(out, P.d_timeline, (size_t)P.nC * (2 * P.T_exec + 3) * 8, cudaMemcpyDeviceToHost));
    return A2A_OK;
  });
}

int a2a_plan_read_link_counters(a2a_plan* plan, int64_t* out) {
  return guard([&]() -> int {
    if (!plan || !out) return fail(A2A_ERR_INVALID, "null argument");
    Plan& P = plan->p;
    if (!P.bound) return fail(A2A_ERR_STATE, "plan not bound");
    DeviceGuard dg(P.device);
    CK(cudaDeviceSynchronize());
    size_t cnt = (size_t)P.T * P.E;
    if (cnt) {
      CK(cudaMemcpy(out, P.d_counters, cnt * 8, cudaMemcpyDeviceToHost));
      CK(cudaMemset(P.d_counters, 0, cnt * 8));
    }
    return A2A_OK;
  });
}

}  // extern "C"
