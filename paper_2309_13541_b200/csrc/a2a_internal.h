// Internal plan representation shared by the host plan builder (a2a_plan.cpp)
// and the device side (a2a_exec.cu).  Not part of the C ABI.
#pragma once

#include <cstdint>
#include <exception>
#include <new>
#include <string>
#include <vector>

#include "a2a_exec.h"

#define A2A_MAX_GPUS 8

#ifdef __CUDACC__
#define A2A_HD __host__ __device__ __forceinline__
#else
#define A2A_HD inline
#endif

namespace a2a {

// Buffer classes a copy item reads from / writes to.  The pointer table of a
// launch is [send(local) | recv(gpu 0..G-1) | scratch(gpu 0..G-1) |
// LL landing region of this execute's epoch parity (gpu 0..G-1)].
inline int loc_send() { return 0; }
inline int loc_recv(int gpu) { return 1 + gpu; }
inline int loc_scratch(int gpu, int G) { return 1 + G + gpu; }
inline int loc_ll(int gpu, int G) { return 1 + 2 * G + gpu; }

// piece kinds (bits): kLLDst = the destination is LL lines of a landing region,
// kLLSrc = the source is LL lines (polled until they carry the epoch); LL
// offsets are payload addresses: payload byte x of a region lives in line x/8
// (bytes 16*(x/8) .. +16).  kDecode marks a same-step decode of remote lines
// into recv (ordering only: last in its step).
enum : int32_t { kCopy = 0, kLLDst = 1, kLLSrc = 2, kDecode = 4 };

// One contiguous byte copy of one hop-op (or self-shard copy), 48 bytes.
struct DevItem {
  int64_t src_off;   // byte offset inside base[src_loc]
  int64_t dst_off;   // byte offset inside base[dst_loc]
  int64_t nbytes;
  int64_t prefix;    // start of this item in the step's concatenated byte space
  int32_t src_loc;
  int32_t dst_loc;
  int32_t edge;      // schedule edge id (-1: self-shard copy, not a link)
  int16_t dst_gpu;
  int16_t kind;      // kCopy or kLLDst / kLLSrc / kDecode bits
};
static_assert(sizeof(DevItem) == 48, "DevItem layout");

// Per-GPU execution tables: items of every step, steps concatenated.
struct GpuTables {
  std::vector<DevItem> items;
  std::vector<int64_t> step_begin;  // [T'+1] item index ranges
  std::vector<int64_t> step_bytes;  // [T']
};

// CTA split + exact producer dependencies for a given CTA count (host-built,
// identical on every rank).  Flag slot of producer (t, g, c) = (t*G + g)*nC + c
// in every GPU's step-flag array.
// One CTA's copy piece (a contiguous sub-range of one item), 32 bytes.
struct DevPiece {
  int64_t src_off, dst_off;
  int32_t nbytes;
  int32_t edge;
  int16_t src_loc, dst_loc;
  int32_t kind;      // kCopy or kLLDst / kLLSrc / kDecode bits
};
static_assert(sizeof(DevPiece) == 32, "DevPiece layout");

// One CTA's program for one step, 32 bytes: piece range, wait-list range,
// destination-GPU mask of its stores.
struct CtaStep {
  int32_t pb, pe;   // [pb, pe) in the GPU's piece array
  int32_t wb, we;   // [wb, we) in the GPU's wait_idx array
  uint32_t mask;    // GPUs written in this step (flags to publish)
  int32_t pad[3];
};
static_assert(sizeof(CtaStep) == 32, "CtaStep layout");

struct SyncTables {
  int32_t nC = 0;
  int32_t weight = 0;                           // remote_weight the split was built with
  std::vector<std::vector<DevPiece>> pieces;    // [g] ordered by (cta, step)
  std::vector<std::vector<CtaStep>> prog;       // [g][c*T' + t]
  std::vector<std::vector<uint32_t>> dst_mask;  // [g][t*nC + c] bit h: (g,c) wrote to h at t
  std::vector<std::vector<int32_t>> wait_off;   // [g][t*nC + c .. +1] into wait_idx[g]
  std::vector<std::vector<int32_t>> wait_idx;   // [g] producer slots to acquire
  std::vector<std::vector<int32_t>> exit_idx;   // [g] every producer slot that writes into g
};

// Dynamic mode: one unit of work = a contiguous sub-range of
// one item; CTAs grab units in list order from a per-GPU atomic counter.
struct DevUnit {
  int64_t src_off, dst_off;
  int32_t nbytes;
  int32_t edge;
  int16_t src_loc, dst_loc;
  int32_t wb, we;     // [wb, we) in the GPU's unit wait list
  uint32_t mask;      // GPUs whose flag array receives this unit's flag
  int32_t step;
};
static_assert(sizeof(DevUnit) == 48, "DevUnit layout");

struct DynTables {
  int32_t nC = 0;
  int64_t unit_bytes = 0;                       // target unit size (0 = auto)
  std::vector<int32_t> unit_base;               // [G+1] global unit id = base[g] + index
  std::vector<std::vector<DevUnit>> units;      // [g] grab order: remote queue, then local queue
  std::vector<int32_t> n_remote;                // [g] units in the remote (NVLink) queue
  std::vector<int32_t> remote_ctas;             // [g] CTAs that start on the remote queue
  int32_t pin = 0;                              // CTAs never switch queues (a2a_plan_set_queue_split)
  std::vector<std::vector<int32_t>> wait_idx;   // [g] global unit ids to acquire
  std::vector<std::vector<int32_t>> exit_idx;   // [g] global unit ids flagged into g
  double est_makespan = 0;                      // host model estimate (s)
  // ready-queue mode (sched_mode 5): per unit its dependents as {global id,
  // in-degree} pairs (DevUnit.wb/we index pairs, DevUnit.mask = own in-degree)
  std::vector<std::vector<int32_t>> deps_out;   // [g] flattened pairs
  std::vector<int32_t> n_init, n_into;          // [g] units ready at start; units writing into g
  int32_t max_units = 0;                        // max units on one GPU (queue array size)
  // chain mode (sched_mode 7): per GPU, task k = units [chain_begin[k], chain_begin[k+1])
  // of that GPU's unit array, run in order by one CTA
  std::vector<std::vector<int32_t>> chain_begin;
  int32_t max_chain = 0;                        // longest task (units)
};

struct Interval {
  int32_t a, b;       // chunk range [a, b)
  int64_t base;       // scratch byte offset of chunk a's first byte
};

struct Plan {
  // ---- descriptor copy
  int32_t n = 0, T = 0, Q = 1, E = 0, G = 1, flags = 0;
  int64_t m = 0;
  std::vector<int32_t> edge_uv;
  std::vector<double> cap;
  std::vector<a2a_op> ops;
  std::vector<std::vector<int64_t>> step_ops;   // op indices per step, list order
  std::vector<int32_t> node_gpu, local_idx;
  int32_t T_exec = 1;                           // max(T, 1): self copies need a step
  bool reuse = false;                           // scratch liveness reuse (A2A_REUSE_SCRATCH)
  bool ll = false;                              // low-latency cross-GPU transport (A2A_PROTO_LL)
  bool ll128 = false;                           // ... with 128-byte lines (A2A_PROTO_LL128)
  int64_t gran = 64;                            // CTA piece boundaries: multiples of gran item bytes
  std::vector<int64_t> ll_off, ll_half;         // per gpu: landing region in scratch, bytes per parity

  // ---- layout / tables (host)
  std::vector<a2a_gpu_info> info;               // per gpu
  std::vector<GpuTables> tables;                // per gpu
  std::vector<int64_t> link_bytes;              // [T * E]

  SyncTables sync;
  DynTables dyn;
  int32_t remote_weight = 1;                    // CTA split cost of an NVLink byte vs a local byte
  int32_t sched_mode = 0;                       // 0 static programs, 1..6 unit queues, 7 chains (8: + L2 discard)
  int64_t dyn_unit_bytes = 0;                   // dynamic unit size (0 = auto)
  int32_t dyn_remote_ctas = 0;                  // CTAs pinned to the NVLink queue (0 = auto split)

  // ---- device binding (a2a_exec.cu)
  bool bound = false, imported = false;
  int32_t rank = -1, device = -1, nC = 0, nT = 1024;
  int32_t engine = 1, tma_chunk = 32768, tma_stages = 6;   // copy engine (a2a_plan_set_engine; LSU for LL)
  int32_t n_recv = 1;                           // arena recv buffers (multi-buffering)
  int32_t sync_mode = 2;                        // a2a_plan_set_sync_mode (2: bar.sync + st.release)
  bool coop = true;                             // cooperative launch (A2A_NONCOOP=1: plain, experiments)
  int64_t flags_bytes = 0;                      // arena flag region size
  std::vector<int64_t> recv_off, scratch_off;   // per gpu, inside that gpu's arena
  std::vector<int64_t> arena_bytes;             // per gpu
  void* arena = nullptr;                        // own arena (cudaMalloc)
  void* peer_arena[A2A_MAX_GPUS] = {nullptr};   // mapped arenas (own included)
  bool peer_opened[A2A_MAX_GPUS] = {false};     // opened via IPC (must close)
  void* d_items = nullptr;
  void* d_step_begin = nullptr;
  void* d_step_bytes = nullptr;
  void* d_dst_mask = nullptr;
  void* d_exit_idx = nullptr;
  void* d_wait_off = nullptr;
  void* d_wait_idx = nullptr;
  void* d_counters = nullptr;
  void* d_timeline = nullptr;
  void* d_ctl = nullptr;                        // [nC] u32 per-CTA epoch (device-side, graph-safe)
  int32_t* h_err = nullptr;                     // mapped pinned error word
  int32_t* d_err = nullptr;
  int64_t timeout_ns = 10000000000LL;
  void* last_stream = nullptr;
  bool launched = false;
};

// LL line geometry: payload bytes per line / line bytes.  A2A_PROTO_LL: 8 / 16
// ({4 B data, epoch, 4 B data, epoch}); A2A_PROTO_LL128: 120 / 128 (payload,
// then the 8-byte epoch flag).  LL offsets are payload addresses.
constexpr int64_t kLL128Payload = 120, kLL128Line = 128;
inline int64_t ll_payload(bool ll128) { return ll128 ? kLL128Payload : 8; }
inline int64_t ll_line(bool ll128) { return ll128 ? kLL128Line : 16; }
// byte of the landing region holding payload address x
inline int64_t ll_byte(bool ll128, int64_t x) {
  if (ll128) return kLL128Line * (x / kLL128Payload) + x % kLL128Payload;
  return 16 * (x >> 3) + ((x & 7) < 4 ? (x & 7) : (x & 7) + 4);
}

// chunk c of an m-byte shard split in Q chunks starts at floor(c*m/Q)
inline int64_t chunk_off(int64_t c, int64_t m, int64_t Q) {
  return (int64_t)(((__int128)c * m) / Q);
}

void set_error(const std::string& msg);
int build_sync(Plan& P, int nC);
int build_dyn(Plan& P, int nC, int64_t unit_bytes);
int simulate(Plan& P, int nC, const a2a_sim_params& prm, double* makespan_s);
int fail(int code, const std::string& msg);

// Every extern "C" entry point runs its body through guard(): no C++
// exception crosses the C ABI (allocation failure -> A2A_ERR_NOMEM, anything
// else -> A2A_ERR_INVALID with the exception text).
template <class F>
int guard(F&& body) noexcept {
  try {
    return body();
  } catch (const std::bad_alloc&) {
    return fail(A2A_ERR_NOMEM, "out of host memory");
  } catch (const std::exception& e) {
    return fail(A2A_ERR_INVALID, std::string("internal error: ") + e.what());
  } catch (...) {
    return fail(A2A_ERR_INVALID, "internal error");
  }
}

// CTA work split shared by host (flag lists) and device (copy ranges)
A2A_HD int64_t cta_lo(int64_t B, int c, int nC) {
  if (c >= nC) return B;
  int64_t x = (int64_t)(((__int128)B * c) / nC);
  return x & ~(int64_t)63;
}

}  // namespace a2a

struct a2a_plan {
  a2a::Plan p;
};
