/*
 * a2a_exec.h — C ABI of the B200 executor for lowered all-to-all schedules.
 *
 * This library takes the slot of the reference's CPU executor
 *   a2aflow.evaluate.replay_timestep_schedule(g, sched, m, b, sync_latency)
 *   (reference pkg/src/a2aflow/evaluate.py:56-127)
 * and actually moves the bytes: every instruction (t, src, dst, s, d, c0, c1)
 * of a mode="ts" ChunkedSchedule (reference pkg/src/a2aflow/schedule.py:49-72)
 * copies bytes [floor(c0*m/Q), floor(c1*m/Q)) of shard (s,d) from node src's
 * buffer to node dst's buffer, hop by hop, on sm_100a kernels; virtual nodes
 * placed on other GPUs are reached with direct NVLink peer stores, steps are
 * ordered with system-scope release/acquire flags, and no NCCL call is made.
 *
 * The reference has no FFI for this path (it is pure Python); the entry points
 * below are what its evaluate.replay_timestep_schedule call site would bind
 * (see INTEGRATION.md for the ctypes stub).  Conventions:
 *   - plain C types only; no C++ exceptions cross the boundary;
 *   - every call returns an a2a_status (0 = OK); on failure the message is in
 *     a2a_last_error() (thread-local).  A rejected schedule returns
 *     A2A_ERR_EVAL with exactly the reference's EvalError text
 *     (evaluate.py:70-73, :91-100, :114-126);
 *   - a plan is not thread-safe; one execute in flight per plan.
 */
#ifndef A2A_EXEC_H
#define A2A_EXEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  A2A_OK = 0,
  A2A_ERR_INVALID = 1, /* bad argument / descriptor                       */
  A2A_ERR_EVAL = 2,    /* schedule rejected; text == reference EvalError  */
  A2A_ERR_CUDA = 3,    /* CUDA runtime error                              */
  A2A_ERR_TIMEOUT = 4, /* a device-side flag wait timed out (peer missing)*/
  A2A_ERR_STATE = 5,   /* call order violated (e.g. execute before bind)  */
  A2A_ERR_NOMEM = 6    /* device or host allocation failed                */
} a2a_status;

/* == schedule.Instruction (reference pkg/src/a2aflow/schedule.py:49-62), mode "ts" */
typedef struct {
  int32_t t, src, dst, s, d, c0, c1;
} a2a_op;

/* descriptor flags */
#define A2A_COPY_SELF 1  /* also copy the self shard send[v][v] -> recv[v][v] */
#define A2A_INTERLEAVE 2 /* split items (split_bytes) and interleave destination GPUs */
#define A2A_REUSE_SCRATCH 4 /* liveness-based scratch reuse (+ WAR/WAW dependencies) */
/* Low-latency transport for cross-GPU hops (static schedule only; not with
 * A2A_INTERLEAVE or A2A_REUSE_SCRATCH): every byte bound for another GPU is
 * stored as 16-byte lines {4 data bytes, epoch, 4 data bytes, epoch} into an
 * epoch-parity double-buffered landing region of the destination GPU, where
 * that GPU's own CTAs poll the lines and write the bytes to their scratch /
 * recv destination.  No system-scope fence or flag on the path, all step flags
 * stay GPU-local, the entry barrier lags one all-to-all, and recv may be any
 * device buffer.  Twice the NVLink bytes: for small shards. */
#define A2A_PROTO_LL 8
/* LL128 variant of the low-latency transport (implies A2A_PROTO_LL): lines of
 * 128 bytes = 120 payload bytes + an 8-byte epoch flag, each line stored and
 * loaded as ONE warp instruction (8 lanes x 16 bytes), as NCCL's LL128 does
 * over NVLink.  1.07x the bytes instead of 2x: small-to-medium shards.  Relies
 * on a warp's 128-byte line store arriving as a unit (tools/ll128_stress.py
 * validates it on the hardware). */
#define A2A_PROTO_LL128 16

typedef struct {
  int32_t n_nodes;         /* Digraph.n (must equal ChunkedSchedule.n)      */
  int32_t n_steps;         /* ChunkedSchedule.nsteps                         */
  int32_t q;               /* ChunkedSchedule.Q                              */
  int32_t n_edges;         /* Digraph.num_edges                              */
  int64_t m_bytes;         /* shard size m (bytes, integer)                  */
  const int32_t* edge_uv;  /* [n_edges][2] Digraph.edges (u, v), edge id = index */
  const double* edge_cap;  /* [n_edges] capacities (only for the modelled T) */
  const a2a_op* ops;       /* instructions in list order                    */
  int64_t n_ops;
  const int32_t* node_gpu; /* [n_nodes] virtual node -> GPU rank; NULL = all on 0 */
  int32_t n_gpus;          /* >= 1                                           */
  int32_t flags;           /* A2A_COPY_SELF | A2A_INTERLEAVE | A2A_REUSE_SCRATCH | A2A_PROTO_LL[128] */
  int64_t split_bytes;     /* piece size for A2A_INTERLEAVE (0 = 256 KiB)    */
} a2a_schedule_desc;

typedef struct a2a_plan a2a_plan;

/* per-GPU shape of a plan (host-side, no device needed) */
typedef struct {
  int32_t n_local_nodes;   /* V_g: virtual nodes placed on this GPU          */
  int32_t first_node;      /* smallest node id on this GPU (-1 if none)      */
  int64_t send_bytes;      /* V_g * N * m: send buffer, [V_g][N][m] u8        */
  int64_t recv_bytes;      /* V_g * N * m: recv buffer, recv[v][s] = shard (s,v) */
  int64_t scratch_bytes;   /* forwarding scratch (+ LL landing region) here  */
  int64_t n_items;         /* copy items this GPU executes (all steps)       */
  int64_t hop_bytes;       /* bytes this GPU copies over schedule links      */
  int64_t egress_bytes;    /* of which to other GPUs (NVLink)                */
  int64_t ingress_bytes;   /* bytes other GPUs write into this GPU           */
  int64_t local_bytes;     /* hop bytes that stay on this GPU (+ self copies)*/
} a2a_gpu_info;

/* ---- native loader for the reference's on-disk formats (plain or .gz) ---- */
typedef struct {
  int32_t n, nsteps, q;
  int32_t mode;            /* 0 = "ts", 1 = "path" */
  double chunk_bytes;
} a2a_sched_header;
/* parse_schedule_xml (reference src/schedule.py:349-384): same rejects, the
 * ScheduleError texts come back as A2A_ERR_EVAL.  *ops is malloc'd: a2a_free. */
int a2a_load_schedule_xml(const char* path, a2a_sched_header* hdr, a2a_op** ops, int64_t* n_ops);
/* path-mode XML + `.routes.json` sidecar (reference src/cli.py:289-292) ->
 * hop-indexed mode="ts" ops (hop i at step i, ts sort key of schedule.py:237).
 * node_map (optional, length map_len) maps host-augmented ids to physical
 * nodes (collapse, n_phys nodes). */
int a2a_lower_path_files(const char* xml_path, const char* routes_path, const int32_t* node_map,
                         int32_t map_len, int32_t n_phys, a2a_sched_header* hdr, a2a_op** ops,
                         int64_t* n_ops);
/* binary op table (format in csrc/a2a_io.cpp): the
 * parsed schedule plus a SHA-256 trailer.  save rejects ops load_schedule_xml
 * would reject (A2A_ERR_EVAL, same texts) and writes atomically (tmp + rename);
 * load checks magic, size and digest (A2A_ERR_INVALID) and then the same op
 * rejects.  *ops from load is malloc'd: a2a_free. */
int a2a_save_schedule_table(const char* path, const a2a_sched_header* hdr, const a2a_op* ops,
                            int64_t n_ops);
int a2a_load_schedule_table(const char* path, a2a_sched_header* hdr, a2a_op** ops, int64_t* n_ops);
/* hex SHA-256 of a file (65 bytes incl. NUL), as the reference manifest's
 * _sha256 (reference src/cli.py:30-35) */
int a2a_sha256_file(const char* path, char* hex_out);
void a2a_free(void* p);

/* ---- plan construction: validation exactly like the reference replay ---- */
int a2a_plan_create(const a2a_schedule_desc* desc, a2a_plan** out);
int a2a_plan_destroy(a2a_plan* plan);
const char* a2a_last_error(void);
const char* a2a_version(void);

/* modelled store-and-forward time, bit-identical to replay_timestep_schedule's T
 * (evaluate.py:101-107) for the same (m, b, sync_latency) */
int a2a_plan_model_time(const a2a_plan* plan, double m, double b, double sync_latency,
                        double* out_T);
/* schedule bytes per (step, edge): out[t * n_edges + e] (int64, this plan's m) */
int a2a_plan_link_bytes(const a2a_plan* plan, int64_t* out);
int a2a_plan_gpu_info(const a2a_plan* plan, int32_t gpu, a2a_gpu_info* out);

/* CTA work split + exact producer dependency lists for `num_ctas` CTAs per GPU
 * (host only; a2a_plan_bind calls it).  Stats: flags each GPU acquires in total
 * and at exit. */
int a2a_plan_prepare(a2a_plan* plan, int32_t num_ctas);
int a2a_plan_sync_stats(const a2a_plan* plan, int32_t gpu, int64_t* n_wait, int64_t* n_exit);
/* Host emulation of the device protocol on host buffers (send[g], recv[g] per GPU
 * rank, same layout as on the device): CTAs of all GPUs run in a random
 * interleaving (xorshift `seed`) constrained only by the dependency lists.
 * Used by the CPU tests to prove the lists are sufficient. */
int a2a_plan_emulate(a2a_plan* plan, int32_t num_ctas, void* const* send, void* const* recv,
                     uint64_t seed);

/* Placement optimiser (host only): balanced virtual-node -> GPU assignment with
 * the same per-GPU node counts as `placement` (in/out), minimising the NVLink
 * term max_g max(egress_g, ingress_g) of the per-edge schedule bytes
 * (edge_bytes[e], e.g. a2a_plan_link_bytes summed over steps); exhaustive for
 * n <= 12, sampled best-improvement swaps otherwise (`iters` rounds). */
int a2a_optimize_placement(int32_t n, int32_t n_edges, const int32_t* edge_uv,
                           const int64_t* edge_bytes, int32_t n_gpus, int32_t iters,
                           uint64_t seed, int32_t* placement);

/* Host audit: every piece / unit of every GPU (for `num_ctas` CTAs and the
 * selected schedule) reads inside its source buffer on the executing GPU and
 * writes inside its destination buffer (the address-math part of memcheck). */
int a2a_plan_check_bounds(a2a_plan* plan, int32_t num_ctas);
/* Static CTA split, before bind: each step's items are cut into equal-cost CTA
 * ranges where a byte bound for another GPU costs `remote_weight` (1..64,
 * default 1) and a local byte 1. */
int a2a_plan_set_split(a2a_plan* plan, int32_t remote_weight);
/* Execution schedule, before bind: 0 = static per-CTA step programs (default),
 * 1 = dynamic units: items cut into units of `unit_bytes` (0 = auto), CTAs grab
 * units in step-major, readiness-ordered lists from a per-GPU atomic counter and
 * acquire per-unit producer flags; 2 = dynamic units ordered by
 * an event-driven list schedule (start times) instead of step-major, so routes
 * pipeline hop by hop at unit granularity; 3 = dynamic units, step-major with
 * critical-path (bottom-level) priority within a step; 4 = one queue per GPU,
 * step-major, NVLink and HBM units merged in proportion to their time; 5 = a
 * per-GPU ready queue: units are enqueued when their last producer finishes
 * (completion counters counted down with system-scope atomics); 6 = as 4, with
 * each step's NVLink units interleaved over their destination GPUs in
 * proportion to their bytes (no incast on one peer); 7 = chains: a unit whose
 * only producer is the previous local hop of the same route (same bytes, its
 * only consumer) runs right after it on the same CTA -- each task (a route's
 * consecutive local hops over one unit) streams through one TMA ring, the next
 * hop reading the previous hop's bytes back from L2, no flag between them;
 * 8 = as 7, and each task discards its dead intermediate scratch lines from L2
 * (discard.global.L2) instead of writing them back.
 * a2a_plan_emulate follows the
 * selected mode.  Stats: units and dependency entries of `gpu`, model makespan. */
int a2a_plan_set_schedule(a2a_plan* plan, int32_t mode, int64_t unit_bytes);
/* Queue split of the two-queue dynamic orders (1-3), before bind: `remote_ctas`
 * CTAs are pinned to the NVLink queue and the others to the HBM queue, and no
 * CTA switches queues (0 = automatic split, CTAs switch when their queue
 * drains).  Clamped so that every non-empty queue keeps at least one CTA. */
int a2a_plan_set_queue_split(a2a_plan* plan, int32_t remote_ctas);
/* Fluid performance model of one execute of the selected execution schedule
 * (static programs or dynamic orders 1-6; simple protocol) for `num_ctas`
 * CTAs per GPU: per-GPU NVLink egress and ingress (GB/s per direction), HBM
 * (read + write GB/s), a per-CTA copy-rate cap, a fixed cost per unit /
 * CTA-step, the flag latency and a launch cost.  Host only; for comparing
 * orders offline (e.g. at 8 GPUs). */
typedef struct {
  double nvlink_gbs, hbm_gbs, cta_gbs;
  double flag_us, unit_us, launch_us;
  double jitter;   /* per-CTA speed factor spread, e.g. 0.2 = +-20% */
  double unit_us_sys;  /* fixed cost per unit / CTA-step when G > 1 (system-scope
                          publication); unit_us applies at G = 1 */
  double incast;       /* NVLink ingress of a GPU that w CTAs (over all peers) write
                          into at once runs at nvlink_gbs / (1 + incast * max(0,
                          w / num_ctas - 1)); 0 = no penalty */
} a2a_sim_params;
int a2a_plan_simulate(a2a_plan* plan, int32_t num_ctas, const a2a_sim_params* params,
                      double* makespan_s);
int a2a_plan_dyn_stats(a2a_plan* plan, int32_t gpu, int32_t num_ctas, int64_t* n_units,
                       int64_t* n_wait, double* est_makespan_s);

/* ---- device side ---- */
/* Bind the plan to one GPU: rank `gpu` of the placement on CUDA device
 * `device_ordinal`, with `num_ctas` persistent CTAs (0 = one per SM).  Allocates
 * the device arena (flags | recv | scratch) and uploads this rank's tables.
 * num_ctas must be equal on all ranks of a multi-GPU plan. */
int a2a_plan_bind(a2a_plan* plan, int32_t gpu, int32_t device_ordinal, int32_t num_ctas);
/* 64-byte cudaIpcMemHandle of this rank's arena (multi-process, n_gpus > 1) */
int a2a_plan_export_handle(const a2a_plan* plan, void* out_handle64);
/* import all ranks' handles ([n_gpus][64] bytes, own entry ignored) */
int a2a_plan_import_handles(a2a_plan* plan, const void* handles);
/* single-process multi-GPU alternative to handles: every rank's arena pointer
 * (a2a_plan_arena), peer access is enabled on this rank's device */
int a2a_plan_arena(const a2a_plan* plan, void** out_ptr);
int a2a_plan_import_pointers(a2a_plan* plan, void* const* arenas);
/* multi-GPU teardown, phase 1: wait for this rank's executes, then close the
 * imported peer arenas (the plan refuses further executes).  Every rank must
 * reach phase 1 before any rank frees its own arena (a2a_plan_destroy): an
 * exported allocation must outlive its importers' mappings. */
int a2a_plan_close_peers(a2a_plan* plan);
/* after bind: the device-layout parameters every rank must agree on, as 8
 * int64 {num_ctas, sched_mode, dyn_unit_bytes, n_recv, flags_bytes,
 * arena_bytes of every GPU summed, engine, protocol LL} -- a rank that
 * computed a different layout would store to wrong offsets of its peers */
int a2a_plan_layout(const a2a_plan* plan, int64_t* out8);
/* pointer to this rank's arena recv buffer ([V_g][N][m]); with n_gpus > 1
 * peers store into it directly, so execute must be given this buffer (any
 * device buffer with A2A_PROTO_LL, where only local CTAs write recv) */
int a2a_plan_recv_buffer(const a2a_plan* plan, void** out_ptr);
/* before bind: number of arena recv buffers (1..4, default 1) so consecutive
 * all-to-alls can alternate buffers (overlap D2H of one with the next); every
 * rank must pass the same buffer index to the same execute */
int a2a_plan_set_recv_buffers(a2a_plan* plan, int32_t count);
int a2a_plan_recv_buffer_at(const a2a_plan* plan, int32_t index, void** out_ptr);

/* execute options */
#define A2A_EXEC_COUNT_LINKS 1 /* accumulate device per-(step,edge) byte counters */

/* Launch one all-to-all on `stream` (cudaStream_t; NULL = legacy default).
 * send: this rank's [V_g][N][m] buffer; recv: [V_g][N][m] (NULL = arena recv).
 * Asynchronous; call a2a_plan_sync to wait and collect device errors.
 * Stream-capturable: the epoch of each all-to-all lives in device memory, so a
 * captured execute (one cooperative kernel node) replays as a fresh all-to-all.
 * Executes of one plan must be stream-ordered on every rank, and every rank
 * must run the same number of them. */
int a2a_plan_execute(a2a_plan* plan, const void* send, void* recv, void* stream,
                     int32_t options);
/* wait for the plan's last execute; returns A2A_ERR_TIMEOUT if a device wait timed out */
int a2a_plan_sync(a2a_plan* plan);
/* device byte counters of this rank, out[t * n_edges + e]; then zeroes them */
int a2a_plan_read_link_counters(a2a_plan* plan, int64_t* out);
/* copy engine, before bind: 0 = SM 128-bit load/store loop,
 * 1 = TMA bulk copies (default; cp.async.bulk global->smem->global, mbarrier
 * ring of `tma_stages` x `tma_chunk` bytes per CTA; 0 = defaults 6 x 32 KiB) */
int a2a_plan_set_engine(a2a_plan* plan, int32_t engine, int32_t tma_chunk, int32_t tma_stages);
/* per-CTA %globaltimer timeline of the last execute: out[c][j], j = 0 start,
 * 1 entry barrier passed, 2+t step t published (0 = no work), 2+T' exit,
 * 3+T'+t step t dependencies acquired (0 = none); *out_cols = 2T'+3
 * (call with out = NULL to get the width) */
int a2a_plan_read_timeline(a2a_plan* plan, uint64_t* out, int32_t* out_cols);
/* step-flag publication variant (tuning/diagnostics): bit0 = fence.acq_rel
 * instead of fence.sc before the release store, bit1 = no explicit fence
 * (bar.sync + st.release cumulativity), bit2 = system scope even on one GPU,
 * bit3 = __nanosleep backoff while polling, bit4 = ld.acquire polling instead
 * of ld.relaxed + fence.acq_rel, bit5 = one fence.acq_rel then relaxed flag
 * stores (peers first).  Default 2.  Race hunting (tests): bit6 = every CTA naps
 * a pseudo-random 0-16 us (1 in 16: up to 260 us) before each step / unit /
 * chain task; bit7 = skip the dependency waits (mutation self-test: a
 * perturbed run must then fail; refused unless A2A_ALLOW_MUTATION=1). */
int a2a_plan_set_sync_mode(a2a_plan* plan, int32_t mode);
/* device-side flag-wait timeout (ns, default 10 s) */
int a2a_plan_set_timeout(a2a_plan* plan, int64_t timeout_ns);

#ifdef __cplusplus
}
#endif
#endif /* A2A_EXEC_H */
