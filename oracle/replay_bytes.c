/*
 * ORACLE — test / CPU-baseline infrastructure only, never a product path.
 *
 * C restatement of the reference CPU executor
 *   a2aflow.evaluate.replay_timestep_schedule   (pkg/src/a2aflow/evaluate.py:56-127)
 * that moves real bytes (the reference tracks chunk-id sets only).  Same state
 * machine and checks as oracle/replay_bytes.py (which tests/test_oracle.py pins
 * to the reference's golden vectors); used as the `cpu_baseline` / `--impl
 * reference` arm of bench.py because it is the fastest faithful CPU port:
 *   - evaluate.py:76-80  s holds all Q chunks of (s,d) initially
 *   - evaluate.py:82-100 per step, ops in list order, checked against holdings
 *                        as of the start of the step ("no link", "does not hold")
 *   - evaluate.py:101-107 modelled T (same float operations)
 *   - evaluate.py:108-113 apply arrivals after the checks
 *   - evaluate.py:114-126 final transpose scan
 * Copies of one step run on `nthreads` OpenMP threads (the step's ops are
 * independent: each reads data held at the start of the step), cut into
 * pieces of at most 1 MiB so a step with few large ops still uses every
 * thread.  oracle_replay_ws takes a caller-owned scratch workspace (one m-byte
 * slot per distinct (holder, s, d) forwarding location, carved in first-use
 * order) so repeated replays do not page-fault fresh scratch every call, as
 * the device plan keeps its scratch between executes.
 * Chunk c = bytes [floor(c*m/Q), floor((c+1)*m/Q)); send/recv are [N][N][m].
 */
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t key;       /* (v*n + s)*n + d, +1 (0 = empty) */
  uint8_t* held;      /* Q-bit bitmap */
  uint8_t* data;      /* m bytes (scratch), NULL when v == d (recv) */
} slot_t;

typedef struct {
  slot_t* tab;
  uint64_t cap;
} map_t;

static uint64_t hash64(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  return x ^ (x >> 33);
}

static slot_t* map_get(map_t* M, uint64_t key, int create, int64_t qbytes) {
  uint64_t k = key + 1, i = hash64(k) & (M->cap - 1);
  for (;;) {
    slot_t* s = &M->tab[i];
    if (s->key == k) return s;
    if (s->key == 0) {
      if (!create) return NULL;
      s->held = (uint8_t*)calloc((size_t)qbytes, 1);
      if (!s->held) return NULL;   /* out of memory: slot stays empty */
      s->key = k;
      return s;
    }
    i = (i + 1) & (M->cap - 1);
  }
}

static int bit(const uint8_t* b, int64_t c) { return (b[c >> 3] >> (c & 7)) & 1; }
static void setbit(uint8_t* b, int64_t c) { b[c >> 3] |= (uint8_t)(1u << (c & 7)); }

#define FAIL(...) do { snprintf(err, errlen, __VA_ARGS__); rc = 2; goto done; } while (0)
#define OOM() do { snprintf(err, errlen, "out of host memory"); rc = 1; goto done; } while (0)

#define PIECE_BYTES ((int64_t)1 << 20)

int oracle_replay_ws(int n, int T, int Q, int64_t m, int E, const int32_t* edge_uv,
                     const double* cap, const int32_t* ops, int64_t n_ops,
                     const uint8_t* send, uint8_t* recv, int nthreads, int copy_self,
                     double m_model, double b, double sync, double* T_out,
                     int64_t* link_bytes, char* err, int errlen,
                     uint8_t* ws, int64_t ws_bytes) {
  int rc = 0;
  int64_t ws_used = 0;
  int64_t* pieces = NULL;         /* [k, lo, hi] copy pieces of one step */
  int64_t pcap = 0;
  const int64_t qbytes = (Q + 7) / 8;
  int64_t* eidx = NULL;           /* dense u*n+v -> edge (n <= 4096) */
  int64_t* order = NULL;          /* ops grouped by step, list order */
  int64_t* step_off = NULL;
  uint8_t* arrivals = NULL;       /* [n][n][Q] counts (saturating) */
  double* lb = NULL;
  uint8_t* mark = NULL;
  map_t M = {0};
  if (n < 1 || n > 4096 || Q < 1) { snprintf(err, errlen, "bad sizes"); return 1; }
  eidx = (int64_t*)malloc(sizeof(int64_t) * (size_t)n * n);
  step_off = (int64_t*)calloc((size_t)T + 2, sizeof(int64_t));
  order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_ops + 1));
  M.cap = 1024;
  while (M.cap < (uint64_t)(4 * n_ops + 16)) M.cap <<= 1;
  M.tab = (slot_t*)calloc((size_t)M.cap, sizeof(slot_t));
  arrivals = (uint8_t*)calloc((size_t)n * n * Q, 1);
  lb = (double*)calloc((size_t)(E > 0 ? E : 1), sizeof(double));
  mark = (uint8_t*)calloc((size_t)(E > 0 ? E : 1), 1);
  if (!eidx || !step_off || !order || !M.tab || !arrivals || !lb || !mark) OOM();
  for (int64_t i = 0; i < (int64_t)n * n; ++i) eidx[i] = -1;
  for (int e = 0; e < E; ++e) {
    const int32_t u = edge_uv[2 * e], v = edge_uv[2 * e + 1];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      snprintf(err, errlen, "edge %d (%d,%d) outside [0, %d)", e, u, v, n);
      rc = 1;
      goto done;
    }
    eidx[(int64_t)u * n + v] = e;
  }
  for (int64_t i = 0; i < n_ops; ++i) {
    int t = ops[7 * i];
    if (t >= 0 && t < T) step_off[t + 1]++;
  }
  for (int t = 0; t < T; ++t) step_off[t + 1] += step_off[t];
  {
    int64_t* fill = (int64_t*)calloc((size_t)T + 1, sizeof(int64_t));
    if (!fill) OOM();
    for (int64_t i = 0; i < n_ops; ++i) {
      int t = ops[7 * i];
      if (t >= 0 && t < T) order[step_off[t] + fill[t]++] = i;
    }
    free(fill);
  }
  if (link_bytes) memset(link_bytes, 0, sizeof(int64_t) * (size_t)T * E);
  if (copy_self)
    for (int v = 0; v < n; ++v)
      memcpy(recv + ((int64_t)v * n + v) * m, send + ((int64_t)v * n + v) * m, (size_t)m);
  const double chunk_bytes = m_model / (double)Q;
  double Tm = 0.0;
  for (int t = 0; t < T; ++t) {
    const int64_t a = step_off[t], z = step_off[t + 1];
    /* checks against holdings at the start of the step */
    for (int64_t k = a; k < z; ++k) {
      const int32_t* o = ops + 7 * order[k];
      int src = o[1], dst = o[2], s = o[3], d = o[4], c0 = o[5], c1 = o[6];
      if (src < 0 || src >= n || dst < 0 || dst >= n || eidx[(int64_t)src * n + dst] < 0)
        FAIL("step %d: no link %d->%d", t, src, dst);
      for (int64_t c = c0; c < c1; ++c) {
        int ok;
        if (s < 0 || s >= n || d < 0 || d >= n) ok = 0;
        else if (src == s && s != d) ok = (c >= 0 && c < Q);
        else {
          slot_t* sl = (c >= 0 && c < Q) ? map_get(&M, ((uint64_t)src * n + s) * n + d, 0, qbytes) : NULL;
          ok = sl && bit(sl->held, c);
        }
        if (!ok) FAIL("step %d: node %d sends chunk %lld of shard (%d,%d) it does not hold", t, src,
                      (long long)c, s, d);
      }
    }
    /* modelled step time (evaluate.py:101-107) */
    double step = 0.0;
    {
      int64_t* touched = (int64_t*)malloc(sizeof(int64_t) * (size_t)(z - a + 1));
      if (!touched) OOM();
      int64_t nt = 0;
      for (int64_t k = a; k < z; ++k) {
        const int32_t* o = ops + 7 * order[k];
        int64_t e = eidx[(int64_t)o[1] * n + o[2]];
        if (!mark[e]) { mark[e] = 1; touched[nt++] = e; }
        lb[e] += (double)(o[6] - o[5]) * chunk_bytes;
      }
      for (int64_t j = 0; j < nt; ++j) {
        double x = lb[touched[j]] / (cap[touched[j]] * b);
        if (x > step) step = x;
        lb[touched[j]] = 0.0;
        mark[touched[j]] = 0;
      }
      free(touched);
    }
    Tm += step + sync;
    /* destination slots exist before the parallel copy */
    for (int64_t k = a; k < z; ++k) {
      const int32_t* o = ops + 7 * order[k];
      int dst = o[2], s = o[3], d = o[4];
      if (o[5] >= o[6]) continue;
      if (dst != d) {
        slot_t* sl = map_get(&M, ((uint64_t)dst * n + s) * n + d, 1, qbytes);
        if (!sl) OOM();
        if (!sl->data) {
          if (ws) {
            if (ws_used + m > ws_bytes) {
              snprintf(err, errlen, "workspace too small (%lld bytes)", (long long)ws_bytes);
              rc = 1;
              goto done;
            }
            sl->data = ws + ws_used;
            ws_used += m;
          } else {
            sl->data = (uint8_t*)calloc((size_t)(m > 0 ? m : 1), 1);
            if (!sl->data) OOM();
          }
        }
      }
    }
    /* pieces of at most PIECE_BYTES */
    int64_t np_ = 0;
    for (int64_t k = a; k < z; ++k) {
      const int32_t* o = ops + 7 * order[k];
      if (o[5] >= o[6]) continue;
      const int64_t lo = (int64_t)(((__int128)o[5] * m) / Q), hi = (int64_t)(((__int128)o[6] * m) / Q);
      for (int64_t x = lo; x < hi; x += PIECE_BYTES) {
        if (np_ == pcap) {
          pcap = pcap ? 2 * pcap : 1024;
          int64_t* grown = (int64_t*)realloc(pieces, sizeof(int64_t) * 3 * (size_t)pcap);
          if (!grown) {
            snprintf(err, errlen, "out of host memory");
            rc = 1;
            goto done;
          }
          pieces = grown;
        }
        pieces[3 * np_] = k;
        pieces[3 * np_ + 1] = x;
        pieces[3 * np_ + 2] = (hi - x < PIECE_BYTES) ? hi : x + PIECE_BYTES;
        ++np_;
      }
    }
    /* byte movement: every op reads a location it held at the start of the step */
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
    for (int64_t j = 0; j < np_; ++j) {
      const int32_t* o = ops + 7 * order[pieces[3 * j]];
      int src = o[1], dst = o[2], s = o[3], d = o[4];
      const int64_t lo = pieces[3 * j + 1], hi = pieces[3 * j + 2];
      const uint8_t* from;
      if (src == s) from = send + ((int64_t)s * n + d) * m;
      else if (src == d) from = recv + ((int64_t)d * n + s) * m;
      else from = map_get(&M, ((uint64_t)src * n + s) * n + d, 0, qbytes)->data;
      uint8_t* to = (dst == d) ? recv + ((int64_t)d * n + s) * m
                               : map_get(&M, ((uint64_t)dst * n + s) * n + d, 0, qbytes)->data;
      memcpy(to + lo, from + lo, (size_t)(hi - lo));
    }
    /* apply holdings / arrivals / link bytes (evaluate.py:108-113) */
    for (int64_t k = a; k < z; ++k) {
      const int32_t* o = ops + 7 * order[k];
      int src = o[1], dst = o[2], s = o[3], d = o[4], c0 = o[5], c1 = o[6];
      if (c0 >= c1) continue;
      if (link_bytes)
        link_bytes[(int64_t)t * E + eidx[(int64_t)src * n + dst]] +=
            (int64_t)(((__int128)c1 * m) / Q) - (int64_t)(((__int128)c0 * m) / Q);
      slot_t* sl = (dst != s) ? map_get(&M, ((uint64_t)dst * n + s) * n + d, 1, qbytes) : NULL;
      if (dst != s && !sl) OOM();
      for (int64_t c = c0; c < c1; ++c) {
        if (sl) setbit(sl->held, c);
        if (dst == d) {
          uint8_t* x = &arrivals[((int64_t)s * n + d) * Q + c];
          if (*x < 255) (*x)++;
        }
      }
    }
  }
  for (int s = 0; s < n; ++s)
    for (int d = 0; d < n; ++d) {
      if (s == d) continue;
      for (int c = 0; c < Q; ++c) {
        int k = arrivals[((int64_t)s * n + d) * Q + c];
        if (k == 0) FAIL("shard (%d,%d) chunk %d never delivered", s, d, c);
        if (k > 1) FAIL("shard (%d,%d) chunk %d delivered %d times", s, d, c, k);
      }
    }
  if (T_out) *T_out = Tm;
done:
  if (M.tab) {
    for (uint64_t i = 0; i < M.cap; ++i)
      if (M.tab[i].key) { free(M.tab[i].held); if (!ws) free(M.tab[i].data); }
    free(M.tab);
  }
  free(eidx); free(order); free(step_off); free(arrivals); free(lb); free(mark); free(pieces);
  return rc;
}

int oracle_replay(int n, int T, int Q, int64_t m, int E, const int32_t* edge_uv,
                  const double* cap, const int32_t* ops, int64_t n_ops,
                  const uint8_t* send, uint8_t* recv, int nthreads, int copy_self,
                  double m_model, double b, double sync, double* T_out,
                  int64_t* link_bytes, char* err, int errlen) {
  return oracle_replay_ws(n, T, Q, m, E, edge_uv, cap, ops, n_ops, send, recv, nthreads,
                          copy_self, m_model, b, sync, T_out, link_bytes, err, errlen, NULL, 0);
}
