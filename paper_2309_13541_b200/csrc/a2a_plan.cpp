// Host plan builder: validation, scratch layout and per-GPU copy tables.
//
// Validation restates the reference executor
//   a2aflow.evaluate.replay_timestep_schedule  (pkg/src/a2aflow/evaluate.py:56-127)
// with holdings kept as interval sets instead of Python sets of chunk ids:
//   * ops grouped by t in list order; t outside [0, nsteps) ignored (:82-90)
//   * per op, against holdings as of the start of the step (:91-100):
//       non-edge   -> "step {t}: no link {src}->{dst}"
//       un-held    -> "step {t}: node {src} sends chunk {c} of shard ({s},{d}) it does not hold"
//   * arrivals applied after the step's checks; holdings only grow (:108-113)
//   * final scan s, d, c ascending (:114-126):
//       "shard ({s},{d}) chunk {c} never delivered" / "... delivered {k} times"
// The same holdings, mapped to byte locations (send at s, recv at d, scratch
// elsewhere), resolve every op's source and destination address.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <new>
#include <queue>
#include <string>
#include <unordered_map>
#include <vector>

#include "a2a_internal.h"

namespace a2a {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

namespace {

// Sorted, disjoint, non-adjacent chunk intervals.
struct IntervalSet {
  std::vector<std::pair<int32_t, int32_t>> iv;

  // first chunk of [c0, c1) not covered, or INT32_MIN if all covered
  int64_t first_missing(int64_t c0, int64_t c1) const {
    if (c0 >= c1) return INT64_MIN;
    auto it = std::upper_bound(iv.begin(), iv.end(), std::make_pair((int32_t)c0, INT32_MAX));
    if (it == iv.begin()) return c0;
    --it;
    if (it->second <= c0) return c0;
    if (it->second >= c1) return INT64_MIN;
    return it->second;
  }

  void add(int32_t a, int32_t b) {
    if (a >= b) return;
    std::vector<std::pair<int32_t, int32_t>> out;
    out.reserve(iv.size() + 1);
    bool placed = false;
    for (auto& x : iv) {
      if (x.second < a) {
        out.push_back(x);
      } else if (b < x.first) {
        if (!placed) { out.emplace_back(a, b); placed = true; }
        out.push_back(x);
      } else {  // overlap or adjacency: merge
        a = std::min(a, x.first);
        b = std::max(b, x.second);
      }
    }
    if (!placed) out.emplace_back(a, b);
    iv.swap(out);
  }
};

inline uint64_t key3(int64_t v, int64_t s, int64_t d, int64_t n) {
  return (uint64_t)((v * n + s) * n + d);
}

std::string fmt_missing(int t, int src, int64_t c, int s, int d) {
  char buf[256];
  snprintf(buf, sizeof buf, "step %d: node %d sends chunk %lld of shard (%d,%d) it does not hold",
           t, src, (long long)c, s, d);
  return buf;
}

}  // namespace

static int order_items(Plan& P, std::vector<std::vector<std::vector<DevItem>>>& per, int64_t split_bytes);
static int build_ll_items(Plan& P, const std::function<int32_t(int32_t, int32_t)>& edge_of);

static int build_plan(Plan& P, const a2a_schedule_desc* D) {
  if (!D) return fail(A2A_ERR_INVALID, "null descriptor");
  if (D->n_nodes < 1) return fail(A2A_ERR_INVALID, "n_nodes must be >= 1");
  if (D->n_steps < 0) return fail(A2A_ERR_INVALID, "n_steps must be >= 0");
  if (D->q < 1) return fail(A2A_ERR_INVALID, "q must be >= 1");
  if (D->m_bytes < 0) return fail(A2A_ERR_INVALID, "m_bytes must be >= 0");
  if (D->n_edges < 0 || (D->n_edges > 0 && !D->edge_uv))
    return fail(A2A_ERR_INVALID, "bad edge list");
  if (D->n_ops < 0 || (D->n_ops > 0 && !D->ops)) return fail(A2A_ERR_INVALID, "bad op list");
  if (D->n_gpus < 1 || D->n_gpus > A2A_MAX_GPUS)
    return fail(A2A_ERR_INVALID, "n_gpus must be in [1, 8]");
  if ((D->flags & (A2A_PROTO_LL | A2A_PROTO_LL128)) && (D->flags & (A2A_INTERLEAVE | A2A_REUSE_SCRATCH)))
    return fail(A2A_ERR_INVALID, "A2A_PROTO_LL cannot be combined with A2A_INTERLEAVE or A2A_REUSE_SCRATCH");
  const int n = D->n_nodes, T = D->n_steps, E = D->n_edges, G = D->n_gpus;
  const int64_t Q = D->q, m = D->m_bytes;
  P.n = n; P.T = T; P.Q = (int32_t)Q; P.E = E; P.G = G; P.m = m; P.flags = D->flags;
  P.ll128 = (D->flags & A2A_PROTO_LL128) != 0;
  P.ll = P.ll128 || (D->flags & A2A_PROTO_LL) != 0;
  if (P.ll) P.engine = 0;   // LL pieces are thread work: the 1024-thread kernel (measured)
  // LL128: CTA pieces start on line boundaries (120 B) and keep 64-byte alignment
  P.gran = P.ll128 ? 15 * 64 : 64;
  P.T_exec = std::max(T, 1);
  P.edge_uv.assign(D->edge_uv, D->edge_uv + 2 * (size_t)E);
  P.cap.resize(E, 1.0);
  if (D->edge_cap) P.cap.assign(D->edge_cap, D->edge_cap + E);
  P.ops.assign(D->ops, D->ops + D->n_ops);
  P.node_gpu.assign(n, 0);
  if (D->node_gpu) {
    for (int v = 0; v < n; ++v) {
      if (D->node_gpu[v] < 0 || D->node_gpu[v] >= G)
        return fail(A2A_ERR_INVALID, "node_gpu entry out of range");
      P.node_gpu[v] = D->node_gpu[v];
    }
  }
  // edge index (Digraph.edge_index, reference src/graphs.py:84-86)
  std::unordered_map<uint64_t, int32_t> eidx;
  eidx.reserve(E * 2 + 1);
  for (int e = 0; e < E; ++e) {
    int u = P.edge_uv[2 * e], v = P.edge_uv[2 * e + 1];
    if (u < 0 || u >= n || v < 0 || v >= n) return fail(A2A_ERR_INVALID, "edge endpoint out of range");
    eidx[((uint64_t)(uint32_t)u << 32) | (uint32_t)v] = e;
  }
  auto edge_of = [&](int32_t u, int32_t v) -> int32_t {
    auto it = eidx.find(((uint64_t)(uint32_t)u << 32) | (uint32_t)v);
    return it == eidx.end() ? -1 : it->second;
  };
  // group by step in list order (evaluate.py:82-84); out-of-range t ignored
  P.step_ops.assign(T, {});
  for (int64_t i = 0; i < (int64_t)P.ops.size(); ++i) {
    int t = P.ops[i].t;
    if (t >= 0 && t < T) P.step_ops[t].push_back(i);
  }

  // ---- replay: holdings as interval sets
  std::unordered_map<uint64_t, IntervalSet> held;     // (v,s,d), v != s (s holds all implicitly)
  std::unordered_map<uint64_t, IntervalSet> written;  // (v,s,d), v != d: scratch contents
  std::vector<std::vector<std::pair<int32_t, int32_t>>> delivered((size_t)n * n);
  auto in_range = [&](int x) { return x >= 0 && x < n; };
  auto first_missing = [&](const a2a_op& o) -> int64_t {
    if (o.c0 >= o.c1) return INT64_MIN;
    if (!in_range(o.s) || !in_range(o.d)) return o.c0;
    if (o.src == o.s && o.s != o.d) {  // initial holdings {0..Q-1} (evaluate.py:76-80)
      if (o.c0 < 0) return o.c0;
      if (o.c1 > Q) return std::max<int64_t>(o.c0, Q);
      return INT64_MIN;
    }
    auto it = held.find(key3(o.src, o.s, o.d, n));
    if (it == held.end()) return o.c0;
    return it->second.first_missing(o.c0, o.c1);
  };
  for (int t = 0; t < T; ++t) {
    for (int64_t i : P.step_ops[t]) {
      const a2a_op& o = P.ops[i];
      if (edge_of(o.src, o.dst) < 0) {
        char buf[160];
        snprintf(buf, sizeof buf, "step %d: no link %d->%d", t, o.src, o.dst);
        return fail(A2A_ERR_EVAL, buf);
      }
      int64_t c = first_missing(o);
      if (c != INT64_MIN) return fail(A2A_ERR_EVAL, fmt_missing(t, o.src, c, o.s, o.d));
    }
    for (int64_t i : P.step_ops[t]) {
      const a2a_op& o = P.ops[i];
      if (o.c0 >= o.c1) continue;
      if (o.dst != o.s) held[key3(o.dst, o.s, o.d, n)].add(o.c0, o.c1);
      if (o.dst != o.d) written[key3(o.dst, o.s, o.d, n)].add(o.c0, o.c1);
      if (o.dst == o.d) delivered[(size_t)o.s * n + o.d].emplace_back(o.c0, o.c1);
    }
  }
  // transpose check (evaluate.py:114-126)
  for (int s = 0; s < n; ++s) {
    for (int d = 0; d < n; ++d) {
      if (s == d) continue;
      auto& dl = delivered[(size_t)s * n + d];
      // sweep: coverage count per chunk, first chunk with count != 1
      std::vector<std::pair<int64_t, int>> ev;
      ev.reserve(dl.size() * 2);
      for (auto& x : dl) { ev.emplace_back(x.first, +1); ev.emplace_back(x.second, -1); }
      std::sort(ev.begin(), ev.end());
      int64_t pos = 0;
      int cover = 0;
      size_t k = 0;
      while (pos < Q) {
        while (k < ev.size() && ev[k].first <= pos) { cover += ev[k].second; ++k; }
        if (cover != 1) {
          char buf[160];
          if (cover == 0)
            snprintf(buf, sizeof buf, "shard (%d,%d) chunk %lld never delivered", s, d, (long long)pos);
          else
            snprintf(buf, sizeof buf, "shard (%d,%d) chunk %lld delivered %d times", s, d,
                     (long long)pos, cover);
          return fail(A2A_ERR_EVAL, buf);
        }
        pos = (k < ev.size()) ? std::min<int64_t>(ev[k].first, Q) : Q;
      }
    }
  }

  // ---- placement: local node index per GPU
  P.local_idx.assign(n, 0);
  P.info.assign(G, a2a_gpu_info{});
  for (int g = 0; g < G; ++g) P.info[g].first_node = -1;
  for (int v = 0; v < n; ++v) {
    auto& I = P.info[P.node_gpu[v]];
    if (I.first_node < 0) I.first_node = v;
    P.local_idx[v] = I.n_local_nodes++;
  }
  for (int g = 0; g < G; ++g) {
    P.info[g].send_bytes = (int64_t)P.info[g].n_local_nodes * n * m;
    P.info[g].recv_bytes = P.info[g].send_bytes;
  }
  if (P.ll) return build_ll_items(P, edge_of);

  // ---- scratch layout: per (v,s,d) the merged intervals ever written there.
  // A slot starts at the same residue mod 64 as the shard offset of its first
  // chunk, so every copy has src == dst (mod 64) whenever m % 64 == 0.
  std::vector<uint64_t> keys;
  keys.reserve(written.size());
  for (auto& kv : written) keys.push_back(kv.first);
  std::sort(keys.begin(), keys.end());  // deterministic across ranks
  std::unordered_map<uint64_t, std::vector<Interval>> slots;
  slots.reserve(keys.size() * 2 + 1);
  std::vector<int64_t> cursor(G, 0);
  const bool reuse = (P.flags & A2A_REUSE_SCRATCH) != 0;
  P.reuse = reuse;
  if (!reuse) {
    for (uint64_t k : keys) {
      int v = (int)(k / ((uint64_t)n * n));
      int g = P.node_gpu[v];
      auto& out = slots[k];
      for (auto& x : written[k].iv) {
        int64_t lo = chunk_off(x.first, m, Q), hi = chunk_off(x.second, m, Q);
        int64_t base = ((cursor[g] + 63) & ~(int64_t)63) + (lo & 63);
        out.push_back(Interval{x.first, x.second, base});
        cursor[g] = base + (hi - lo);
      }
    }
  } else {
    // Liveness reuse (SURVEY.md §7 hard part 4): each slot interval lives from
    // its first write to its last access; an offline first-fit allocator hands
    // out regions whose previous occupant is dead (strictly earlier step).
    // build_sync adds the WAR/WAW dependencies that make reuse safe.
    struct Ref { uint64_t key; int32_t a, b; int64_t lo, hi; int start, end, gpu; };
    std::vector<Ref> refs;
    std::unordered_map<uint64_t, std::vector<int>> by_key;
    for (uint64_t k : keys) {
      int v = (int)(k / ((uint64_t)n * n));
      for (auto& x : written[k].iv) {
        by_key[k].push_back((int)refs.size());
        refs.push_back(Ref{k, x.first, x.second, chunk_off(x.first, m, Q), chunk_off(x.second, m, Q),
                           INT32_MAX, -1, P.node_gpu[v]});
      }
    }
    auto find = [&](int v, int s_, int d_, int32_t c0) -> Ref* {
      auto it = by_key.find(key3(v, s_, d_, n));
      if (it == by_key.end()) return nullptr;
      for (int r : it->second)
        if (refs[r].a <= c0 && c0 < refs[r].b) return &refs[r];
      return nullptr;
    };
    for (int t = 0; t < T; ++t)
      for (int64_t i : P.step_ops[t]) {
        const a2a_op& o = P.ops[i];
        if (o.c0 >= o.c1) continue;
        if (o.dst != o.d) {
          Ref* r = find(o.dst, o.s, o.d, o.c0);
          if (r) { r->start = std::min(r->start, t); r->end = std::max(r->end, t); }
        }
        if (o.src != o.s && o.src != o.d) {
          Ref* r = find(o.src, o.s, o.d, o.c0);
          if (r) r->end = std::max(r->end, t);
        }
      }
    std::vector<int> order(refs.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      if (refs[x].gpu != refs[y].gpu) return refs[x].gpu < refs[y].gpu;
      return refs[x].start < refs[y].start;
    });
    std::vector<std::map<int64_t, int64_t>> freel(G);           // offset -> size
    std::vector<std::vector<std::array<int64_t, 3>>> active(G);   // {end, off, size}
    std::unordered_map<int, int64_t> base_of;
    auto release = [&](int g, int64_t off, int64_t size) {
      auto& F = freel[g];
      auto it = F.emplace(off, size).first;
      auto nx = std::next(it);
      if (nx != F.end() && it->first + it->second == nx->first) { it->second += nx->second; F.erase(nx); }
      if (it != F.begin()) {
        auto pv = std::prev(it);
        if (pv->first + pv->second == it->first) { pv->second += it->second; F.erase(it); }
      }
    };
    for (int r : order) {
      Ref& R = refs[r];
      const int g = R.gpu;
      auto& A = active[g];
      for (size_t j = 0; j < A.size();) {
        if (A[j][0] < R.start) { release(g, A[j][1], A[j][2]); A[j] = A.back(); A.pop_back(); }
        else ++j;
      }
      const int64_t need = R.hi - R.lo, res = R.lo & 63;
      int64_t base = -1;
      for (auto it = freel[g].begin(); it != freel[g].end(); ++it) {
        int64_t b = it->first + (((res - it->first) % 64) + 64) % 64;
        if (b + need <= it->first + it->second) {
          const int64_t off = it->first, size = it->second;
          freel[g].erase(it);
          if (b > off) freel[g].emplace(off, b - off);
          if (b + need < off + size) freel[g].emplace(b + need, off + size - (b + need));
          base = b;
          break;
        }
      }
      if (base < 0) {
        base = ((cursor[g] + 63) & ~(int64_t)63) + res;
        cursor[g] = base + need;
      }
      if (need > 0) A.push_back({R.end, base, need});
      base_of[r] = base;
    }
    for (uint64_t k : keys) {
      auto& out = slots[k];
      for (int r : by_key[k]) out.push_back(Interval{refs[r].a, refs[r].b, base_of[r]});
    }
  }
  for (int g = 0; g < G; ++g) P.info[g].scratch_bytes = (cursor[g] + 4095) & ~(int64_t)4095;
  auto slot_addr = [&](int v, int s, int d, int32_t c0, int64_t byte_lo, int64_t* out) -> bool {
    auto it = slots.find(key3(v, s, d, n));
    if (it == slots.end()) return false;
    for (auto& x : it->second)
      if (x.a <= c0 && c0 < x.b) {
        *out = x.base + (byte_lo - chunk_off(x.a, m, Q));
        return true;
      }
    return false;
  };

  // ---- copy items per GPU per step
  const int TE = P.T_exec;
  P.tables.assign(G, GpuTables{});
  P.link_bytes.assign((size_t)T * E, 0);
  std::vector<std::vector<std::vector<DevItem>>> per(G, std::vector<std::vector<DevItem>>(TE));
  for (int t = 0; t < T; ++t) {
    for (int64_t i : P.step_ops[t]) {
      const a2a_op& o = P.ops[i];
      if (o.c0 >= o.c1) continue;
      int64_t lo = chunk_off(o.c0, m, Q), hi = chunk_off(o.c1, m, Q);
      int e = edge_of(o.src, o.dst);
      P.link_bytes[(size_t)t * E + e] += hi - lo;
      if (hi == lo) continue;
      int g = P.node_gpu[o.src], h = P.node_gpu[o.dst];
      DevItem it{};
      it.nbytes = hi - lo;
      it.edge = e;
      it.dst_gpu = h;
      if (o.src == o.s) {
        it.src_loc = loc_send();
        it.src_off = ((int64_t)P.local_idx[o.src] * n + o.d) * m + lo;
      } else if (o.src == o.d) {
        it.src_loc = loc_recv(g);
        it.src_off = ((int64_t)P.local_idx[o.src] * n + o.s) * m + lo;
      } else {
        it.src_loc = loc_scratch(g, G);
        if (!slot_addr(o.src, o.s, o.d, o.c0, lo, &it.src_off))
          return fail(A2A_ERR_INVALID, "internal: source chunk has no scratch slot");
      }
      if (o.dst == o.d) {
        it.dst_loc = loc_recv(h);
        it.dst_off = ((int64_t)P.local_idx[o.dst] * n + o.s) * m + lo;
      } else {
        it.dst_loc = loc_scratch(h, G);
        if (!slot_addr(o.dst, o.s, o.d, o.c0, lo, &it.dst_off))
          return fail(A2A_ERR_INVALID, "internal: destination chunk has no scratch slot");
      }
      per[g][t].push_back(it);
      auto& Ig = P.info[g];
      Ig.hop_bytes += it.nbytes;
      if (h != g) {
        Ig.egress_bytes += it.nbytes;
        P.info[h].ingress_bytes += it.nbytes;
      } else {
        Ig.local_bytes += it.nbytes;
      }
    }
  }
  if ((P.flags & A2A_COPY_SELF) && m > 0) {
    for (int v = 0; v < n; ++v) {
      int g = P.node_gpu[v];
      DevItem it{};
      it.src_loc = loc_send();
      it.dst_loc = loc_recv(g);
      it.src_off = it.dst_off = ((int64_t)P.local_idx[v] * n + v) * m;
      it.nbytes = m;
      it.edge = -1;
      it.dst_gpu = g;
      per[g][0].push_back(it);
      P.info[g].local_bytes += m;
    }
  }
  return order_items(P, per, D->split_bytes);
}

// Per (gpu, step) item order + byte prefixes.  Default: grouped by destination
// GPU (stable), so CTAs cover few destinations each.  A2A_INTERLEAVE: items are
// split into <= split_bytes pieces (multiples of 64 B, alignment kept) and
// the destination classes are merged in proportion to their byte totals, so
// every CTA range drives every NVLink peer (and local HBM) at once.
static int order_items(Plan& P, std::vector<std::vector<std::vector<DevItem>>>& per, int64_t split_bytes) {
  const int G = P.G, TE = P.T_exec;
  const bool interleave = (P.flags & A2A_INTERLEAVE) && G > 1;
  const int64_t split = std::max<int64_t>(64, (split_bytes > 0 ? split_bytes : 262144) & ~63LL);
  for (int g = 0; g < G; ++g) {
    auto& tb = P.tables[g];
    tb.step_begin.assign(TE + 1, 0);
    tb.step_bytes.assign(TE, 0);
    for (int t = 0; t < TE; ++t) {
      auto& L = per[g][t];
      std::stable_sort(L.begin(), L.end(), [&](const DevItem& a, const DevItem& b) {
        // LL same-step decodes last: every CTA stores its step's lines before
        // it polls lines of the same step (deadlock freedom)
        int ka = (a.kind & kDecode) ? G : (a.dst_gpu - g + G) % G;
        int kb = (b.kind & kDecode) ? G : (b.dst_gpu - g + G) % G;
        return ka < kb;
      });
      if (interleave) {
        std::vector<std::vector<DevItem>> bucket(G);
        std::vector<int64_t> total(G, 0), emitted(G, 0);
        std::vector<size_t> pos(G, 0);
        for (auto& it : L) {
          for (int64_t x = 0; x < it.nbytes; x += split) {
            DevItem pc = it;
            pc.src_off += x;
            pc.dst_off += x;
            pc.nbytes = std::min(split, it.nbytes - x);
            bucket[it.dst_gpu].push_back(pc);
          }
          total[it.dst_gpu] += it.nbytes;
        }
        std::vector<DevItem> out;
        out.reserve(L.size() * 2);
        for (;;) {
          int best = -1;
          double bf = 2.0;
          for (int h = 0; h < G; ++h) {
            if (pos[h] >= bucket[h].size()) continue;
            double f = (double)emitted[h] / (double)total[h];
            if (f < bf) { bf = f; best = h; }
          }
          if (best < 0) break;
          const DevItem& pc = bucket[best][pos[best]++];
          emitted[best] += pc.nbytes;
          out.push_back(pc);
        }
        L.swap(out);
      }
      tb.step_begin[t] = (int64_t)tb.items.size();
      int64_t pre = 0;
      for (auto& it : L) {
        it.prefix = pre;
        pre += it.nbytes;
        tb.items.push_back(it);
      }
      tb.step_bytes[t] = pre;
    }
    tb.step_begin[TE] = (int64_t)tb.items.size();
    P.info[g].n_items = (int64_t)tb.items.size();
  }
  return A2A_OK;
}

// ---- A2A_PROTO_LL items ------------------------------------------------------
//
// Every hop lands as LL lines (16-byte {4 data bytes, epoch, 4 data bytes,
// epoch}) in a fresh slot of the destination node's GPU, and every forwarding
// hop polls its source lines directly: no scratch copy, no step flag, no
// fence anywhere on the path.  Hop 0 reads the caller's send buffer, the last
// hop writes plain bytes into recv.  LL offsets are payload addresses (byte x
// of a region's payload lives in line x/8); slots start at multiples of 8.  A
// forwarding op whose chunks arrived through several earlier ops is split at
// those arrivals, so each item reads one slot.  The landing region of each GPU
// is double-buffered by epoch parity (see the kernel's lagged entry).
static int build_ll_items(Plan& P, const std::function<int32_t(int32_t, int32_t)>& edge_of) {
  const int n = P.n, T = P.T, G = P.G, TE = P.T_exec;
  const int64_t Q = P.Q, m = P.m;
  struct Arrival { int32_t c0, c1, t; int64_t pa; };   // chunks [c0,c1) at payload address pa
  std::unordered_map<uint64_t, std::vector<Arrival>> at;   // (node, s, d) -> arrivals
  std::vector<int64_t> cursor(G, 0);                        // landing payload bytes per GPU
  std::vector<std::vector<std::vector<DevItem>>> per(G, std::vector<std::vector<DevItem>>(TE));
  P.tables.assign(G, GpuTables{});
  P.link_bytes.assign((size_t)T * P.E, 0);
  for (int t = 0; t < T; ++t) {
    std::vector<std::pair<uint64_t, Arrival>> fresh;   // usable from step t + 1 on
    for (int64_t i : P.step_ops[t]) {
      const a2a_op& o = P.ops[i];
      if (o.c0 >= o.c1) continue;
      const int e = edge_of(o.src, o.dst);
      P.link_bytes[(size_t)t * P.E + e] += chunk_off(o.c1, m, Q) - chunk_off(o.c0, m, Q);
      if (o.src == o.d && o.src != o.s)
        return fail(A2A_ERR_INVALID, "A2A_PROTO_LL: the schedule forwards chunks out of their destination");
      const int g = P.node_gpu[o.src], h = P.node_gpu[o.dst];
      // source segments: [ca, cb) read from send (hop 0) or from one arrival slot
      for (int32_t ca = o.c0; ca < o.c1;) {
        int32_t cb = o.c1;
        int src_loc = loc_send();
        int64_t src_off = 0, lo = chunk_off(ca, m, Q);
        if (o.src == o.s) {
          src_off = ((int64_t)P.local_idx[o.src] * n + o.d) * m + lo;
        } else {
          const Arrival* best = nullptr;
          auto it = at.find(key3(o.src, o.s, o.d, n));
          if (it != at.end())
            for (const Arrival& a : it->second)
              if (a.t < t && a.c0 <= ca && ca < a.c1 && (!best || a.c1 > best->c1)) best = &a;
          if (!best) return fail(A2A_ERR_INVALID, "internal: LL source chunk has no arrival");
          cb = std::min(cb, best->c1);
          src_loc = loc_ll(g, G);
          src_off = best->pa + (lo - chunk_off(best->c0, m, Q));
        }
        const int64_t hi = chunk_off(cb, m, Q);
        if (o.dst != o.d)   // arrival record even for empty byte ranges (m < Q)
          fresh.push_back({key3(o.dst, o.s, o.d, n), Arrival{ca, cb, t, cursor[h]}});
        if (hi > lo) {
          DevItem it{};
          it.nbytes = hi - lo;
          it.edge = e;
          it.dst_gpu = (int16_t)h;
          it.src_loc = src_loc;
          it.src_off = src_off;
          it.kind = src_loc == loc_send() ? kCopy : kLLSrc;
          const int64_t recv_off = ((int64_t)P.local_idx[o.dst] * n + o.s) * m + lo;
          if (o.dst == o.d && h == g) {   // local final hop: plain bytes into recv
            it.dst_loc = loc_recv(h);
            it.dst_off = recv_off;
          } else {
            it.dst_loc = loc_ll(h, G);
            it.dst_off = cursor[h];
            it.kind |= kLLDst;
            if (o.dst == o.d) {   // remote final hop: h decodes the lines into recv in the same step
              DevItem dc{};
              dc.nbytes = it.nbytes;
              dc.edge = -1;
              dc.dst_gpu = (int16_t)h;
              dc.src_loc = loc_ll(h, G);
              dc.src_off = cursor[h];
              dc.dst_loc = loc_recv(h);
              dc.dst_off = recv_off;
              dc.kind = kLLSrc | kDecode;
              per[h][t].push_back(dc);
            }
            const int64_t pl = ll_payload(P.ll128);   // slots start on a line
            cursor[h] += (it.nbytes + pl - 1) / pl * pl;
          }
          per[g][t].push_back(it);
          auto& Ig = P.info[g];
          Ig.hop_bytes += it.nbytes;
          if (h != g) {
            Ig.egress_bytes += it.nbytes;
            P.info[h].ingress_bytes += it.nbytes;
          } else {
            Ig.local_bytes += it.nbytes;
          }
        }
        ca = cb;
      }
    }
    for (auto& f : fresh) at[f.first].push_back(f.second);
  }
  if ((P.flags & A2A_COPY_SELF) && m > 0) {
    for (int v = 0; v < n; ++v) {
      const int g = P.node_gpu[v];
      DevItem it{};
      it.src_loc = loc_send();
      it.dst_loc = loc_recv(g);
      it.src_off = it.dst_off = ((int64_t)P.local_idx[v] * n + v) * m;
      it.nbytes = m;
      it.edge = -1;
      it.dst_gpu = (int16_t)g;
      per[g][0].push_back(it);
      P.info[g].local_bytes += m;
    }
  }
  P.ll_off.assign(G, 0);
  P.ll_half.assign(G, 0);
  for (int g = 0; g < G; ++g) {
    const int64_t lines = cursor[g] / ll_payload(P.ll128);
    P.ll_half[g] = (lines * ll_line(P.ll128) + 4095) & ~(int64_t)4095;   // line bytes per parity
    P.info[g].scratch_bytes = 2 * P.ll_half[g];               // epoch parity 0 | 1
  }
  return order_items(P, per, 0);
}

// ---- CTA split and exact producer dependencies ---------------------------
//
// Every GPU splits each step's concatenated item bytes into nC contiguous
// ranges (cta_lo).  A piece of an item written by CTA (t, g, c) lands in a
// destination byte segment of some GPU's recv or scratch; a consumer piece
// (t', h, c') that reads bytes of its own recv/scratch must acquire every
// producer whose segment overlaps its source range and whose step t < t'.
namespace {
struct Seg {
  int64_t a, b;
  int32_t t, slot;
};
// CTA split of one step: the step's items are cut into nC contiguous ranges of
// equal *cost*, where a byte bound for another GPU (NVLink) costs `wr` and a
// local byte (HBM) costs 1 -- an SM moves local bytes several times faster
// than it can push them over NVLink, so equal-byte ranges would leave the
// NVLink CTAs finishing last.  Boundaries inside an item fall on 64-byte
// multiples (the item end excepted), so every piece keeps src == dst (mod 64).
// offsets of the piece starting at byte x of an item (LL: payload addresses)
inline int64_t piece_src(const DevItem& it, int64_t x) { return it.src_off + x; }
inline int64_t piece_dst(const DevItem& it, int64_t x) { return it.dst_off + x; }
template <typename F>
void for_each_piece(const GpuTables& tb, int g, int t, int nC, int wr, int64_t gran, F&& f) {
  const int64_t b0 = tb.step_begin[t], b1 = tb.step_begin[t + 1];
  if (b1 <= b0) return;
  std::vector<int64_t> pw(b1 - b0 + 1, 0);  // weighted prefix
  for (int64_t j = b0; j < b1; ++j) {
    const DevItem& it = tb.items[j];
    pw[j - b0 + 1] = pw[j - b0] + (it.dst_gpu != g ? wr : 1) * it.nbytes;
  }
  const int64_t W = pw[b1 - b0];
  auto pos = [&](int64_t j, int64_t b) -> int64_t {  // byte position of cost b in item j
    const DevItem& it = tb.items[j];
    const int64_t w = it.dst_gpu != g ? wr : 1, P0 = pw[j - b0];
    if (b <= P0) return 0;
    if (b >= P0 + w * it.nbytes) return it.nbytes;
    return std::min<int64_t>(it.nbytes, ((b - P0) / w) / gran * gran);
  };
  int64_t k = b0;
  for (int c = 0; c < nC; ++c) {
    const int64_t lo = (int64_t)(((__int128)W * c) / nC), hi = (int64_t)(((__int128)W * (c + 1)) / nC);
    if (hi <= lo) continue;
    while (k < b1 && pw[k - b0 + 1] <= lo) ++k;
    for (int64_t j = k; j < b1 && pw[j - b0] < hi; ++j) {
      const int64_t x0 = pos(j, lo), x1 = pos(j, hi);
      if (x1 > x0) f(c, tb.items[j], x0, x1);
    }
  }
}
}  // namespace

int build_sync(Plan& P, int nC) {
  if (P.sync.nC == nC && P.sync.weight == P.remote_weight) return A2A_OK;
  if (nC < 1) return fail(A2A_ERR_INVALID, "num_ctas must be >= 1");
  const int G = P.G, TE = P.T_exec;
  SyncTables S;
  S.nC = nC;
  S.weight = P.remote_weight;
  S.dst_mask.assign(G, std::vector<uint32_t>((size_t)TE * nC, 0));
  // segs[h][0] = writes into h's recv, segs[h][1] = into h's scratch
  std::vector<std::array<std::vector<Seg>, 2>> segs(G);
  for (int g = 0; g < G; ++g) {
    for (int t = 0; t < TE; ++t) {
      for_each_piece(P.tables[g], g, t, nC, P.remote_weight, P.gran, [&](int c, const DevItem& it, int64_t x0, int64_t x1) {
        if (P.ll) return;   // LL: no flags, consumers poll the lines
        S.dst_mask[g][(size_t)t * nC + c] |= 1u << it.dst_gpu;
        const int cls = (it.dst_loc == loc_recv(it.dst_gpu)) ? 0 : 1;
        segs[it.dst_gpu][cls].push_back(
            Seg{it.dst_off + x0, it.dst_off + x1, t, (int32_t)(((int64_t)t * G + g) * nC + c)});
      });
    }
  }
  // sorted by start, with running max of ends for the backward overlap walk
  std::vector<std::array<std::vector<int64_t>, 2>> maxend(G);
  for (int h = 0; h < G; ++h)
    for (int cls = 0; cls < 2; ++cls) {
      auto& v = segs[h][cls];
      std::sort(v.begin(), v.end(), [](const Seg& x, const Seg& y) { return x.a < y.a; });
      auto& me = maxend[h][cls];
      me.resize(v.size());
      int64_t m = INT64_MIN;
      for (size_t i = 0; i < v.size(); ++i) me[i] = m = std::max(m, v[i].b);
    }
  S.wait_off.assign(G, {});
  S.wait_idx.assign(G, {});
  S.exit_idx.assign(G, {});
  // per[g][t*nC + c]: producer slots CTA (g, c) must acquire before step t
  std::vector<std::vector<std::vector<int32_t>>> per_all(G, std::vector<std::vector<int32_t>>((size_t)TE * nC));
  if (P.reuse) {
    // WAR / WAW: a write into reused scratch bytes waits for every earlier
    // read (local CTAs of the owning GPU) and write of those bytes; the earlier
    // CTAs also publish their flag to the writer's GPU.
    std::vector<std::vector<Seg>> rseg(G), wseg(G);
    std::vector<std::vector<int32_t>> rcta(G), wg(G);   // producer GPU of each segment
    for (int g = 0; g < G; ++g)
      for (int t = 0; t < TE; ++t)
        for_each_piece(P.tables[g], g, t, nC, P.remote_weight, P.gran, [&](int c, const DevItem& it, int64_t x0, int64_t x1) {
          const int32_t slot = (int32_t)(((int64_t)t * G + g) * nC + c);
          if (it.src_loc == loc_scratch(g, G)) {
            rseg[g].push_back(Seg{it.src_off + x0, it.src_off + x1, t, slot});
            rcta[g].push_back(g);
          }
          if (it.dst_loc == loc_scratch(it.dst_gpu, G)) {
            wseg[it.dst_gpu].push_back(Seg{it.dst_off + x0, it.dst_off + x1, t, slot});
            wg[it.dst_gpu].push_back(g);
          }
        });
    for (int h = 0; h < G; ++h) {
      // accesses of h's scratch, sorted by start with running max end
      struct Acc { Seg s; int32_t gpu; };
      std::vector<Acc> acc;
      for (size_t i = 0; i < rseg[h].size(); ++i) acc.push_back(Acc{rseg[h][i], rcta[h][i]});
      for (size_t i = 0; i < wseg[h].size(); ++i) acc.push_back(Acc{wseg[h][i], wg[h][i]});
      std::sort(acc.begin(), acc.end(), [](const Acc& x, const Acc& y) { return x.s.a < y.s.a; });
      std::vector<int64_t> me(acc.size());
      int64_t mx = INT64_MIN;
      for (size_t i = 0; i < acc.size(); ++i) me[i] = mx = std::max(mx, acc[i].s.b);
      for (size_t i = 0; i < wseg[h].size(); ++i) {
        const Seg& w = wseg[h][i];
        const int g = wg[h][i];
        const int c = (int)(w.slot % nC);
        size_t j = std::lower_bound(acc.begin(), acc.end(), w.b,
                                    [](const Acc& x, int64_t b) { return x.s.a < b; }) - acc.begin();
        while (j > 0) {
          --j;
          if (me[j] <= w.a) break;
          const Acc& q = acc[j];
          if (q.s.b > w.a && q.s.t < w.t) {
            per_all[g][(size_t)w.t * nC + c].push_back(q.s.slot);
            const int qt = q.s.t, qc = (int)(q.s.slot % nC);
            S.dst_mask[q.gpu][(size_t)qt * nC + qc] |= 1u << g;
          }
        }
      }
    }
  }
  for (int h = 0; h < G; ++h) {
    auto& off = S.wait_off[h];
    auto& idx = S.wait_idx[h];
    off.assign((size_t)TE * nC + 1, 0);
    auto& per = per_all[h];
    for (int t = 0; t < TE; ++t) {
      for_each_piece(P.tables[h], h, t, nC, P.remote_weight, P.gran, [&](int c, const DevItem& it, int64_t x0, int64_t x1) {
        if (it.src_loc == loc_send() || P.ll) return;
        const int cls = (it.src_loc == loc_recv(h)) ? 0 : 1;
        const int64_t a = it.src_off + x0, b = it.src_off + x1;
        const auto& v = segs[h][cls];
        const auto& me = maxend[h][cls];
        // segments with start < b, walking back while some end can exceed a
        size_t j = std::lower_bound(v.begin(), v.end(), b,
                                    [](const Seg& s, int64_t x) { return s.a < x; }) - v.begin();
        auto& out = per[(size_t)t * nC + c];
        while (j > 0) {
          --j;
          if (me[j] <= a) break;
          if (v[j].b > a && v[j].t < t) out.push_back(v[j].slot);
        }
      });
    }
    for (size_t k = 0; k < per.size(); ++k) {
      auto& d = per[k];
      std::sort(d.begin(), d.end());
      d.erase(std::unique(d.begin(), d.end()), d.end());
      off[k] = (int32_t)idx.size();
      idx.insert(idx.end(), d.begin(), d.end());
    }
    off[per.size()] = (int32_t)idx.size();
    for (int t = 0; t < TE; ++t)
      for (int g = 0; g < G; ++g)
        for (int c = 0; c < nC; ++c)
          if (S.dst_mask[g][(size_t)t * nC + c] & (1u << h))
            S.exit_idx[h].push_back((int32_t)(((int64_t)t * G + g) * nC + c));
  }
  // per-CTA programs: exact piece lists (split below 1 GiB so nbytes fits int32)
  S.pieces.assign(G, {});
  S.prog.assign(G, {});
  for (int g = 0; g < G; ++g) {
    std::vector<std::vector<std::vector<DevPiece>>> per_ct(nC, std::vector<std::vector<DevPiece>>(TE));
    for (int t = 0; t < TE; ++t)
      for_each_piece(P.tables[g], g, t, nC, P.remote_weight, P.gran, [&](int c, const DevItem& it, int64_t x0, int64_t x1) {
        for (int64_t x = x0; x < x1; x += (1LL << 30)) {
          DevPiece pc{};
          pc.src_off = piece_src(it, x);
          pc.dst_off = piece_dst(it, x);
          pc.nbytes = (int32_t)std::min<int64_t>(1LL << 30, x1 - x);
          pc.edge = it.edge;
          pc.src_loc = (int16_t)it.src_loc;
          pc.dst_loc = (int16_t)it.dst_loc;
          pc.kind = it.kind;
          per_ct[c][t].push_back(pc);
        }
      });
    auto& pcs = S.pieces[g];
    auto& prog = S.prog[g];
    prog.assign((size_t)nC * TE, CtaStep{});
    for (int c = 0; c < nC; ++c)
      for (int t = 0; t < TE; ++t) {
        CtaStep& cs = prog[(size_t)c * TE + t];
        cs.pb = (int32_t)pcs.size();
        pcs.insert(pcs.end(), per_ct[c][t].begin(), per_ct[c][t].end());
        cs.pe = (int32_t)pcs.size();
        cs.wb = S.wait_off[g][(size_t)t * nC + c];
        cs.we = S.wait_off[g][(size_t)t * nC + c + 1];
        cs.mask = S.dst_mask[g][(size_t)t * nC + c];
      }
  }
  P.sync = std::move(S);
  return A2A_OK;
}

// Host emulation of the device protocol: CTAs of all GPUs run their step
// ranges in a random interleaving constrained ONLY by the dependency lists;
// memory is host memory.  Insufficient dependencies show up as wrong bytes.
// A CTA runs its step's pieces in program order (one piece per emulation
// event).  A2A_PROTO_LL: a piece with an LL source blocks until every line it
// polls carries the epoch; lines are stored and decoded in the device format.
static int emulate(Plan& P, int nC, uint8_t* const* send, uint8_t* const* recv, uint64_t seed) {
  int rc = build_sync(P, nC);
  if (rc) return rc;
  const int G = P.G, TE = P.T_exec;
  const uint32_t kEpoch = 1;
  std::vector<std::vector<uint8_t>> scratch(G), ll(G);
  for (int g = 0; g < G; ++g) {
    scratch[g].assign((size_t)P.info[g].scratch_bytes + 64, 0);
    ll[g].assign((size_t)(P.ll ? P.ll_half[g] : 0) + 64, 0);
  }
  // per-GPU flag arrays: a producer's flag is visible on GPU h only if its
  // destination mask has bit h (exactly what the kernel publishes)
  std::vector<std::vector<char>> flag(G, std::vector<char>((size_t)TE * G * nC, 0));
  // per (g, c, t): pieces in program order
  struct Piece { int32_t src_loc, dst_loc, kind; int64_t src, dst, n; };
  using Work = std::vector<std::vector<std::vector<Piece>>>;
  std::vector<Work> work(G, Work(nC, std::vector<std::vector<Piece>>(TE)));
  for (int g = 0; g < G; ++g)
    for (int t = 0; t < TE; ++t) {
      for_each_piece(P.tables[g], g, t, nC, P.remote_weight, P.gran, [&](int c, const DevItem& it, int64_t x0, int64_t x1) {
        work[g][c][t].push_back(
            Piece{it.src_loc, it.dst_loc, it.kind, piece_src(it, x0), piece_dst(it, x0), x1 - x0});
      });
    }
  auto base = [&](int g, int loc) -> uint8_t* {
    if (loc == loc_send()) return send[g];
    if (loc >= 1 && loc < 1 + G) return recv[loc - 1];
    if (loc < 1 + 2 * G) return scratch[loc - 1 - G].data();
    return ll[loc - 1 - 2 * G].data();
  };
  const bool l128 = P.ll128;
  const int64_t PL = ll_payload(l128), LB = ll_line(l128);
  auto lines_ready = [&](int g, const Piece& pc) {
    const uint8_t* L = base(g, pc.src_loc);
    for (int64_t k = pc.src / PL; k <= (pc.src + pc.n - 1) / PL; ++k) {
      if (l128) {
        uint64_t f;
        std::memcpy(&f, L + LB * k + kLL128Payload, 8);
        if (f != kEpoch) return false;
        continue;
      }
      uint32_t f0, f1;
      std::memcpy(&f0, L + 16 * k + 4, 4);
      std::memcpy(&f1, L + 16 * k + 12, 4);
      if (f0 != kEpoch || f1 != kEpoch) return false;
    }
    return true;
  };
  std::vector<std::vector<int>> next(G, std::vector<int>(nC, 0)), pos(G, std::vector<int>(nC, 0));
  uint64_t x = seed * 0x9E3779B97F4A7C15ULL + 1;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (;;) {
    std::vector<std::pair<int, int>> ready;
    bool left = false;
    for (int g = 0; g < G; ++g)
      for (int c = 0; c < nC; ++c) {
        int& t = next[g][c];
        while (t < TE && work[g][c][t].empty()) ++t;
        if (t >= TE) continue;
        left = true;
        bool ok = true;
        if (pos[g][c] == 0) {
          const auto& off = P.sync.wait_off[g];
          for (int32_t i = off[(size_t)t * nC + c]; i < off[(size_t)t * nC + c + 1] && ok; ++i)
            ok = flag[g][P.sync.wait_idx[g][i]];
        }
        const Piece& pc = work[g][c][t][pos[g][c]];
        if (ok && (pc.kind & kLLSrc)) ok = lines_ready(g, pc);
        if (ok) ready.emplace_back(g, c);
      }
    if (!left) break;
    if (ready.empty()) return fail(A2A_ERR_INVALID, "emulation deadlock: unsatisfiable dependencies");
    auto [g, c] = ready[rnd() % ready.size()];
    const int t = next[g][c];
    const Piece& pc = work[g][c][t][pos[g][c]];
    std::vector<uint8_t> buf((size_t)pc.n);
    const uint8_t* sb = base(g, pc.src_loc);
    if (pc.kind & kLLSrc) {
      for (int64_t j = 0; j < pc.n; ++j) buf[j] = sb[ll_byte(l128, pc.src + j)];
    } else {
      std::memcpy(buf.data(), sb + pc.src, (size_t)pc.n);
    }
    uint8_t* db = base(g, pc.dst_loc);
    if ((pc.kind & kLLDst) && l128) {   // whole 128-byte lines (dst on a line boundary)
      for (int64_t k = 0; k < (pc.n + PL - 1) / PL; ++k) {
        uint8_t line[kLL128Line] = {0};
        const int64_t w = std::min<int64_t>(PL, pc.n - PL * k);
        std::memcpy(line, buf.data() + PL * k, (size_t)w);
        const uint64_t f = kEpoch;
        std::memcpy(line + kLL128Payload, &f, 8);
        std::memcpy(db + LB * (pc.dst / PL + k), line, kLL128Line);
      }
    } else if (pc.kind & kLLDst) {   // whole lines (dst payload address is a multiple of 8)
      for (int64_t k = 0; k < (pc.n + 7) / 8; ++k) {
        uint8_t line[16] = {0};
        const int64_t w = std::min<int64_t>(8, pc.n - 8 * k);
        for (int64_t j = 0; j < w; ++j) line[(j < 4 ? 0 : 4) + j] = buf[8 * k + j];
        std::memcpy(line + 4, &kEpoch, 4);
        std::memcpy(line + 12, &kEpoch, 4);
        std::memcpy(db + 16 * ((pc.dst >> 3) + k), line, 16);
      }
    } else {
      std::memcpy(db + pc.dst, buf.data(), (size_t)pc.n);
    }
    if (++pos[g][c] < (int)work[g][c][t].size()) continue;
    uint32_t mask = P.sync.dst_mask[g][(size_t)t * nC + c];
    for (int h = 0; h < G; ++h)
      if (mask & (1u << h)) flag[h][((size_t)t * G + g) * nC + c] = 1;
    pos[g][c] = 0;
    ++next[g][c];
  }
  return A2A_OK;
}

// ---- dynamic unit schedule --------------------------------
//
// Items are cut into units of <= unit_bytes (multiples of 64 B from the item
// start, so src/dst stay congruent).  A unit depends on every earlier-step
// unit whose destination bytes overlap its source bytes (RAW) and, with
// scratch reuse, on earlier readers/writers of the bytes it overwrites
// (WAR/WAW).  Each GPU's list is step-major (deadlock freedom with in-order
// grabbing: a unit only waits for units of earlier steps, which precede it in
// every list); within a step units are ordered by their estimated ready time
// from a simple pipe model (NVLink egress/ingress and HBM copy per GPU).
int build_dyn(Plan& P, int nC, int64_t unit_bytes) {
  DynTables& D = P.dyn;
  if (D.nC == nC && D.unit_bytes == unit_bytes && !D.units.empty()) return A2A_OK;
  if (nC < 1) return fail(A2A_ERR_INVALID, "num_ctas must be >= 1");
  const int G = P.G, TE = P.T_exec;
  struct TU {
    DevUnit u;
    int g, t, dst_gpu;
    double ready = 0, finish = 0;
    std::vector<int> deps;
    uint32_t notify = 0;
  };
  std::vector<TU> all;
  std::vector<std::vector<std::vector<int>>> per(G, std::vector<std::vector<int>>(TE));
  for (int g = 0; g < G; ++g) {
    const GpuTables& tb = P.tables[g];
    for (int t = 0; t < TE; ++t) {
      int64_t target = unit_bytes > 0 ? unit_bytes
                                      : std::min<int64_t>(2 << 20, std::max<int64_t>(256 << 10, tb.step_bytes[t] / (2LL * nC)));
      target = std::max<int64_t>(64, std::min<int64_t>(target, 1LL << 30) & ~63LL);
      for (int64_t k = tb.step_begin[t]; k < tb.step_begin[t + 1]; ++k) {
        const DevItem& it = tb.items[k];
        // chains link local hops only; an NVLink unit pays a system-scope flag,
        // so remote items keep >= 1 MiB units in chain mode
        const int64_t tgt = (P.sched_mode >= 7 && it.dst_gpu != g) ? std::max<int64_t>(target, 1 << 20) : target;
        for (int64_t x = 0; x < it.nbytes; x += tgt) {
          TU tu;
          tu.u = DevUnit{};
          tu.u.src_off = it.src_off + x;
          tu.u.dst_off = it.dst_off + x;
          tu.u.nbytes = (int32_t)std::min(tgt, it.nbytes - x);
          tu.u.edge = it.edge;
          tu.u.src_loc = (int16_t)it.src_loc;
          tu.u.dst_loc = (int16_t)it.dst_loc;
          tu.u.step = t;
          tu.g = g;
          tu.t = t;
          tu.dst_gpu = it.dst_gpu;
          per[g][t].push_back((int)all.size());
          all.push_back(std::move(tu));
        }
      }
    }
  }
  // writes into each GPU's recv (cls 0) / scratch (cls 1), sorted, for overlap queries
  struct WS { int64_t a, b; int t, id; };
  std::vector<std::array<std::vector<WS>, 2>> ws(G);
  std::vector<std::vector<WS>> rs(G);  // scratch reads (for WAR)
  for (int i = 0; i < (int)all.size(); ++i) {
    const TU& x = all[i];
    const int h = x.dst_gpu;
    const int cls = (x.u.dst_loc == loc_recv(h)) ? 0 : 1;
    ws[h][cls].push_back(WS{x.u.dst_off, x.u.dst_off + x.u.nbytes, x.t, i});
    if (x.u.src_loc == loc_scratch(x.g, G)) rs[x.g].push_back(WS{x.u.src_off, x.u.src_off + x.u.nbytes, x.t, i});
  }
  auto prep = [](std::vector<WS>& v, std::vector<int64_t>& me) {
    std::sort(v.begin(), v.end(), [](const WS& p, const WS& q) { return p.a < q.a; });
    me.resize(v.size());
    int64_t m = INT64_MIN;
    for (size_t i = 0; i < v.size(); ++i) me[i] = m = std::max(m, v[i].b);
  };
  auto query = [](const std::vector<WS>& v, const std::vector<int64_t>& me, int64_t a, int64_t b,
                  int tmax, std::vector<int>& out) {
    size_t j = std::lower_bound(v.begin(), v.end(), b, [](const WS& s, int64_t x) { return s.a < x; }) - v.begin();
    while (j > 0) {
      --j;
      if (me[j] <= a) break;
      if (v[j].b > a && v[j].t < tmax) out.push_back(v[j].id);
    }
  };
  std::vector<std::array<std::vector<int64_t>, 2>> wme(G);
  std::vector<std::vector<int64_t>> rme(G);
  for (int h = 0; h < G; ++h) {
    prep(ws[h][0], wme[h][0]);
    prep(ws[h][1], wme[h][1]);
    prep(rs[h], rme[h]);
  }
  for (int i = 0; i < (int)all.size(); ++i) {
    TU& x = all[i];
    if (x.u.src_loc != loc_send()) {  // RAW on the executing GPU's own recv/scratch
      const int cls = (x.u.src_loc == loc_recv(x.g)) ? 0 : 1;
      query(ws[x.g][cls], wme[x.g][cls], x.u.src_off, x.u.src_off + x.u.nbytes, x.t, x.deps);
    }
    if (P.reuse && x.u.dst_loc == loc_scratch(x.dst_gpu, G)) {  // WAR / WAW
      std::vector<int> q;
      const int h = x.dst_gpu;
      query(rs[h], rme[h], x.u.dst_off, x.u.dst_off + x.u.nbytes, x.t, q);
      query(ws[h][1], wme[h][1], x.u.dst_off, x.u.dst_off + x.u.nbytes, x.t, q);
      for (int j : q) {
        x.deps.push_back(j);
        all[j].notify |= 1u << x.g;
      }
    }
    std::sort(x.deps.begin(), x.deps.end());
    x.deps.erase(std::unique(x.deps.begin(), x.deps.end()), x.deps.end());
  }
  // chain mode (sched_mode 7): a unit v whose only producer u is the previous
  // hop of the same route -- u wrote exactly v's source bytes into its own
  // GPU's scratch and v is u's only consumer -- runs right after u on the same
  // CTA: the route's hops stream through L2 (v reads what u just stored) with
  // no flag between them.  Linked units are TMA-clean (16-byte aligned
  // offsets, whole 16-byte words) and span at least one TMA ring of chunks,
  // so the ring never waits on its own stores (see the kernel's chain_body).
  std::vector<int> chain_next(all.size(), -1);
  std::vector<char> chain_prev(all.size(), 0);
  if (P.sched_mode >= 7 && !P.reuse) {
    std::vector<int> ndep(all.size(), 0);
    for (const TU& x : all)
      for (int d : x.deps) ++ndep[d];
    const int64_t min_bytes = (int64_t)std::max(1, P.tma_stages) * std::max(16, P.tma_chunk);
    for (int v = 0; v < (int)all.size(); ++v) {
      const TU& y = all[v];
      if (y.deps.size() != 1) continue;
      const int u = y.deps[0];
      const TU& x = all[u];
      if (ndep[u] != 1 || chain_next[u] >= 0 || x.g != x.dst_gpu || y.g != x.g) continue;
      if (x.u.dst_loc != loc_scratch(x.g, G) || y.u.src_loc != loc_scratch(y.g, G)) continue;
      if (x.u.dst_off != y.u.src_off || x.u.nbytes != y.u.nbytes || x.u.nbytes < min_bytes) continue;
      if ((x.u.dst_off | x.u.src_off | y.u.dst_off | x.u.nbytes) & 15) continue;
      chain_next[u] = v;
      chain_prev[v] = 1;
    }
  }
  // readiness model: remote bytes at ~700 GB/s per GPU direction, local copies at ~3.2 TB/s
  const double nv = 700e9, hbm = 3.2e12;
  std::vector<double> eg_free(G, 0), in_free(G, 0), hbm_free(G, 0);
  std::vector<double> key(all.size(), 0);   // queue order key (step-major or start time)
  auto place = [&](TU& x) {
    if (x.dst_gpu != x.g) {
      // egress AND ingress pipes: the makespan estimate is pessimistic (no
      // fluid sharing), but the resulting order spreads concurrent transfers
      // over receivers and avoids incast on one GPU (measured: GK(8,2) at 4
      // GPUs 0.70 ms vs 1.02 ms with an egress-only model)
      double st = std::max(x.ready, std::max(eg_free[x.g], in_free[x.dst_gpu]));
      x.finish = st + x.u.nbytes / nv;
      eg_free[x.g] = in_free[x.dst_gpu] = x.finish;
      return st;
    }
    double st = std::max(x.ready, hbm_free[x.g]);
    x.finish = st + x.u.nbytes / hbm;
    hbm_free[x.g] = x.finish;
    return st;
  };
  if (P.sched_mode == 2) {
    // event-driven list schedule over the unit DAG: pop the unit that becomes
    // ready first, place it on its pipe; the queue order is the start time,
    // which is a topological order (start >= ready >= producers' finish).
    // Routes then pipeline hop by hop at unit granularity (cut-through).
    std::vector<std::vector<int>> succ(all.size());
    std::vector<int> indeg(all.size(), 0);
    for (int i = 0; i < (int)all.size(); ++i)
      for (int d : all[i].deps) { succ[d].push_back(i); ++indeg[i]; }
    typedef std::pair<double, int> KI;
    std::priority_queue<KI, std::vector<KI>, std::greater<KI>> pq;
    for (int i = 0; i < (int)all.size(); ++i) {
      all[i].ready = 0;
      if (indeg[i] == 0) pq.emplace(0.0, i);
    }
    while (!pq.empty()) {
      const int id = pq.top().second;
      pq.pop();
      TU& x = all[id];
      key[id] = place(x);
      D.est_makespan = std::max(D.est_makespan, x.finish);
      for (int sx : succ[id]) {
        all[sx].ready = std::max(all[sx].ready, x.finish);
        if (--indeg[sx] == 0) pq.emplace(all[sx].ready, sx);
      }
    }
    for (int g = 0; g < G; ++g)
      for (int t = 0; t < TE; ++t)
        std::stable_sort(per[g][t].begin(), per[g][t].end(),
                         [&](int a, int b) { return key[a] < key[b]; });
  } else if (P.sched_mode == 4 || P.sched_mode == 6 || P.sched_mode >= 7) {
    // single queue, step-major; within a step the NVLink and HBM units are
    // merged in proportion to their estimated time (remote byte ~ hbm/nv local
    // bytes), each class ordered by critical path, so both pipes stay busy and
    // neither class runs ahead of the other.  Mode 6 ("spread") also
    // interleaves the NVLink units over their destination GPUs in proportion
    // to each destination's bytes, starting at g+1, so the units in flight at
    // any moment cover every peer (no incast: a critical-path order keeps one
    // source node's units together, i.e. a few destination GPUs at a time)
    std::vector<std::vector<int>> succ(all.size());
    for (int i = 0; i < (int)all.size(); ++i)
      for (int d : all[i].deps) succ[d].push_back(i);
    std::vector<double> bl(all.size(), 0.0);
    for (int t = TE - 1; t >= 0; --t)
      for (int g = 0; g < G; ++g)
        for (int id : per[g][t]) {
          double best = 0;
          for (int sx : succ[id]) best = std::max(best, bl[sx]);
          bl[id] = best + all[id].u.nbytes / (all[id].dst_gpu != all[id].g ? nv : hbm);
        }
    // chains (mode >= 7): a head costs its whole chain (it is run with its
    // linked units, which are emitted with it and cost nothing on their own step)
    auto lcost = [&](int id) -> double {
      if (P.sched_mode < 7) return all[id].u.nbytes / hbm;
      if (chain_prev[id]) return 0.0;
      double c = 0;
      for (int x = id; x >= 0; x = chain_next[x]) c += all[x].u.nbytes / hbm;
      return c;
    };
    for (int g = 0; g < G; ++g) {
      double k = 0;
      for (int t = 0; t < TE; ++t) {
        std::vector<int> rq, lq;
        double rt = 0, lt = 0;
        for (int id : per[g][t]) {
          if (all[id].dst_gpu != g) { rq.push_back(id); rt += all[id].u.nbytes / nv; }
          else { lq.push_back(id); lt += lcost(id); }
        }
        auto bysl = [&](int a, int b) { return bl[a] > bl[b]; };
        std::stable_sort(rq.begin(), rq.end(), bysl);
        std::stable_sort(lq.begin(), lq.end(), bysl);
        if (P.sched_mode == 6 && G > 2) {
          std::vector<std::vector<int>> byd(G);
          std::vector<double> tot(G, 0), done(G, 0);
          for (int id : rq) {
            byd[all[id].dst_gpu].push_back(id);
            tot[all[id].dst_gpu] += all[id].u.nbytes;
          }
          std::vector<size_t> pos(G, 0);
          rq.clear();
          for (;;) {
            int best = -1;
            double bf = 0;
            for (int k = 1; k < G; ++k) {
              const int h = (g + k) % G;
              if (pos[h] >= byd[h].size()) continue;
              const double f = done[h] / tot[h];
              if (best < 0 || f < bf) { best = h; bf = f; }
            }
            if (best < 0) break;
            const int id = byd[best][pos[best]++];
            done[best] += all[id].u.nbytes;
            rq.push_back(id);
          }
        }
        std::vector<int> merged;
        size_t i = 0, j = 0;
        double er = 0, el = 0;
        while (i < rq.size() || j < lq.size()) {
          const bool take_r = j >= lq.size() ||
                              (i < rq.size() && (rt > 0 ? er / rt : 1.0) <= (lt > 0 ? el / lt : 1.0));
          if (take_r) { er += all[rq[i]].u.nbytes / nv; merged.push_back(rq[i++]); }
          else { el += lcost(lq[j]); merged.push_back(lq[j++]); }
        }
        per[g][t] = merged;
        for (int id : per[g][t]) key[id] = k++;
      }
    }
  } else if (P.sched_mode == 3) {
    // critical-path priorities (HLFET): bottom level = own cost + the longest
    // cost chain through successors; within a step, larger bottom level first
    // (early hops of long routes before units that end a route)
    std::vector<std::vector<int>> succ(all.size());
    for (int i = 0; i < (int)all.size(); ++i)
      for (int d : all[i].deps) succ[d].push_back(i);
    std::vector<double> bl(all.size(), 0.0);
    for (int t = TE - 1; t >= 0; --t)
      for (int g = 0; g < G; ++g)
        for (int id : per[g][t]) {
          const TU& x = all[id];
          double best = 0;
          for (int sx : succ[id]) best = std::max(best, bl[sx]);
          bl[id] = best + x.u.nbytes / (x.dst_gpu != x.g ? nv : hbm);
        }
    for (int g = 0; g < G; ++g) {
      double k = 0;
      for (int t = 0; t < TE; ++t) {
        std::stable_sort(per[g][t].begin(), per[g][t].end(),
                         [&](int a, int b) { return bl[a] > bl[b]; });
        for (int id : per[g][t]) key[id] = k++;
      }
    }
  } else {
    for (int t = 0; t < TE; ++t) {
      std::vector<int> step_units;
      for (int g = 0; g < G; ++g) {
        for (int id : per[g][t]) {
          TU& x = all[id];
          x.ready = 0;
          for (int d : x.deps) x.ready = std::max(x.ready, all[d].finish);
        }
        std::stable_sort(per[g][t].begin(), per[g][t].end(), [&](int a, int b) {
          if (all[a].ready != all[b].ready) return all[a].ready < all[b].ready;
          const bool ra = all[a].dst_gpu != all[a].g, rb = all[b].dst_gpu != all[b].g;
          return ra > rb;  // remote first: NVLink is the scarce pipe
        });
        step_units.insert(step_units.end(), per[g][t].begin(), per[g][t].end());
      }
      std::stable_sort(step_units.begin(), step_units.end(),
                       [&](int a, int b) { return all[a].ready < all[b].ready; });
      for (int id : step_units) {
        place(all[id]);
        D.est_makespan = std::max(D.est_makespan, all[id].finish);
      }
    }
    // step-major key
    for (int g = 0; g < G; ++g) {
      double k = 0;
      for (int t = 0; t < TE; ++t)
        for (int id : per[g][t]) key[id] = k++;
    }
  }
  // global ids in grab order: per GPU the remote (NVLink) queue, then the local
  // (HBM) queue, each step-major; CTAs split between the queues so both pipes
  // stay busy (a CTA moves to the other queue when its own drains)
  D.unit_base.assign(G + 1, 0);
  D.n_remote.assign(G, 0);
  D.remote_ctas.assign(G, 0);
  std::vector<int> gid(all.size(), -1);
  std::vector<std::vector<int>> qorder(G);
  D.units.assign(G, {});
  D.chain_begin.assign(G, {});
  D.max_chain = 0;
  for (int g = 0; g < G; ++g) {
    double rb = 0, lb = 0;
    // one queue in key order (n_remote = 0, no CTA on queue 0): the mix order,
    // and any order with a single CTA -- two queues need a CTA each, or a CTA
    // stuck on one queue could wait for a unit only the other queue holds
    // (ready-queue mode: one array, units without dependencies first -- they
    // seed the queue -- each part in key order)
    if (P.sched_mode >= 4 || nC < 2) {
      std::vector<int> q;
      for (int t = 0; t < TE; ++t)
        for (int id : per[g][t]) q.push_back(id);
      std::stable_sort(q.begin(), q.end(), [&](int a, int b) {
        if (P.sched_mode == 5 && all[a].deps.empty() != all[b].deps.empty()) return all[a].deps.empty();
        return key[a] < key[b];
      });
      if (P.sched_mode >= 7) {
        // tasks in the order of their first unit (step-major): each chain head
        // followed by its linked units; a task only waits (at its head) on units
        // of earlier steps, whose tasks precede it in every queue
        std::vector<int> cq;
        D.chain_begin[g].clear();
        for (int id : q) {
          if (chain_prev[id]) continue;
          D.chain_begin[g].push_back((int32_t)cq.size());
          for (int x = id; x >= 0; x = chain_next[x]) cq.push_back(x);
        }
        D.chain_begin[g].push_back((int32_t)cq.size());
        D.max_chain = 1;
        for (size_t k = 0; k + 1 < D.chain_begin[g].size(); ++k)
          D.max_chain = std::max(D.max_chain, D.chain_begin[g][k + 1] - D.chain_begin[g][k]);
        q = cq;
      }
      qorder[g] = q;
      int k = 0;
      for (int id : qorder[g]) gid[id] = D.unit_base[g] + k++;
      D.unit_base[g + 1] = D.unit_base[g] + k;
      D.remote_ctas[g] = 0;
      continue;
    }
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<int> q;
      for (int t = 0; t < TE; ++t)
        for (int id : per[g][t]) {
          const bool remote = all[id].dst_gpu != g;
          if (remote != (pass == 0)) continue;
          q.push_back(id);
          (remote ? rb : lb) += all[id].u.nbytes;
          if (remote) D.n_remote[g]++;
        }
      std::stable_sort(q.begin(), q.end(), [&](int a, int b) { return key[a] < key[b]; });
      qorder[g].insert(qorder[g].end(), q.begin(), q.end());
    }
    int k = 0;
    for (int id : qorder[g]) gid[id] = D.unit_base[g] + k++;
    D.unit_base[g + 1] = D.unit_base[g] + k;
    // CTAs on the remote queue: proportional to the pipe times, at least 1/4
    // of the CTAs when there is NVLink work (remote stores need many in flight)
    const double tr = rb / nv, tl = lb / hbm;
    int nr = (tr + tl) > 0 ? (int)std::lround(nC * tr / (tr + tl)) : 0;
    if (D.n_remote[g] > 0) nr = std::max(nr, std::max(1, nC / 4));
    if (D.n_remote[g] < (int)qorder[g].size()) nr = std::min(nr, nC - std::max(1, nC / 8));
    D.remote_ctas[g] = std::max(0, std::min(nr, nC));
    if (P.dyn_remote_ctas > 0) {
      // pinned split: a fixed number of CTAs on the NVLink queue, the rest on
      // the HBM queue, and no CTA switches queues.  Fewer concurrent NVLink
      // units each finish sooner, so their dependents are ready by the time
      // they are grabbed (step overlap).  Deadlock-free as long as every
      // non-empty queue keeps >= 1 CTA (same induction as above).
      const bool has_r = D.n_remote[g] > 0, has_l = D.n_remote[g] < (int)qorder[g].size();
      D.remote_ctas[g] = !has_r ? 0 : has_l ? std::min(P.dyn_remote_ctas, nC - 1) : nC;
    }
  }
  D.pin = (P.dyn_remote_ctas > 0 && nC >= 2 && P.sched_mode < 4) ? 1 : 0;
  D.wait_idx.assign(G, {});
  D.exit_idx.assign(G, {});
  for (int g = 0; g < G; ++g)
    for (int id : qorder[g]) {
      {
        TU& x = all[id];
        DevUnit u = x.u;
        u.wb = (int32_t)D.wait_idx[g].size();
        if (!chain_prev[id])   // a linked unit's only producer ran just before it, on its CTA
          for (int d : x.deps) D.wait_idx[g].push_back(gid[d]);
        u.we = (int32_t)D.wait_idx[g].size();
        u.mask = (1u << x.dst_gpu) | x.notify;
        D.units[g].push_back(u);
        for (int h = 0; h < G; ++h)
          if (u.mask & (1u << h)) D.exit_idx[h].push_back(gid[id]);
      }
    }
  if (P.sched_mode == 5) {
    // dependents of every unit with the dependent's in-degree: a finished unit
    // counts down its dependents on their GPUs and enqueues the ones it completes
    const int total = D.unit_base[G];
    std::vector<std::vector<int32_t>> dependents(total);
    std::vector<int32_t> indeg(total, 0);
    for (int g = 0; g < G; ++g)
      for (size_t i = 0; i < D.units[g].size(); ++i) {
        const DevUnit& u = D.units[g][i];
        const int32_t me = D.unit_base[g] + (int32_t)i;
        indeg[me] = u.we - u.wb;
        for (int32_t k = u.wb; k < u.we; ++k) dependents[D.wait_idx[g][k]].push_back(me);
      }
    D.deps_out.assign(G, {});
    D.n_init.assign(G, 0);
    D.n_into.assign(G, 0);
    D.max_units = 0;
    for (int g = 0; g < G; ++g) {
      D.max_units = std::max<int32_t>(D.max_units, (int32_t)D.units[g].size());
      for (size_t i = 0; i < D.units[g].size(); ++i) {
        DevUnit& u = D.units[g][i];
        const int32_t me = D.unit_base[g] + (int32_t)i;
        if (indeg[me] == 0) D.n_init[g]++;
        u.mask = (uint32_t)indeg[me];
        u.wb = (int32_t)(D.deps_out[g].size() / 2);
        for (int32_t d : dependents[me]) {
          D.deps_out[g].push_back(d);
          D.deps_out[g].push_back(indeg[d]);
        }
        u.we = (int32_t)(D.deps_out[g].size() / 2);
      }
    }
    for (int g = 0; g < G; ++g)
      for (size_t i = 0; i < D.units[g].size(); ++i) {
        const DevUnit& u = D.units[g][i];
        const int h = u.dst_loc >= 1 && u.dst_loc < 1 + G ? u.dst_loc - 1 : u.dst_loc - 1 - G;
        D.n_into[h]++;
      }
  }
  D.nC = nC;
  D.unit_bytes = unit_bytes;
  return A2A_OK;
}

// Host emulation of the ready-queue protocol (sched_mode 5): per-GPU FIFO
// queues seeded with the dependency-free units; a CTA claims the next queue
// position, runs the unit once the position is filled, then counts down its
// dependents (on any GPU) and enqueues the ones it completes.  Claims, runs and
// releases interleave randomly across all CTAs of all GPUs; a stuck state is
// an error.
static int emulate_ready(Plan& P, int nC, uint8_t* const* send, uint8_t* const* recv,
                         uint64_t seed, int64_t unit_bytes) {
  int rc = build_dyn(P, nC, unit_bytes);
  if (rc) return rc;
  const DynTables& D = P.dyn;
  const int G = P.G;
  std::vector<std::vector<uint8_t>> scratch(G);
  for (int g = 0; g < G; ++g) scratch[g].assign((size_t)P.info[g].scratch_bytes + 64, 0);
  auto base = [&](int g, int loc) -> uint8_t* {
    if (loc == loc_send()) return send[g];
    if (loc >= 1 && loc < 1 + G) return recv[loc - 1];
    return scratch[loc - 1 - G].data();
  };
  std::vector<std::vector<int32_t>> queue(G), done(G);
  std::vector<int32_t> head(G, 0);
  for (int g = 0; g < G; ++g) {
    done[g].assign(D.units[g].size(), 0);
    for (int32_t i = 0; i < D.n_init[g]; ++i) queue[g].push_back(i);
  }
  std::vector<std::vector<int32_t>> pos(G, std::vector<int32_t>(nC, -1));   // claimed position
  uint64_t x = seed * 0x9E3779B97F4A7C15ULL + 5;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (;;) {
    std::vector<std::pair<int, int>> act;
    bool pending = false;
    for (int g = 0; g < G; ++g)
      for (int c = 0; c < nC; ++c) {
        const int32_t k = pos[g][c];
        if (k < 0) {
          if (head[g] < (int32_t)D.units[g].size()) act.emplace_back(g, c);   // claim
        } else if (k < (int32_t)queue[g].size()) {
          act.emplace_back(g, c);                                             // run
        } else {
          pending = true;                                                     // waits for its slot
        }
      }
    if (act.empty()) {
      if (pending) return fail(A2A_ERR_INVALID, "ready-queue emulation deadlock");
      break;
    }
    auto [g, c] = act[rnd() % act.size()];
    if (pos[g][c] < 0) {
      pos[g][c] = head[g]++;
      continue;
    }
    const int32_t li = queue[g][pos[g][c]];
    pos[g][c] = -1;
    const DevUnit& u = D.units[g][li];
    std::memmove(base(g, u.dst_loc) + u.dst_off, base(g, u.src_loc) + u.src_off, (size_t)u.nbytes);
    for (int32_t k = u.wb; k < u.we; ++k) {
      const int32_t gid = D.deps_out[g][2 * k], deg = D.deps_out[g][2 * k + 1];
      int h = 0;
      while (gid >= D.unit_base[h + 1]) ++h;
      const int32_t lj = gid - D.unit_base[h];
      if (++done[h][lj] == deg) queue[h].push_back(lj);
    }
  }
  for (int g = 0; g < G; ++g)
    if ((int32_t)queue[g].size() != (int32_t)D.units[g].size())
      return fail(A2A_ERR_INVALID, "ready-queue emulation: units never became ready");
  return A2A_OK;
}

// Host emulation of the dynamic protocol: CTAs grab units in list order and
// execute them once their producers' flags are visible on their GPU; random
// interleavings; a stuck state is a deadlock error.
constexpr uint32_t kEmuEpochs = 3;  // executes per emulation (counters carry across)

static int emulate_dyn(Plan& P, int nC, uint8_t* const* send, uint8_t* const* recv, uint64_t seed,
                       int64_t unit_bytes) {
  int rc = build_dyn(P, nC, unit_bytes);
  if (rc) return rc;
  const DynTables& D = P.dyn;
  const int G = P.G;
  std::vector<std::vector<uint8_t>> scratch(G);
  for (int g = 0; g < G; ++g) scratch[g].assign((size_t)P.info[g].scratch_bytes + 64, 0);
  const int total = D.unit_base[G];
  // two queues per GPU: [0, n_remote) and [n_remote, n); CTA c starts on the
  // remote queue iff c < remote_ctas[g] and switches when its queue drains
  // (unless pinned).  The grab counters persist across executes exactly as on
  // the device: a grab's queue position is counter - (epoch-1)*(units +
  // visitors), visitors = CTAs that end with one failing grab on that queue.
  std::vector<std::array<int, 2>> qn(G);
  std::vector<std::array<uint64_t, 2>> ctr(G, std::array<uint64_t, 2>{0, 0});
  for (int g = 0; g < G; ++g) qn[g] = {D.n_remote[g], (int)D.units[g].size() - D.n_remote[g]};
  auto visitors = [&](int g, int q) -> int64_t {
    return !D.pin ? nC : q == 0 ? D.remote_ctas[g] : nC - D.remote_ctas[g];
  };
  for (uint32_t epoch = 1; epoch <= kEmuEpochs; ++epoch) {
  for (int g = 0; g < G; ++g) std::fill(scratch[g].begin(), scratch[g].end(), 0);
  std::vector<std::vector<char>> flag(G, std::vector<char>((size_t)total, 0));
  std::vector<std::vector<int>> held(G, std::vector<int>(nC, -1));
  std::vector<std::vector<int>> cq(G, std::vector<int>(nC)), visited(G, std::vector<int>(nC, 0));
  std::vector<std::vector<char>> fin(G, std::vector<char>(nC, 0));
  for (int g = 0; g < G; ++g)
    for (int c = 0; c < nC; ++c) cq[g][c] = c < D.remote_ctas[g] ? 0 : 1;
  int64_t ran = 0;
  auto base = [&](int g, int loc) -> uint8_t* {
    if (loc == loc_send()) return send[g];
    if (loc >= 1 && loc < 1 + G) return recv[loc - 1];
    return scratch[loc - 1 - G].data();
  };
  // the kernel's fetch: own queue first, then the other; one failing grab per
  // visited queue; returns the unit index or -1 (CTA done)
  auto grab = [&](int g, int c) -> int {
    for (;;) {
      const int q = cq[g][c];
      const int64_t j = (int64_t)(ctr[g][q]++ - (uint64_t)(epoch - 1) * (uint64_t)(qn[g][q] + visitors(g, q)));
      if (j < 0) return -2;
      if (j < qn[g][q]) return (q == 0 ? 0 : D.n_remote[g]) + (int)j;
      if (++visited[g][c] == 2 || D.pin) return -1;
      cq[g][c] ^= 1;
    }
  };
  uint64_t x = seed * 0x9E3779B97F4A7C15ULL + 3;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
  for (;;) {
    std::vector<std::pair<int, int>> act;  // (g, c): grab or run
    bool busy = false;
    for (int g = 0; g < G; ++g)
      for (int c = 0; c < nC; ++c) {
        int u = held[g][c];
        if (u < 0) {
          if (!fin[g][c]) act.emplace_back(g, c);
          continue;
        }
        busy = true;
        const DevUnit& du = D.units[g][u];
        bool ok = true;
        for (int32_t i = du.wb; i < du.we && ok; ++i) ok = flag[g][D.wait_idx[g][i]];
        if (ok) act.emplace_back(g, c);
      }
    if (act.empty()) {
      if (busy) return fail(A2A_ERR_INVALID, "dynamic emulation deadlock");
      break;
    }
    auto [g, c] = act[rnd() % act.size()];
    if (held[g][c] < 0) {
      const int u = grab(g, c);
      if (u == -2) return fail(A2A_ERR_INVALID, "dynamic emulation: grab counter base mismatch across executes");
      if (u < 0) fin[g][c] = 1;
      else held[g][c] = u;
    } else {
      const DevUnit& du = D.units[g][held[g][c]];
      std::memmove(base(g, du.dst_loc) + du.dst_off, base(g, du.src_loc) + du.src_off, (size_t)du.nbytes);
      const int id = D.unit_base[g] + held[g][c];
      for (int h = 0; h < G; ++h)
        if (du.mask & (1u << h)) flag[h][id] = 1;
      held[g][c] = -1;
      ++ran;
    }
  }
  if (ran != total) return fail(A2A_ERR_INVALID, "dynamic emulation: units skipped in an execute");
  }
  return A2A_OK;
}

// Host emulation of the chain protocol (sched_mode 7): CTAs grab tasks (chains
// of units) from one per-GPU queue; a task waits only at its head unit (its
// dependency list), runs its units in order (one emulation event each, other
// CTAs interleave), and publishes the flags of all its units when it ends --
// exactly what chain_body does.  Three executes, persistent grab counters.
static int emulate_chain(Plan& P, int nC, uint8_t* const* send, uint8_t* const* recv, uint64_t seed,
                         int64_t unit_bytes) {
  int rc = build_dyn(P, nC, unit_bytes);
  if (rc) return rc;
  const DynTables& D = P.dyn;
  const int G = P.G;
  std::vector<std::vector<uint8_t>> scratch(G);
  for (int g = 0; g < G; ++g) scratch[g].assign((size_t)P.info[g].scratch_bytes + 64, 0);
  const int total = D.unit_base[G];
  std::vector<uint64_t> ctr(G, 0);
  for (uint32_t epoch = 1; epoch <= kEmuEpochs; ++epoch) {
    for (int g = 0; g < G; ++g) std::fill(scratch[g].begin(), scratch[g].end(), 0);
    std::vector<std::vector<char>> flag(G, std::vector<char>((size_t)total, 0));
    std::vector<std::vector<int>> task(G, std::vector<int>(nC, -1)), pos(G, std::vector<int>(nC, 0));
    std::vector<std::vector<char>> fin(G, std::vector<char>(nC, 0));
    int64_t ran = 0;
    auto base = [&](int g, int loc) -> uint8_t* {
      if (loc == loc_send()) return send[g];
      if (loc >= 1 && loc < 1 + G) return recv[loc - 1];
      return scratch[loc - 1 - G].data();
    };
    uint64_t x = seed * 0x9E3779B97F4A7C15ULL + 5;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    for (;;) {
      std::vector<std::pair<int, int>> act;
      bool busy = false;
      for (int g = 0; g < G; ++g)
        for (int c = 0; c < nC; ++c) {
          const int k = task[g][c];
          if (k < 0) {
            if (!fin[g][c]) act.emplace_back(g, c);
            continue;
          }
          busy = true;
          bool ok = true;
          if (pos[g][c] == 0) {   // the head's dependencies
            const DevUnit& du = D.units[g][D.chain_begin[g][k]];
            for (int32_t i = du.wb; i < du.we && ok; ++i) ok = flag[g][D.wait_idx[g][i]];
          }
          if (ok) act.emplace_back(g, c);
        }
      if (act.empty()) {
        if (busy) return fail(A2A_ERR_INVALID, "chain emulation deadlock");
        break;
      }
      auto [g, c] = act[rnd() % act.size()];
      if (task[g][c] < 0) {
        const int64_t nt = (int64_t)D.chain_begin[g].size() - 1;
        const int64_t j = (int64_t)(ctr[g]++ - (uint64_t)(epoch - 1) * (uint64_t)(nt + nC));
        if (j < 0) return fail(A2A_ERR_INVALID, "chain emulation: grab counter base mismatch across executes");
        if (j >= nt) fin[g][c] = 1;
        else { task[g][c] = (int)j; pos[g][c] = 0; }
        continue;
      }
      const int k = task[g][c];
      const int32_t ub = D.chain_begin[g][k], ue = D.chain_begin[g][k + 1];
      const DevUnit& du = D.units[g][ub + pos[g][c]];
      std::memmove(base(g, du.dst_loc) + du.dst_off, base(g, du.src_loc) + du.src_off, (size_t)du.nbytes);
      ++ran;
      if (ub + ++pos[g][c] < ue) continue;
      if (P.sched_mode == 8)   // discarded L2 lines read back undefined: poison the dead scratch
        for (int32_t i = ub; i + 1 < ue; ++i) {
          const DevUnit& w = D.units[g][i];
          std::memset(base(g, w.dst_loc) + w.dst_off, 0xCD, (size_t)w.nbytes);
        }
      for (int32_t i = ub; i < ue; ++i) {   // task end: every unit's flag
        const DevUnit& w = D.units[g][i];
        for (int h = 0; h < G; ++h)
          if (w.mask & (1u << h)) flag[h][D.unit_base[g] + i] = 1;
      }
      task[g][c] = -1;
    }
    if (ran != total) return fail(A2A_ERR_INVALID, "chain emulation: units skipped in an execute");
  }
  return A2A_OK;
}

}  // namespace a2a

using namespace a2a;

extern "C" {

const char* a2a_last_error(void) { return g_last_error.c_str(); }
const char* a2a_version(void) { return "b200-a2a 0.1.0 (sm_100a)"; }

int a2a_plan_create(const a2a_schedule_desc* desc, a2a_plan** out) {
  return guard([&]() -> int {
    if (!out) return fail(A2A_ERR_INVALID, "null output pointer");
    *out = nullptr;
    a2a_plan* plan = new (std::nothrow) a2a_plan();
    if (!plan) return fail(A2A_ERR_NOMEM, "out of host memory");
    int rc;
    try {
      rc = build_plan(plan->p, desc);
    } catch (const std::bad_alloc&) {
      rc = fail(A2A_ERR_NOMEM, "out of host memory building the plan");
    } catch (...) {
      rc = fail(A2A_ERR_INVALID, "internal error building the plan");
    }
    if (rc != A2A_OK) {
      delete plan;
      return rc;
    }
    g_last_error.clear();
    *out = plan;
    return A2A_OK;
  });
}

int a2a_plan_model_time(const a2a_plan* plan, double m, double b, double sync_latency,
                        double* out_T) {
  return guard([&]() -> int {
    if (!plan || !out_T) return fail(A2A_ERR_INVALID, "null argument");
    const Plan& P = plan->p;
    // evaluate.py:74, :88-107 — same float operations in the same order
    const double chunk_bytes = m / (double)P.Q;
    std::vector<double> lb(P.E, 0.0);
    std::vector<char> used(P.E, 0);
    std::unordered_map<uint64_t, int32_t> eidx;
    for (int e = 0; e < P.E; ++e)
      eidx[((uint64_t)(uint32_t)P.edge_uv[2 * e] << 32) | (uint32_t)P.edge_uv[2 * e + 1]] = e;
    double T = 0.0;
    for (int t = 0; t < P.T; ++t) {
      std::vector<int32_t> touched;
      for (int64_t i : P.step_ops[t]) {
        const a2a_op& o = P.ops[i];
        int e = eidx[((uint64_t)(uint32_t)o.src << 32) | (uint32_t)o.dst];
        if (!used[e]) { used[e] = 1; lb[e] = 0.0; touched.push_back(e); }
        lb[e] += (double)(o.c1 - o.c0) * chunk_bytes;
      }
      double step = 0.0;
      for (int e : touched) {
        double x = lb[e] / (P.cap[e] * b);
        if (x > step) step = x;
        used[e] = 0;
      }
      T += step + sync_latency;
    }
    *out_T = T;
    return A2A_OK;
  });
}

int a2a_plan_link_bytes(const a2a_plan* plan, int64_t* out) {
  return guard([&]() -> int {
    if (!plan || !out) return fail(A2A_ERR_INVALID, "null argument");
    std::memcpy(out, plan->p.link_bytes.data(), plan->p.link_bytes.size() * sizeof(int64_t));
    return A2A_OK;
  });
}

int a2a_plan_prepare(a2a_plan* plan, int32_t num_ctas) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    if (plan->p.bound && plan->p.sync.nC != num_ctas)
      return fail(A2A_ERR_STATE, "plan already bound with another CTA count");
    try {
      return build_sync(plan->p, num_ctas);
    } catch (const std::bad_alloc&) {
      return fail(A2A_ERR_NOMEM, "out of host memory building the CTA tables");
    }
  });
}

// Host audit of every device copy range (what memcheck would catch in the
// address math): each piece / unit reads inside its source buffer and writes
// inside its destination buffer on the owning GPU.
int a2a_plan_check_bounds(a2a_plan* plan, int32_t num_ctas) {
  return guard([&]() -> int {
    if (!plan) return fail(A2A_ERR_INVALID, "null plan");
    Plan& P = plan->p;
    const int G = P.G;
    int rc = P.sched_mode >= 1 ? build_dyn(P, num_ctas, P.dyn_unit_bytes) : build_sync(P, num_ctas);
    if (rc) return rc;
    auto size_of = [&](int g, int loc) -> int64_t {
      if (loc == loc_send()) return P.info[g].send_bytes;
      if (loc >= 1 && loc < 1 + G) return P.info[loc - 1].recv_bytes;
      if (loc >= 1 + G && loc < 1 + 2 * G) return P.info[loc - 1 - G].scratch_bytes;
      // LL landing region: payload capacity (lines are 16 bytes per 8 payload bytes)
      if (P.ll && loc >= 1 + 2 * G && loc < 1 + 3 * G)
        return P.ll_half[loc - 1 - 2 * G] / ll_line(P.ll128) * ll_payload(P.ll128);
      return -1;
    };
    auto check = [&](int g, int sl, int64_t so, int dl, int64_t dof, int64_t n, int kind = kCopy) -> bool {
      const bool sll = sl >= loc_ll(0, G) && sl < loc_ll(G, G), dll = dl >= loc_ll(0, G) && dl < loc_ll(G, G);
      if (sll != ((kind & kLLSrc) != 0) || dll != ((kind & kLLDst) != 0)) return false;
      const int64_t PL = ll_payload(P.ll128);
      if (dll && (dof % PL)) return false;                        // stores whole lines
      const int64_t ss = size_of(g, sl), ds = size_of(g, dl);
      const int64_t nd = dll ? (n + PL - 1) / PL * PL : n;
      return n > 0 && ss >= 0 && ds >= 0 && so >= 0 && dof >= 0 && so + n <= ss && dof + nd <= ds;
    };
    char buf[200];
    for (int g = 0; g < G; ++g) {
      if (P.sched_mode >= 1) {
        for (const DevUnit& u : P.dyn.units[g])
          if (!check(g, u.src_loc, u.src_off, u.dst_loc, u.dst_off, u.nbytes) ||
              !(u.src_loc == loc_send() || u.src_loc == loc_recv(g) || u.src_loc == loc_scratch(g, G))) {
            snprintf(buf, sizeof buf, "gpu %d: unit out of bounds (src %d+%lld, dst %d+%lld, %d B)", g,
                     u.src_loc, (long long)u.src_off, u.dst_loc, (long long)u.dst_off, u.nbytes);
            return fail(A2A_ERR_INVALID, buf);
          }
      } else {
        for (const DevPiece& q : P.sync.pieces[g])
          if (!check(g, q.src_loc, q.src_off, q.dst_loc, q.dst_off, q.nbytes, q.kind) ||
              !(q.src_loc == loc_send() || q.src_loc == loc_recv(g) || q.src_loc == loc_scratch(g, G) ||
                q.src_loc == loc_ll(g, G)) ||
              (P.ll && !(q.kind & kLLDst) && q.dst_loc != loc_recv(g))) {   // LL: plain stores stay local
            snprintf(buf, sizeof buf, "gpu %d: piece out of bounds (src %d+%lld, dst %d+%lld, %d B)", g,
                     q.src_loc, (long long)q.src_off, q.dst_loc, (long long)q.dst_off, q.nbytes);
            return fail(A2A_ERR_INVALID, buf);
          }
      }
    }
    return A2A_OK;
  });
}

int a2a_plan_set_split(a2a_plan* plan, int32_t remote_weight) {
  return guard([&]() -> int {
    if (!plan || remote_weight < 1 || remote_weight > 64) return fail(A2A_ERR_INVALID, "bad remote weight");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "set the CTA split before a2a_plan_bind");
    plan->p.remote_weight = remote_weight;
    return A2A_OK;
  });
}

int a2a_plan_set_schedule(a2a_plan* plan, int32_t mode, int64_t unit_bytes) {
  return guard([&]() -> int {
    if (!plan || mode < 0 || mode > 8 || unit_bytes < 0) return fail(A2A_ERR_INVALID, "bad schedule mode");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "set the schedule mode before a2a_plan_bind");
    if (plan->p.ll && mode != 0)
      return fail(A2A_ERR_INVALID, "A2A_PROTO_LL plans run the static schedule only");
    plan->p.sched_mode = mode;
    plan->p.dyn_unit_bytes = unit_bytes;
    plan->p.dyn = DynTables{};
    return A2A_OK;
  });
}

int a2a_plan_set_queue_split(a2a_plan* plan, int32_t remote_ctas) {
  return guard([&]() -> int {
    if (!plan || remote_ctas < 0) return fail(A2A_ERR_INVALID, "bad remote CTA count");
    if (plan->p.bound) return fail(A2A_ERR_STATE, "set the queue split before a2a_plan_bind");
    plan->p.dyn_remote_ctas = remote_ctas;
    plan->p.dyn = DynTables{};
    return A2A_OK;
  });
}

int a2a_plan_dyn_stats(a2a_plan* plan, int32_t gpu, int32_t num_ctas, int64_t* n_units,
                       int64_t* n_wait, double* est_makespan_s) {
  return guard([&]() -> int {
    if (!plan || !n_units || !n_wait || !est_makespan_s) return fail(A2A_ERR_INVALID, "null argument");
    if (gpu < 0 || gpu >= plan->p.G) return fail(A2A_ERR_INVALID, "gpu out of range");
    int rc = build_dyn(plan->p, num_ctas, plan->p.dyn_unit_bytes);
    if (rc) return rc;
    *n_units = (int64_t)plan->p.dyn.units[gpu].size();
    *n_wait = (int64_t)plan->p.dyn.wait_idx[gpu].size();
    *est_makespan_s = plan->p.dyn.est_makespan;
    return A2A_OK;
  });
}

int a2a_plan_sync_stats(const a2a_plan* plan, int32_t gpu, int64_t* n_wait, int64_t* n_exit) {
  return guard([&]() -> int {
    if (!plan || !n_wait || !n_exit) return fail(A2A_ERR_INVALID, "null argument");
    const SyncTables& S = plan->p.sync;
    if (S.nC == 0) return fail(A2A_ERR_STATE, "call a2a_plan_prepare first");
    if (gpu < 0 || gpu >= plan->p.G) return fail(A2A_ERR_INVALID, "gpu out of range");
    *n_wait = (int64_t)S.wait_idx[gpu].size();
    *n_exit = (int64_t)S.exit_idx[gpu].size();
    return A2A_OK;
  });
}

int a2a_plan_emulate(a2a_plan* plan, int32_t num_ctas, void* const* send, void* const* recv,
                     uint64_t seed) {
  return guard([&]() -> int {
    if (!plan || !send || !recv) return fail(A2A_ERR_INVALID, "null argument");
    try {
      if (plan->p.sched_mode == 5)
        return emulate_ready(plan->p, num_ctas, (uint8_t* const*)send, (uint8_t* const*)recv, seed,
                             plan->p.dyn_unit_bytes);
      if (plan->p.sched_mode >= 1)
        return plan->p.sched_mode >= 7
                   ? emulate_chain(plan->p, num_ctas, (uint8_t* const*)send, (uint8_t* const*)recv, seed,
                                   plan->p.dyn_unit_bytes)
                   : emulate_dyn(plan->p, num_ctas, (uint8_t* const*)send, (uint8_t* const*)recv, seed,
                                 plan->p.dyn_unit_bytes);
      return emulate(plan->p, num_ctas, (uint8_t* const*)send, (uint8_t* const*)recv, seed);
    } catch (const std::bad_alloc&) {
      return fail(A2A_ERR_NOMEM, "out of host memory in emulation");
    }
  });
}

// ---- placement optimiser ---------------------------
// Objective: max over GPUs of max(egress, ingress) cross-GPU bytes — the
// NVLink term of the topology bound — then total cross bytes as tie-break.
// Balanced placements only (node counts per GPU as in `placement`).
namespace {
struct PlaceEval {
  int n, E, G;
  const int32_t* uv;
  const int64_t* w;
  std::vector<std::vector<std::pair<int, int64_t>>> out_e, in_e;  // (nbr, bytes)
  void init() {
    out_e.assign(n, {});
    in_e.assign(n, {});
    for (int e = 0; e < E; ++e) {
      if (w[e] == 0) continue;
      out_e[uv[2 * e]].emplace_back(uv[2 * e + 1], w[e]);
      in_e[uv[2 * e + 1]].emplace_back(uv[2 * e], w[e]);
    }
  }
  void loads(const std::vector<int>& P, std::vector<int64_t>& eg, std::vector<int64_t>& ing,
             int64_t& cross) const {
    eg.assign(G, 0);
    ing.assign(G, 0);
    cross = 0;
    for (int e = 0; e < E; ++e) {
      int a = P[uv[2 * e]], b = P[uv[2 * e + 1]];
      if (a != b) { eg[a] += w[e]; ing[b] += w[e]; cross += w[e]; }
    }
  }
  std::pair<int64_t, int64_t> cost(const std::vector<int>& P) const {
    std::vector<int64_t> eg, ing;
    int64_t cross;
    loads(P, eg, ing, cross);
    int64_t mx = 0;
    for (int g = 0; g < G; ++g) mx = std::max(mx, std::max(eg[g], ing[g]));
    return {mx, cross};
  }
};
}  // namespace

int a2a_optimize_placement(int32_t n, int32_t n_edges, const int32_t* edge_uv,
                           const int64_t* edge_bytes, int32_t n_gpus, int32_t iters,
                           uint64_t seed, int32_t* placement) {
  return guard([&]() -> int {
    if (n < 1 || n_edges < 0 || !edge_uv || !edge_bytes || !placement || n_gpus < 1 ||
        n_gpus > A2A_MAX_GPUS)
      return fail(A2A_ERR_INVALID, "bad placement arguments");
    PlaceEval ev{n, n_edges, n_gpus, edge_uv, edge_bytes, {}, {}};
    ev.init();
    std::vector<int> P(placement, placement + n);
    for (int v = 0; v < n; ++v)
      if (P[v] < 0 || P[v] >= n_gpus) return fail(A2A_ERR_INVALID, "placement entry out of range");
    auto best = ev.cost(P);
    std::vector<int> bestP = P;
    if (n <= 12 && n_gpus > 1) {
      // exhaustive over balanced assignments with the same per-GPU counts,
      // canonical (GPU labels are interchangeable only if counts match: keep labels)
      std::vector<int> cnt(n_gpus, 0), cap(n_gpus, 0);
      for (int v = 0; v < n; ++v) cap[P[v]]++;
      std::vector<int> cur(n, 0);
      std::function<void(int)> rec = [&](int v) {
        if (v == n) {
          auto c = ev.cost(cur);
          if (c < best) { best = c; bestP = cur; }
          return;
        }
        for (int g = 0; g < n_gpus; ++g) {
          if (cnt[g] >= cap[g]) continue;
          // symmetry: the first node of each empty equal-capacity GPU goes to the lowest one
          bool skip = false;
          if (cnt[g] == 0)
            for (int h = 0; h < g; ++h)
              if (cnt[h] == 0 && cap[h] == cap[g]) { skip = true; break; }
          if (skip) continue;
          cnt[g]++;
          cur[v] = g;
          rec(v + 1);
          cnt[g]--;
        }
      };
      rec(0);
    } else if (n_gpus > 1) {
      // local search: best-improvement swaps touching the bottleneck GPU, random restarts of ties
      uint64_t x = seed * 0x9E3779B97F4A7C15ULL + 7;
      auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
      std::vector<int64_t> eg, ing;
      int64_t cross;
      for (int it = 0; it < std::max(1, iters); ++it) {
        ev.loads(P, eg, ing, cross);
        int gw = 0;
        int64_t mx = -1;
        for (int g = 0; g < n_gpus; ++g)
          if (std::max(eg[g], ing[g]) > mx) { mx = std::max(eg[g], ing[g]); gw = g; }
        std::pair<int64_t, int64_t> cbest = ev.cost(P);
        int bu = -1, bv = -1;
        // sample candidate pairs (u on the bottleneck GPU, v elsewhere)
        std::vector<int> on, off;
        for (int v = 0; v < n; ++v) (P[v] == gw ? on : off).push_back(v);
        const int samples = std::min<int64_t>((int64_t)on.size() * off.size(), 4096);
        for (int k = 0; k < samples; ++k) {
          int u = on[rnd() % on.size()], v = off[rnd() % off.size()];
          std::swap(P[u], P[v]);
          auto c = ev.cost(P);
          std::swap(P[u], P[v]);
          if (c < cbest) { cbest = c; bu = u; bv = v; }
        }
        if (bu < 0) break;
        std::swap(P[bu], P[bv]);
        if (cbest < best) { best = cbest; bestP = P; }
      }
    }
    std::copy(bestP.begin(), bestP.end(), placement);
    return A2A_OK;
  });
}

int a2a_plan_gpu_info(const a2a_plan* plan, int32_t gpu, a2a_gpu_info* out) {
  return guard([&]() -> int {
    if (!plan || !out) return fail(A2A_ERR_INVALID, "null argument");
    if (gpu < 0 || gpu >= plan->p.G) return fail(A2A_ERR_INVALID, "gpu out of range");
    *out = plan->p.info[gpu];
    return A2A_OK;
  });
}

}  // extern "C"
