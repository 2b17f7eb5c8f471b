// Fluid performance model of one execute (a2a_plan_simulate): the exact
// per-CTA programs (static) or unit queues (dynamic orders 1-6) the device
// runs, on a machine of per-GPU resources -- NVLink egress, NVLink ingress
// (both per direction) and HBM (read + write bytes) -- with a per-CTA copy-rate
// cap, a fixed cost per unit / CTA-step, a flag latency and an optional incast
// penalty (a GPU's NVLink ingress shrinks when more CTAs than one GPU's worth
// write into it at once).  Concurrent copies
// share each resource equally per byte of demand; a copy runs at the smallest
// share over the resources it uses (or its CTA cap).  Used offline to compare
// execution orders (e.g. at 8 GPUs, which the build container cannot reach);
// calibrated against measured 1/2/4-GPU runs (tools/sim_calibrate.py).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <limits>
#include <queue>
#include <vector>

#include "a2a_internal.h"

namespace a2a {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

struct SimTask {
  double bytes = 0;        // bytes to copy
  int nres = 0;
  int res[3 * A2A_MAX_GPUS];
  double w[3 * A2A_MAX_GPUS];       // resource demand per byte copied
  std::vector<int32_t> deps;        // flag ids that must be visible before start
  int32_t flag = -1;                // flag id published on completion
};

// demand of `nb` bytes copied by GPU g into GPU h (resources: egress g,
// ingress G+g, HBM 2G+g)
void add_bytes(SimTask& t, std::vector<double>& acc, int G, int g, int h, double nb) {
  if (h != g) {
    acc[g] += nb;
    acc[G + h] += nb;
    acc[2 * G + g] += nb;
    acc[2 * G + h] += nb;
  } else {
    acc[2 * G + g] += 2 * nb;
  }
  t.bytes += nb;
}

void finish_task(SimTask& t, const std::vector<double>& acc) {
  t.nres = 0;
  if (t.bytes <= 0) return;
  for (int r = 0; r < (int)acc.size(); ++r)
    if (acc[r] > 0) {
      t.res[t.nres] = r;
      t.w[t.nres++] = acc[r] / t.bytes;
    }
}

int dst_gpu_of(int loc, int G) {
  if (loc >= 1 && loc < 1 + G) return loc - 1;
  if (loc >= 1 + G && loc < 1 + 2 * G) return loc - 1 - G;
  return -1;
}

}  // namespace

int simulate(Plan& P, int nC, const a2a_sim_params& prm, double* out) {
  if (P.ll) return fail(A2A_ERR_INVALID, "simulate: LL plans are not modelled");
  if (P.sched_mode >= 7) return fail(A2A_ERR_INVALID, "simulate: chain plans are not modelled");
  if (!(prm.nvlink_gbs > 0 && prm.hbm_gbs > 0 && prm.cta_gbs > 0))
    return fail(A2A_ERR_INVALID, "simulate: bandwidths must be positive");
  const int G = P.G, TE = P.T_exec, R = 3 * G;
  const bool dyn = P.sched_mode >= 1, ready = P.sched_mode == 5;
  int rc = dyn ? build_dyn(P, nC, P.dyn_unit_bytes) : build_sync(P, nC);
  if (rc) return rc;
  std::vector<double> cap(R);
  for (int g = 0; g < G; ++g) {
    cap[g] = cap[G + g] = prm.nvlink_gbs * 1e9;
    cap[2 * G + g] = prm.hbm_gbs * 1e9;
  }
  // ---- tasks: static = one per (g, c, t) in step order; dynamic = one per unit
  std::vector<SimTask> tasks;
  int32_t n_flags = 0;
  std::vector<double> acc(R);
  if (!dyn) {
    const SyncTables& S = P.sync;
    n_flags = TE * G * nC;
    tasks.resize((size_t)G * nC * TE);
    for (int g = 0; g < G; ++g)
      for (int c = 0; c < nC; ++c)
        for (int t = 0; t < TE; ++t) {
          SimTask& k = tasks[((size_t)g * nC + c) * TE + t];
          std::fill(acc.begin(), acc.end(), 0.0);
          const CtaStep& cs = S.prog[g][(size_t)c * TE + t];
          for (int32_t i = cs.pb; i < cs.pe; ++i) {
            const DevPiece& pc = S.pieces[g][i];
            add_bytes(k, acc, G, g, dst_gpu_of(pc.dst_loc, G), (double)pc.nbytes);
          }
          finish_task(k, acc);
          const int32_t a = S.wait_off[g][(size_t)t * nC + c], b = S.wait_off[g][(size_t)t * nC + c + 1];
          k.deps.assign(S.wait_idx[g].begin() + a, S.wait_idx[g].begin() + b);
          k.flag = (int32_t)(((int64_t)t * G + g) * nC + c);
        }
  } else {
    const DynTables& D = P.dyn;
    n_flags = D.unit_base[G];
    tasks.resize((size_t)n_flags);
    for (int g = 0; g < G; ++g)
      for (size_t i = 0; i < D.units[g].size(); ++i) {
        const DevUnit& u = D.units[g][i];
        SimTask& k = tasks[D.unit_base[g] + i];
        std::fill(acc.begin(), acc.end(), 0.0);
        add_bytes(k, acc, G, g, dst_gpu_of(u.dst_loc, G), (double)u.nbytes);
        finish_task(k, acc);
        // ready queue: a unit is enqueued only once its producers finished,
        // so it carries no waits (u.wb/we index its dependents instead)
        if (!ready) k.deps.assign(D.wait_idx[g].begin() + u.wb, D.wait_idx[g].begin() + u.we);
        k.flag = D.unit_base[g] + (int32_t)i;
      }
  }
  // ---- workers = CTAs; which task a CTA runs next
  const int W = G * nC;
  std::vector<int> step(W, 0);                  // static: next step
  std::vector<int> cq(W, 0), visited(W, 0);     // dynamic: queue state
  std::vector<std::array<int64_t, 2>> qnext(G), qend(G);
  if (dyn) {
    const DynTables& D = P.dyn;
    for (int g = 0; g < G; ++g) {
      qnext[g] = {0, D.n_remote[g]};
      qend[g] = {D.n_remote[g], (int64_t)D.units[g].size()};
      for (int c = 0; c < nC; ++c) cq[g * nC + c] = c < D.remote_ctas[g] ? 0 : 1;
    }
  }
  auto next_task = [&](int w) -> int64_t {
    const int g = w / nC, c = w % nC;
    if (!dyn) {
      if (step[w] >= TE) return -1;
      return ((int64_t)g * nC + c) * TE + step[w]++;
    }
    const DynTables& D = P.dyn;
    for (;;) {
      const int q = cq[w];
      if (qnext[g][q] < qend[g][q]) return D.unit_base[g] + qnext[g][q]++;
      if (++visited[w] == 2 || D.pin) return -1;
      cq[w] ^= 1;
    }
  };
  // ---- ready queue (mode 5): per-GPU FIFO of enqueued units; the k-th CTA
  //      to claim a position on GPU g runs the k-th unit enqueued there
  std::vector<int> ugpu, rem;
  std::vector<int64_t> claim(G, 0);
  std::vector<std::vector<int32_t>> pushed(G);
  std::vector<std::vector<int>> slot_waiter(G);
  if (ready) {
    const DynTables& D = P.dyn;
    ugpu.resize(tasks.size());
    rem.resize(tasks.size());
    for (int g = 0; g < G; ++g) {
      slot_waiter[g].assign(D.units[g].size(), -1);
      for (size_t i = 0; i < D.units[g].size(); ++i) {
        ugpu[D.unit_base[g] + i] = g;
        rem[D.unit_base[g] + i] = (int)D.units[g][i].mask;     // in-degree
      }
      for (int32_t i = 0; i < D.n_init[g]; ++i) pushed[g].push_back(D.unit_base[g] + i);
    }
  }
  // ---- event loop
  std::vector<double> flag_at((size_t)n_flags, kInf);          // visible from
  std::vector<std::vector<int>> waiters((size_t)n_flags);
  std::vector<int64_t> cur(W, -1);
  std::vector<double> left(W, 0.0), rate(W, 0.0);
  std::vector<int> running;
  typedef std::pair<double, int> Ev;                          // (time, worker): try to start
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> pq;
  double now = 0;
  int64_t done = 0;
  const int64_t total = (int64_t)tasks.size();
  const double unit_s = (G > 1 ? prm.unit_us_sys : prm.unit_us) * 1e-6, flag_s = prm.flag_us * 1e-6, cta = prm.cta_gbs * 1e9;
  for (int w = 0; w < W; ++w) pq.emplace(0.0, w);
  // per-CTA speed factor in [1 - jitter, 1 + jitter] (deterministic hash): a
  // weighted share, so CTAs do not all finish their units at the same instant
  std::vector<double> kw(W, 1.0);
  for (int w = 0; w < W; ++w) {
    uint64_t x = (uint64_t)w * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ULL; x ^= x >> 29;
    kw[w] = 1.0 + prm.jitter * (2.0 * (double)(x >> 11) / 9007199254740992.0 - 1.0);
  }
  auto try_start = [&](int w) {
    if (cur[w] < 0 && ready) {
      const int g = w / nC;
      const int64_t pos = claim[g]++;
      if (pos >= (int64_t)slot_waiter[g].size()) return;      // past the last unit: exit
      if (pos >= (int64_t)pushed[g].size()) { slot_waiter[g][pos] = w; return; }
      cur[w] = pushed[g][pos];
    }
    if (cur[w] < 0) {
      cur[w] = next_task(w);
      if (cur[w] < 0) return;
    }
    const SimTask& k = tasks[cur[w]];
    double ready = now;
    for (int32_t d : k.deps) {
      if (flag_at[d] == kInf) { waiters[d].push_back(w); return; }
      ready = std::max(ready, flag_at[d]);
    }
    if (ready > now) { pq.emplace(ready, w); return; }
    left[w] = k.bytes;
    running.push_back(w);
  };
  std::vector<double> load(R);
  std::vector<int> writers(G);
  std::vector<int> still;
  for (;;) {
    while (!pq.empty() && pq.top().first <= now) {
      const int w = pq.top().second;
      pq.pop();
      if (w >= W) {                      // ready queue: unit w - W enqueued now
        const int32_t d = w - W;
        const int h = ugpu[d];
        const size_t pos = pushed[h].size();
        pushed[h].push_back(d);
        const int x = slot_waiter[h][pos];
        if (x >= 0) {
          cur[x] = d;
          pq.emplace(now, x);
        }
        continue;
      }
      try_start(w);
    }
    // zero-byte tasks complete at once
    bool any = false;
    still.clear();
    for (int w : running) {
      if (left[w] <= 0) {
        SimTask& k = tasks[cur[w]];
        flag_at[k.flag] = now + flag_s;
        for (int x : waiters[k.flag]) pq.emplace(now + flag_s, x);
        waiters[k.flag].clear();
        if (ready) {                     // count down dependents, enqueue completed ones
          const DynTables& D = P.dyn;
          const int g = ugpu[cur[w]];
          const DevUnit& u = D.units[g][cur[w] - D.unit_base[g]];
          for (int32_t j = u.wb; j < u.we; ++j) {
            const int32_t d = D.deps_out[g][2 * (size_t)j];
            if (--rem[d] == 0) pq.emplace(now + flag_s, W + d);
          }
        }
        cur[w] = -1;
        ++done;
        pq.emplace(now + unit_s, w);
        any = true;
      } else {
        still.push_back(w);
      }
    }
    running.swap(still);
    if (any) continue;
    if (running.empty() && pq.empty()) break;
    // rates: equal share per byte of demand on every resource
    std::fill(load.begin(), load.end(), 0.0);
    std::fill(writers.begin(), writers.end(), 0);
    for (int w : running) {
      const SimTask& k = tasks[cur[w]];
      for (int i = 0; i < k.nres; ++i) {
        load[k.res[i]] += kw[w] * k.w[i];
        if (k.res[i] >= G && k.res[i] < 2 * G) ++writers[k.res[i] - G];
      }
    }
    if (prm.incast > 0)   // more concurrent writer CTAs than one GPU's worth
      for (int h = 0; h < G; ++h) {
        const double over = std::max(0.0, (double)writers[h] / nC - 1.0);
        cap[G + h] = prm.nvlink_gbs * 1e9 / (1.0 + prm.incast * over);
      }
    double dt = pq.empty() ? kInf : pq.top().first - now;
    for (int w : running) {
      const SimTask& k = tasks[cur[w]];
      double r = cta;
      for (int i = 0; i < k.nres; ++i) r = std::min(r, cap[k.res[i]] / load[k.res[i]]);
      rate[w] = kw[w] * r;
      dt = std::min(dt, left[w] / r);
    }
    if (!(dt < kInf)) return fail(A2A_ERR_INVALID, "simulate: deadlock (no runnable CTA)");
    for (int w : running) left[w] = std::max(0.0, left[w] - rate[w] * dt);
    now += dt;
    // snap copies that finish within rounding of this instant
    for (int w : running)
      if (left[w] < 1e-6 * tasks[cur[w]].bytes + 1e-3) left[w] = 0;
  }
  if (done != total) return fail(A2A_ERR_INVALID, "simulate: tasks left unfinished (deadlock)");
  *out = now + prm.launch_us * 1e-6;
  return A2A_OK;
}

}  // namespace a2a

using namespace a2a;

extern "C" {

int a2a_plan_simulate(a2a_plan* plan, int32_t num_ctas, const a2a_sim_params* params,
                      double* makespan_s) {
  return guard([&]() -> int {
    if (!plan || !params || !makespan_s) return fail(A2A_ERR_INVALID, "null argument");
    return simulate(plan->p, num_ctas, *params, makespan_s);
  });
}

}  // extern "C"
