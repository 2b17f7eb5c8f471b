/* The C ABI of include/a2a_exec.h used from plain C99 (no C++, no Python, no
 * GPU): plan creation with the reference replay's validation, modelled T,
 * per-link bytes, a rejected schedule's EvalError text, the binary op table
 * round trip and the manifest digest.  Built and run by tests/test_c_abi.py,
 * which checks the printed values against the Python binding. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "a2a_exec.h"

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  /* complete digraph on 3 nodes, edges in sorted (u, v) order */
  const int32_t uv[6][2] = {{0, 1}, {0, 2}, {1, 0}, {1, 2}, {2, 0}, {2, 1}};
  const double cap[6] = {1, 1, 1, 1, 1, 1};
  a2a_op ops[6];
  int k = 0;
  for (int s = 0; s < 3; ++s)
    for (int d = 0; d < 3; ++d)
      if (s != d) {
        a2a_op o = {0, s, d, s, d, 0, 2};
        ops[k++] = o;
      }
  a2a_schedule_desc desc;
  memset(&desc, 0, sizeof desc);
  desc.n_nodes = 3;
  desc.n_steps = 1;
  desc.q = 2;
  desc.n_edges = 6;
  desc.m_bytes = 1000;
  desc.edge_uv = &uv[0][0];
  desc.edge_cap = cap;
  desc.ops = ops;
  desc.n_ops = 6;
  desc.n_gpus = 1;
  desc.flags = A2A_COPY_SELF;
  a2a_plan* plan = NULL;
  if (a2a_plan_create(&desc, &plan) != A2A_OK) {
    printf("create failed: %s\n", a2a_last_error());
    return 1;
  }
  double T = 0;
  if (a2a_plan_model_time(plan, 3.0, 0.5, 0.25, &T) != A2A_OK) return 1;
  printf("T=%.17g\n", T);
  int64_t links[6];
  if (a2a_plan_link_bytes(plan, links) != A2A_OK) return 1;
  int64_t tot = 0;
  for (int e = 0; e < 6; ++e) tot += links[e];
  printf("link_bytes=%lld\n", (long long)tot);
  a2a_plan_destroy(plan);

  /* the first op now sends along a link the graph does not have */
  ops[0].dst = 0;
  ops[0].src = 0;
  plan = NULL;
  int rc = a2a_plan_create(&desc, &plan);
  printf("reject=%d:%s\n", rc, a2a_last_error());
  if (plan) a2a_plan_destroy(plan);
  ops[0].dst = 1;

  /* binary op table round trip + digest */
  a2a_sched_header h = {3, 1, 2, 0, 500.0};
  if (a2a_save_schedule_table(argv[1], &h, ops, 6) != A2A_OK) return 1;
  a2a_sched_header h2;
  a2a_op* back = NULL;
  int64_t n_back = 0;
  if (a2a_load_schedule_table(argv[1], &h2, &back, &n_back) != A2A_OK) return 1;
  const int same = n_back == 6 && memcmp(back, ops, sizeof ops) == 0 && h2.n == 3 &&
                   h2.nsteps == 1 && h2.q == 2 && h2.mode == 0 && h2.chunk_bytes == 500.0;
  a2a_free(back);
  printf("table=%s\n", same ? "ok" : "differs");
  char hex[65];
  if (a2a_sha256_file(argv[1], hex) != A2A_OK) return 1;
  printf("sha256=%s\n", hex);
  printf("version=%s\n", a2a_version());
  return 0;
}
