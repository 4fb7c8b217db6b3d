/*
 * fj_example.c — the C-ABI used from plain C (no Python, no torch):
 * the 2-node path P2 with s = (1, 0) has z = (2/3, 1/3) (Lemma 1, P:87–89;
 * SPEC S:200) and P = 1/18, D = 1/9 (Table tab:measures).
 * Host pointers throughout: the library stages them to the device.
 *
 *   gcc -O2 -I../include fj_example.c -L../paper_2507_14864_b200 -lfj \
 *       -Wl,-rpath,$PWD/../paper_2507_14864_b200 -o fj_example
 */
#include <math.h>
#include <stdio.h>

#include "fj.h"

int main(void) {
  /* undirected edge 0–1 as the in-CSR: row 0 = {1}, row 1 = {0} */
  const int64_t row_ptr[3] = {0, 1, 2};
  const int32_t col[2] = {1, 0};
  const float s[2] = {1.0f, 0.0f};
  float z[2] = {0, 0};
  fj_graph_t g = NULL;
  if (fj_graph_create(2, 2, row_ptr, col, NULL, 0, NULL, &g) != FJ_OK) {
    fprintf(stderr, "create: %s\n", fj_last_error());
    return 1;
  }
  fj_stats st;
  fj_opts o;
  fj_opts_default(&o);
  if (fj_solve_ex(g, s, 1e-6, 1.0, &o, z, &st) != FJ_OK) {
    fprintf(stderr, "solve: %s\n", fj_last_error());
    return 1;
  }
  double P = 0, D = 0;
  if (fj_measures(g, z, &P, &D) != FJ_OK) {
    fprintf(stderr, "measures: %s\n", fj_last_error());
    return 1;
  }
  printf("z = (%.7f, %.7f)  P = %.9f  D = %.9f  sweeps = %lld  cert = %.3f\n", z[0], z[1], P, D,
         (long long)st.sweeps, st.cert_ratio);
  /* invalid input is reported, not crashed on: a self-loop */
  const int64_t rp2[2] = {0, 1};
  const int32_t c2[1] = {0};
  fj_graph_t bad = NULL;
  const fj_status rc = fj_graph_create(1, 1, rp2, c2, NULL, 1, NULL, &bad);
  printf("self-loop -> status %d (%s)\n", (int)rc, fj_last_error());
  fj_graph_destroy(g);
  const int ok = fabs(z[0] - 2.0 / 3) < 1e-6 && fabs(z[1] - 1.0 / 3) < 1e-6 &&
                 fabs(P - 1.0 / 18) < 1e-6 && fabs(D - 1.0 / 9) < 1e-6 && rc == FJ_ERR_INVALID;
  puts(ok ? "OK" : "MISMATCH");
  return ok ? 0 : 2;
}
