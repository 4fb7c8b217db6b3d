/*
 * fj_shard_example.c — the sharded C-ABI from plain C:
 * the undirected path 0–1–2–3–4–5 split into two shards {0,1,2} and {3,4,5}
 * with the in-process transport (both shards in this process, one device),
 * solved to ε = 1e-6 and compared with fj_solve on the whole graph and with
 * the closed form of the path (Lemma 1: (I+L)z = s, solved here by
 * the Thomas algorithm for the tridiagonal system).
 *
 *   gcc -O2 -I../include fj_shard_example.c -L../paper_2507_14864_b200 -l:libfj.so \
 *       -Wl,-rpath,$PWD/../paper_2507_14864_b200 -lm -o fj_shard_example
 */
#include <math.h>
#include <stdio.h>

#include "fj.h"

#define N 6

int main(void) {
  const float s[N] = {1.0f, 0.0f, 0.5f, 0.25f, 1.0f, 0.0f};
  /* the path as one CSR (undirected: in-rows = out-rows) */
  const int64_t rp[N + 1] = {0, 1, 3, 5, 7, 9, 10};
  const int32_t col[10] = {1, 0, 2, 1, 3, 2, 4, 3, 5, 4};
  /* closed form: tridiagonal (1+d_i) z_i − z_{i−1} − z_{i+1} = s_i */
  double a[N], b[N], c[N], d[N], zc[N];
  for (int i = 0; i < N; i++) {
    a[i] = i > 0 ? -1.0 : 0.0;
    c[i] = i + 1 < N ? -1.0 : 0.0;
    b[i] = 1.0 + (double)(rp[i + 1] - rp[i]);
    d[i] = s[i];
  }
  for (int i = 1; i < N; i++) {
    const double f = a[i] / b[i - 1];
    b[i] -= f * c[i - 1];
    d[i] -= f * d[i - 1];
  }
  zc[N - 1] = d[N - 1] / b[N - 1];
  for (int i = N - 2; i >= 0; i--) zc[i] = (d[i] - c[i] * zc[i + 1]) / b[i];

  /* two shards of the out-rows: rows 0..2 and 3..5 (global column ids) */
  const int64_t begin[3] = {0, 3, 6};
  const int64_t rp0[4] = {0, 1, 3, 5}, rp1[4] = {0, 2, 4, 5};
  const int32_t c0[5] = {1, 0, 2, 1, 3}, c1[5] = {2, 4, 3, 5, 4};
  fj_comm_t comm = NULL;
  fj_shard_t sh[2] = {NULL, NULL};
  if (fj_comm_create_local(2, &comm) != FJ_OK ||
      fj_shard_create(comm, 0, N, begin, rp0, c0, NULL, 0, &sh[0]) != FJ_OK ||
      fj_shard_create(comm, 1, N, begin, rp1, c1, NULL, 0, &sh[1]) != FJ_OK ||
      fj_shard_connect(sh, 2) != FJ_OK) {
    fprintf(stderr, "setup: %s\n", fj_last_error());
    return 1;
  }
  float z0[3], z1[3];
  const float *sl[2] = {s, s + 3};
  float *zl[2] = {z0, z1};
  fj_stats st;
  if (fj_shard_solve(sh, 2, sl, 1e-6, 1.0, NULL, zl, NULL, &st) != FJ_OK) {
    fprintf(stderr, "solve: %s\n", fj_last_error());
    return 1;
  }
  int64_t nl = 0, halo = 0;
  fj_shard_info(sh[0], &nl, &halo);
  /* the whole graph through fj_solve */
  fj_graph_t g = NULL;
  float zg[N];
  if (fj_graph_create(N, 10, rp, col, NULL, 0, NULL, &g) != FJ_OK ||
      fj_solve(g, s, 1e-6, 1.0, zg) != FJ_OK) {
    fprintf(stderr, "single: %s\n", fj_last_error());
    return 1;
  }
  double err = 0.0;
  for (int i = 0; i < N; i++) {
    const double zs = i < 3 ? z0[i] : z1[i - 3];
    err = fmax(err, fabs(zs - zc[i]) / fmax(fabs(zc[i]), 1e-5));
    err = fmax(err, fabs((double)zg[i] - zc[i]) / fmax(fabs(zc[i]), 1e-5));
    printf("z[%d] shards %.7f  single %.7f  closed form %.7f\n", i, zs, zg[i], zc[i]);
  }
  printf("sweeps %lld, shard 0 owns %lld rows and reads a halo of %lld\n", (long long)st.sweeps,
         (long long)nl, (long long)halo);
  fj_graph_destroy(g);
  fj_shard_destroy(sh[0]);
  fj_shard_destroy(sh[1]);
  fj_comm_destroy(comm);
  const int ok = err < 1e-5 && halo == 1;
  puts(ok ? "OK" : "MISMATCH");
  return ok ? 0 : 2;
}
