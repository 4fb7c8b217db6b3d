/*
 * oracle.c — plain, slow, single-threaded fp64 CPU oracle of the FJ hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_2507_14864_b200/) and does not import it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation /
 * algorithm named beside it); readings R1..R23 are listed in DESIGN.md §2.
 *
 * Graph input is the C-ABI in-CSR (reading R1/R2): row v lists the u with an
 * arc u→v (u listens to v) and weight a_uv (NULL = unit weights).
 * All arithmetic is IEEE fp64, compiled with -ffp-contract=off (no FMA
 * contraction), in the order the paper states.
 */
#define _POSIX_C_SOURCE 199309L
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

typedef struct {
  int64_t pushes;       /* pops of Q ("number of updates")            */
  int64_t touched;      /* Σ over pops of |N_v| (edge updates)        */
  int64_t cert_rounds;  /* residual-certificate rounds (reading R5/§8c)      */
  double cert_ratio;    /* final max_v |R_v| / h_v                            */
  double c;             /* shift constant used (Alg. 2)               */
  double eps_prime;     /* ε' = σε/(c+σ) (Alg. 2)                     */
  double seconds;       /* solve wall time (steady clock)                     */
  int status;           /* 0 ok, 3 watchdog / divergence                     */
} or_stats;

static double now_s(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec + 1e-9 * (double)t.tv_nsec;
}

static double a_of(const float *w, int64_t e) { return w ? (double)w[e] : 1.0; }

/* d_u = Σ_v a_uv ("d_i = Σ_j a_ij"); with the in-CSR, arc u→v sits in
   row v, so d_u accumulates over every row that lists u. */
void or_degrees(int64_t n, const int64_t *rp, const int32_t *col, const float *w, double *d) {
  for (int64_t u = 0; u < n; u++) d[u] = 0.0;
  for (int64_t v = 0; v < n; v++)
    for (int64_t e = rp[v]; e < rp[v + 1]; e++) d[col[e]] += a_of(w, e);
}

/* ------------------------------------------------------------ FIFO queue */
typedef struct {
  int64_t *buf, cap, head, size;
  unsigned char *inq;
} fifo;

static void q_push(fifo *q, int64_t v) {
  q->buf[(q->head + q->size) % q->cap] = v;
  q->size++;
  q->inq[v] = 1;
}
static int64_t q_pop(fifo *q) {
  int64_t v = q->buf[q->head];
  q->head = (q->head + 1) % q->cap;
  q->size--;
  q->inq[v] = 0;
  return v;
}

/*
 * Algorithm 1 BoundLocalIter, verbatim, on a caller-supplied
 * residual r (initialised to s, or s' under Alg. 2), estimate zhat and
 * boundary h ("h = ε s").  `order` lists the nodes appended to Q first
 * ("for v ∈ V: Q.append(v)"; ascending ids, reading R8).
 *   pop v; ẑ_v += r_v/(1+d_v)
 *   for u ∈ N_v: r_u += r_v/(1+d_v); if r_u > h_u and u ∉ Q: append
 *   r_v = 0
 * Weighted arcs carry a_uv on the scatter (Lemma 3 proof term A(I+D)^-1 e_v,
 * P:242; reading R3).  Returns 0, or 3 when max_pushes is exceeded.
 */
int or_bound_local_iter(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                        const double *d, double *r, double *zhat, const double *h,
                        const int64_t *order, int64_t norder, int64_t max_pushes,
                        or_stats *st) {
  fifo q = {malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1)), n > 0 ? n : 1, 0, 0,
            calloc((size_t)(n > 0 ? n : 1), 1)};
  for (int64_t i = 0; i < norder; i++)
    if (!q.inq[order[i]]) q_push(&q, order[i]);
  int rc = 0;
  while (q.size > 0) {
    if (max_pushes >= 0 && st->pushes >= max_pushes) { rc = 3; break; }
    int64_t v = q_pop(&q);
    st->pushes++;
    st->touched += rp[v + 1] - rp[v];
    double rv = r[v];
    zhat[v] = zhat[v] + rv / (1.0 + d[v]);
    for (int64_t e = rp[v]; e < rp[v + 1]; e++) {
      int64_t u = col[e];
      r[u] = r[u] + a_of(w, e) * (rv / (1.0 + d[v]));
      if (r[u] > h[u] && !q.inq[u]) q_push(&q, u);
    }
    r[v] = 0.0;
  }
  free(q.buf);
  free(q.inq);
  return rc;
}

/*
 * Algorithm 3 BoundLocalIterSOR, verbatim:
 *   pop v; ẑ_v += ω/(1+d_v) · r_v                                   (equ:sor1)
 *   for u ∈ N_v: r_u += ω/(1+d_v) · r_v; if |r_u| > h_u, u ∉ Q: append (equ:sor3)
 *   r_v = (1−ω) r_v; if |r_v| > h_v and v ∉ Q: append               (equ:sor2)
 * The divergence sentinel (‖r‖∞ > 1e6 ‖s'‖∞) is checked every n
 * pops.  Returns 0, or 3 on watchdog / divergence.
 */
int or_bound_local_iter_sor(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                            const double *d, double *r, double *zhat, const double *h,
                            double omega, const int64_t *order, int64_t norder,
                            int64_t max_pushes, double sentinel, or_stats *st) {
  fifo q = {malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1)), n > 0 ? n : 1, 0, 0,
            calloc((size_t)(n > 0 ? n : 1), 1)};
  for (int64_t i = 0; i < norder; i++)
    if (!q.inq[order[i]]) q_push(&q, order[i]);
  int rc = 0;
  int64_t since = 0;
  while (q.size > 0) {
    if (max_pushes >= 0 && st->pushes >= max_pushes) { rc = 3; break; }
    int64_t v = q_pop(&q);
    st->pushes++;
    st->touched += rp[v + 1] - rp[v];
    double rv = r[v];
    double q_v = (omega * rv) / (1.0 + d[v]); /* ω/(1+d_v)·r_v; bit-equal to Alg. 1 at ω = 1 */
    zhat[v] = zhat[v] + q_v;
    for (int64_t e = rp[v]; e < rp[v + 1]; e++) {
      int64_t u = col[e];
      r[u] = r[u] + a_of(w, e) * q_v;
      if (fabs(r[u]) > h[u] && !q.inq[u]) q_push(&q, u);
    }
    r[v] = (1.0 - omega) * rv;
    if (fabs(r[v]) > h[v] && !q.inq[v]) q_push(&q, v);
    if (++since >= n) {
      since = 0;
      double mx = 0;
      for (int64_t i = 0; i < n; i++) mx = fmax(mx, fabs(r[i]));
      if (!(mx <= sentinel)) { rc = 3; break; }
    }
  }
  free(q.buf);
  free(q.inq);
  return rc;
}

/* Neumaier compensated accumulation (for the residual certificate). */
typedef struct { double s, c; } ksum;
static void kadd(ksum *k, double x) {
  double t = k->s + x;
  if (fabs(k->s) >= fabs(x)) k->c += (k->s - t) + x;
  else k->c += (x - t) + k->s;
  k->s = t;
}
static double kval(const ksum *k) { return k->s + k->c; }
/* add the exact product a*b (TwoProduct via fma: p + err == a*b exactly) */
static void kaddprod(ksum *k, double a, double b) {
  double p = a * b;
  kadd(k, p);
  kadd(k, fma(a, b, -p));
}

/*
 * Residual of the shifted system (Lemma 3: z − ẑ = (I+L)^{-1} r, so
 * r = s' − (I+L) ẑ exactly):  R_u = s'_u − (1+d_u) ẑ_u + Σ_v a_uv ẑ_v,
 * accumulated with compensated sums.  Writes R (nullable) and returns
 * max_u |R_u| / h_u (the termination certificate, Lemma 6 proof P:474).
 */
double or_certificate(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                      const double *d, const double *sprime, const double *zhat,
                      const double *h, double *R) {
  ksum *acc = (ksum *)calloc((size_t)(n > 0 ? n : 1), sizeof(ksum));
  for (int64_t u = 0; u < n; u++) {
    kadd(&acc[u], sprime[u]);
    kadd(&acc[u], -(zhat[u]));
    kaddprod(&acc[u], -d[u], zhat[u]);
  }
  for (int64_t v = 0; v < n; v++)
    for (int64_t e = rp[v]; e < rp[v + 1]; e++) kaddprod(&acc[col[e]], a_of(w, e), zhat[v]);
  double mx = 0;
  for (int64_t u = 0; u < n; u++) {
    double x = kval(&acc[u]);
    if (R) R[u] = x;
    double ratio = fabs(x) / h[u];
    if (!(ratio <= mx)) mx = ratio; /* NaN propagates */
  }
  free(acc);
  return mx;
}

/*
 * Shift and thresholds of Algorithm 2 ImprovedBLI / ImprovedBLISOR
 * (P:330–343):  c = σ + max(0, −min s) unless overridden (reading R5),
 * ε' = σε/(c+σ), s' = s + c.
 *   s_min ≥ 0 :  h_v = ε' s'_v                     (Alg. 2 passes ε', R4)
 *   s_min < 0 :  h_v = (ε/2)·max(σ s'_v/(c+σ), σ)  (floored, reading R5)
 */
void or_thresholds(int64_t n, const float *s, double eps, double sigma, double c_override,
                   double *sprime, double *h, double *c_out, double *epsp_out) {
  double smin = INFINITY;
  for (int64_t i = 0; i < n; i++) smin = fmin(smin, (double)s[i]);
  if (n == 0) smin = 0;
  double c = c_override > 0 ? c_override : sigma + fmax(0.0, -smin);
  double epsp = sigma / (c + sigma) * eps;
  for (int64_t i = 0; i < n; i++) {
    sprime[i] = (double)s[i] + c;
    if (smin >= 0) h[i] = epsp * sprime[i];
    else h[i] = eps / 2.0 * fmax(sigma * sprime[i] / (c + sigma), sigma);
  }
  *c_out = c;
  *epsp_out = epsp;
}

/*
 * ImprovedBLI (Alg. 2 around Alg. 1, when alg == 1) or ImprovedBLISOR
 * (Alg. 2 around Alg. 3, alg == 3), then the fp64 residual certificate with
 * at most `max_cert_rounds` resumes (reading R5/§8c: r = R, enqueue the
 * violators in ascending order, continue the same loop), then ẑ = ẑ' − c
 * (P:341).
 * Outputs: z (unshifted, fp64), optional zprime (ẑ'), optional r (final
 * tracked residual), stats.  max_pushes < 0 means unbounded; a finite cap
 * returns the mid-run state (for Lemma 3 checks) with status 3.
 */
int or_improved(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                const float *s, double eps, double sigma, double c_override, double omega,
                int alg, int64_t max_pushes, int max_cert_rounds, double *z, double *zprime,
                double *r_out, or_stats *st) {
  double t0 = now_s();
  memset(st, 0, sizeof(*st));
  size_t N = (size_t)(n > 0 ? n : 1);
  double *d = malloc(sizeof(double) * N), *sp = malloc(sizeof(double) * N);
  double *h = malloc(sizeof(double) * N), *r = malloc(sizeof(double) * N);
  double *zh = calloc(N, sizeof(double)), *R = malloc(sizeof(double) * N);
  int64_t *order = malloc(sizeof(int64_t) * N);
  or_degrees(n, rp, col, w, d);
  or_thresholds(n, s, eps, sigma, c_override, sp, h, &st->c, &st->eps_prime);
  double smax = 0;
  for (int64_t i = 0; i < n; i++) {
    r[i] = sp[i]; /* r_v = s_v + c */
    order[i] = i;
    smax = fmax(smax, fabs(sp[i]));
  }
  int64_t norder = n;
  int rc = 0;
  for (;;) {
    if (alg == 1)
      rc = or_bound_local_iter(n, rp, col, w, d, r, zh, h, order, norder, max_pushes, st);
    else
      rc = or_bound_local_iter_sor(n, rp, col, w, d, r, zh, h, omega, order, norder,
                                   max_pushes, 1e6 * smax, st);
    if (rc != 0) break;
    st->cert_ratio = or_certificate(n, rp, col, w, d, sp, zh, h, R);
    if (st->cert_ratio <= 1.0 || st->cert_rounds >= max_cert_rounds) break;
    st->cert_rounds++;
    norder = 0;
    for (int64_t i = 0; i < n; i++) {
      r[i] = R[i];
      if (fabs(R[i]) > h[i]) order[norder++] = i;
    }
  }
  if (rc == 0 && st->cert_ratio > 1.0) rc = 3;
  for (int64_t i = 0; i < n; i++) {
    z[i] = zh[i] - st->c; /* ẑ_v = ẑ_v − c */
    if (zprime) zprime[i] = zh[i];
    if (r_out) r_out[i] = r[i];
  }
  st->status = rc;
  st->seconds = now_s() - t0;
  free(d); free(sp); free(h); free(r); free(zh); free(R); free(order);
  return rc;
}

/*
 * Measures of Table `tab:measures` with z̃ = z − (zᵀ1/n)1:
 *   out[0] P = Σ_i z̃_i²       (two-pass mean, reading R15)
 *   out[1] D = Σ_{(i,j)∈E} a_ij (z_i − z_j)²  (each undirected edge
 *          once = half the stored-arc sum, each directed arc once; R13/R14)
 *   out[2] I = Σ_i (z_i − s_i)²
 *   out[3] C = Σ_i z_i²
 * Compensated fp64 sums.  s may be NULL (I is then 0).
 */
void or_measures(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                 const double *z, const float *s, int directed, double *out) {
  ksum sz = {0, 0}, P = {0, 0}, D = {0, 0}, I = {0, 0}, C = {0, 0};
  for (int64_t i = 0; i < n; i++) kadd(&sz, z[i]);
  double mean = n > 0 ? kval(&sz) / (double)n : 0.0;
  for (int64_t i = 0; i < n; i++) {
    double t = z[i] - mean;
    kadd(&P, t * t);
    kadd(&C, z[i] * z[i]);
    if (s) { double u = z[i] - (double)s[i]; kadd(&I, u * u); }
  }
  for (int64_t v = 0; v < n; v++)
    for (int64_t e = rp[v]; e < rp[v + 1]; e++) {
      double t = z[col[e]] - z[v];
      kadd(&D, a_of(w, e) * t * t);
    }
  out[0] = kval(&P);
  out[1] = directed ? kval(&D) : kval(&D) / 2.0;
  out[2] = kval(&I);
  out[3] = kval(&C);
}

/* Synchronous FJ iteration, Eq. (1):
   z_i^{t+1} = (s_i + Σ_j a_ij z_j^t) / (1 + Σ_j a_ij), `iters` steps from z = s.
   A cross-check of the equilibrium of Lemma 1, not of the method. */
void or_fj_iterate(int64_t n, const int64_t *rp, const int32_t *col, const float *w,
                   const float *s, int64_t iters, double *z) {
  size_t N = (size_t)(n > 0 ? n : 1);
  double *d = malloc(sizeof(double) * N), *acc = malloc(sizeof(double) * N);
  or_degrees(n, rp, col, w, d);
  for (int64_t i = 0; i < n; i++) z[i] = (double)s[i];
  for (int64_t t = 0; t < iters; t++) {
    for (int64_t i = 0; i < n; i++) acc[i] = (double)s[i];
    for (int64_t v = 0; v < n; v++)
      for (int64_t e = rp[v]; e < rp[v + 1]; e++) acc[col[e]] += a_of(w, e) * z[v];
    for (int64_t i = 0; i < n; i++) z[i] = acc[i] / (1.0 + d[i]);
  }
  free(d);
  free(acc);
}
