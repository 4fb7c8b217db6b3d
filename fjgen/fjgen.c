/*
 * fjgen.c — seeded synthetic graph / opinion generators shared by the oracle
 * and the CUDA path.
 *
 * This module holds NO arithmetic of the Friedkin–Johnsen method: it only draws
 * graphs and internal opinions.  Both `oracle/` and the GPU library consume its
 * output; neither depends on the other.
 *
 * Output format: the in-CSR of the C-ABI (reading R1/R2):
 *   row v lists the nodes u with an arc u→v ("u listens to v", a_uv > 0),
 *   columns strictly ascending, no self-loops, no duplicates.
 *
 * RNG: counter-based SplitMix64 of (seed, stream, counter); every real value is
 * drawn in fp64 and rounded once to fp32 (reading R17).  Stream ids:
 * 0 graph, 1 opinions, 2 weights, 3 zero mask, 4 shortcuts, 5 noise.
 *
 * Parallelism: OpenMP over independent counters; results are independent of the
 * thread count (every draw is a pure function of its counter; the arc list is
 * canonicalised by sorting).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------ RNG */
static inline uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t rkey(uint64_t seed, uint64_t stream) {
  return sm64(sm64(seed) ^ (stream * 0xD1B54A32D192ED03ull + 0x8CB92BA72F3D8DD7ull));
}
static inline uint64_t ru64(uint64_t key, uint64_t ctr) { return sm64(key ^ sm64(ctr)); }
/* uniform in [0,1) with 53 random bits */
static inline double ru01(uint64_t key, uint64_t ctr) {
  return (double)(ru64(key, ctr) >> 11) * 0x1.0p-53;
}

uint64_t fjgen_u64(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return ru64(rkey(seed, stream), ctr);
}
double fjgen_u01(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return ru01(rkey(seed, stream), ctr);
}

static int nthreads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------ parallel LSD radix sort */
/* Sorts keys[0..m) ascending on bits [0, nbits).  tmp has room for m keys.
   Returns pointer to the buffer that holds the sorted result. */
static uint64_t *radix_sort_u64(uint64_t *keys, uint64_t *tmp, int64_t m, int nbits) {
  const int D = 16, R = 1 << D;
  int T = nthreads();
  int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * (size_t)R * T);
  uint64_t *src = keys, *dst = tmp;
  for (int shift = 0; shift < nbits; shift += D) {
    memset(hist, 0, sizeof(int64_t) * (size_t)R * T);
#pragma omp parallel num_threads(T)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      int64_t lo = m * t / T, hi = m * (t + 1) / T;
      int64_t *h = hist + (size_t)R * t;
      for (int64_t i = lo; i < hi; i++) h[(src[i] >> shift) & (R - 1)]++;
    }
    int64_t run = 0;
    for (int b = 0; b < R; b++)
      for (int t = 0; t < T; t++) {
        int64_t c = hist[(size_t)R * t + b];
        hist[(size_t)R * t + b] = run;
        run += c;
      }
#pragma omp parallel num_threads(T)
    {
      int t = 0;
#ifdef _OPENMP
      t = omp_get_thread_num();
#endif
      int64_t lo = m * t / T, hi = m * (t + 1) / T;
      int64_t *h = hist + (size_t)R * t;
      for (int64_t i = lo; i < hi; i++) dst[h[(src[i] >> shift) & (R - 1)]++] = src[i];
    }
    uint64_t *x = src; src = dst; dst = x;
  }
  free(hist);
  return src;
}

static int bits_for(int64_t n) {
  int b = 1;
  while (((int64_t)1 << b) < n) b++;
  return b;
}

/* Canonicalise an arc list given as keys (row << 32 | col): drop self-loops
   (row == col), sort, drop duplicates.  Writes row_ptr[n+1] and col[]; returns
   the number of unique arcs.  keys/tmp are scratch (m entries each). */
static int64_t arcs_to_csr(int64_t n, uint64_t *keys, uint64_t *tmp, int64_t m,
                           int64_t *row_ptr, int32_t *col) {
  int64_t k = 0;
  const int bn = bits_for(n);
  for (int64_t i = 0; i < m; i++) {
    uint64_t r = keys[i] >> 32, c = keys[i] & 0xffffffffull;
    if (r != c) keys[k++] = (r << bn) | c; /* compact key */
  }
  uint64_t *s = radix_sort_u64(keys, tmp, k, 2 * bn);
  uint64_t mask = ((uint64_t)1 << bn) - 1;
  int64_t u = 0;
  for (int64_t i = 0; i <= n; i++) row_ptr[i] = 0;
  for (int64_t i = 0; i < k; i++) {
    if (i > 0 && s[i] == s[i - 1]) continue;
    int64_t r = (int64_t)(s[i] >> bn);
    col[u++] = (int32_t)(s[i] & mask);
    row_ptr[r + 1]++;
  }
  for (int64_t i = 0; i < n; i++) row_ptr[i + 1] += row_ptr[i];
  return u;
}

/* ------------------------------------------------------------- graphs */

/* Undirected G(n,p): every pair i<j independently with probability p, sampled
   by geometric skipping over the linearised pair index (Batagelj–Brandes).
   Writes both arcs of each edge.  keys must hold 2*cap entries.
   Returns number of arcs written to keys (before canonicalisation), or -1. */
static int64_t er_arcs(int64_t n, double p, uint64_t seed, uint64_t *keys, int64_t cap) {
  uint64_t key = rkey(seed, 0);
  int64_t m = 0, v = 1, w = -1;
  uint64_t ctr = 0;
  double lq = log(1.0 - p);
  while (v < n) {
    double r = ru01(key, ctr++);
    w = w + 1 + (int64_t)floor(log(1.0 - r) / lq);
    while (w >= v && v < n) { w -= v; v++; }
    if (v < n) {
      if (m + 2 > cap) return -1;
      keys[m++] = ((uint64_t)v << 32) | (uint64_t)w;
      keys[m++] = ((uint64_t)w << 32) | (uint64_t)v;
    }
  }
  return m;
}

/* R-MAT: `draws` draws of `scale` levels, MSB first, quadrants (a,b,c,d):
   b and d set the dst bit, c and d set the src bit.  Arc src→dst means src
   listens to dst, so the in-CSR row is dst and the column is src. */
static void rmat_arcs(int scale, int64_t draws, double a, double b, double c,
                      uint64_t seed, uint64_t *keys) {
  uint64_t key = rkey(seed, 0);
  double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t k = 0; k < draws; k++) {
    uint64_t src = 0, dst = 0;
    for (int l = 0; l < scale; l++) {
      double u = ru01(key, (uint64_t)k * (uint64_t)scale + (uint64_t)l);
      int bit = scale - 1 - l;
      if (u < a) {
      } else if (u < ab) dst |= (uint64_t)1 << bit;
      else if (u < abc) src |= (uint64_t)1 << bit;
      else { src |= (uint64_t)1 << bit; dst |= (uint64_t)1 << bit; }
    }
    keys[k] = (dst << 32) | src;
  }
}

/* Chung–Lu expected degrees w_i = A (i + i0)^(-1/(gamma-1)), with A, i0 chosen
   so that w_0 = wmax and mean(w) = avg (bisection on i0). */
static void chunglu_weights(int64_t n, double gamma, double avg, double wmax, double *w) {
  double al = 1.0 / (gamma - 1.0);
  double lo = 1e-9, hi = 1e12;
  enum { NCH = 64 };
  for (int it = 0; it < 90; it++) {
    double i0 = sqrt(lo * hi);
    double A = wmax * pow(i0, al), part[NCH];
    /* fixed chunking: the sum is independent of the thread count */
#pragma omp parallel for schedule(static, 1)
    for (int ch = 0; ch < NCH; ch++) {
      double acc = 0;
      for (int64_t i = n * ch / NCH; i < n * (ch + 1) / NCH; i++) acc += A * pow((double)i + i0, -al);
      part[ch] = acc;
    }
    double sum = 0;
    for (int ch = 0; ch < NCH; ch++) sum += part[ch];
    /* with w_0 pinned, the mean grows with i0 (slower decay) */
    if (sum / (double)n > avg) hi = i0;
    else lo = i0;
  }
  double i0 = sqrt(lo * hi), A = wmax * pow(i0, al);
#pragma omp parallel for
  for (int64_t i = 0; i < n; i++) w[i] = A * pow((double)i + i0, -al);
}

/* Miller–Hagberg O(n+m) sampling of p_uv = min(1, w_u w_v / S), u < v, w
   non-increasing.  Per-u counter streams make it order independent.  Two
   passes: count, then write. */
static int64_t chunglu_edges_for(int64_t u, int64_t n, const double *w, double S,
                                 uint64_t key, uint64_t *out) {
  int64_t cnt = 0, v = u + 1;
  uint64_t ctr = (uint64_t)u << 24;
  if (v >= n) return 0;
  double p = fmin(w[u] * w[v] / S, 1.0);
  while (v < n && p > 0) {
    if (p != 1.0) {
      double r = ru01(key, ctr++);
      v += (int64_t)floor(log(1.0 - r) / log(1.0 - p));
    }
    if (v < n) {
      double q = fmin(w[u] * w[v] / S, 1.0);
      double r = ru01(key, ctr++);
      if (r < q / p) {
        if (out) {
          out[2 * cnt] = ((uint64_t)v << 32) | (uint64_t)u;
          out[2 * cnt + 1] = ((uint64_t)u << 32) | (uint64_t)v;
        }
        cnt++;
      }
      p = q;
      v++;
    }
  }
  return cnt;
}

/* ------------------------------------------------------------ public API */
/* All graph builders write the canonical in-CSR.  The caller passes capacity
   hints; on success return the arc count m (>=0), on failure -1.
   Two-phase use: call with row_ptr == NULL to get the arc count; then call
   again with arrays of the right size. To keep it simple every builder
   allocates its own scratch and returns a malloc'ed CSR via out-params. */

typedef struct {
  int64_t n, m;
  int64_t *row_ptr;
  int32_t *col;
} fjgen_csr;

void fjgen_free(void *p) { free(p); }

static int finish(int64_t n, uint64_t *keys, int64_t m, fjgen_csr *out) {
  uint64_t *tmp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(m > 0 ? m : 1));
  out->n = n;
  out->row_ptr = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  out->col = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
  if (!tmp || !out->row_ptr || !out->col) return -1;
  out->m = arcs_to_csr(n, keys, tmp, m, out->row_ptr, out->col);
  free(tmp);
  free(keys);
  return 0;
}

int fjgen_er(int64_t n, double p, uint64_t seed, fjgen_csr *out) {
  double mean = p * (double)n * (double)(n - 1) / 2.0;
  int64_t cap = (int64_t)(2.0 * (mean + 10.0 * sqrt(mean + 1.0) + 64.0));
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)cap);
  if (!keys) return -1;
  int64_t m = er_arcs(n, p, seed, keys, cap);
  if (m < 0) { free(keys); return -1; }
  return finish(n, keys, m, out);
}

int fjgen_rmat(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
               fjgen_csr *out) {
  int64_t n = (int64_t)1 << scale, draws = edge_factor * n;
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)draws);
  if (!keys) return -1;
  rmat_arcs(scale, draws, a, b, c, seed, keys);
  return finish(n, keys, draws, out);
}

int fjgen_chunglu(int64_t n, double gamma, double avg, double wmax, uint64_t seed,
                  fjgen_csr *out, double *wexp_out /* nullable, n */) {
  double *w = (double *)malloc(sizeof(double) * (size_t)n);
  int64_t *cnt = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!w || !cnt) return -1;
  chunglu_weights(n, gamma, avg, wmax, w);
  if (wexp_out) memcpy(wexp_out, w, sizeof(double) * (size_t)n);
  double S = 0;
  for (int64_t i = 0; i < n; i++) S += w[i];
  uint64_t key = rkey(seed, 0);
  cnt[0] = 0;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; u++) cnt[u + 1] = chunglu_edges_for(u, n, w, S, key, NULL);
  for (int64_t u = 0; u < n; u++) cnt[u + 1] += cnt[u];
  int64_t E = cnt[n];
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(2 * E + 1));
  if (!keys) return -1;
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t u = 0; u < n; u++) chunglu_edges_for(u, n, w, S, key, keys + 2 * cnt[u]);
  free(w);
  free(cnt);
  return finish(n, keys, 2 * E, out);
}

/* N×N 4-neighbour grid, id = y*N + x, plus exactly floor(frac*N*N) seeded
   nodes each given one undirected shortcut to a uniform node (redrawn on a
   self-loop or a duplicate). */
int fjgen_lattice(int64_t N, double frac, uint64_t seed, fjgen_csr *out) {
  int64_t n = N * N, k = (int64_t)floor(frac * (double)n + 1e-9);
  int64_t grid_arcs = 4 * N * (N - 1);
  uint64_t *keys = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(grid_arcs + 2 * k + 1));
  if (!keys) return -1;
  int64_t m = 0;
  for (int64_t y = 0; y < N; y++)
    for (int64_t x = 0; x < N; x++) {
      uint64_t i = (uint64_t)(y * N + x);
      if (x + 1 < N) { keys[m++] = (i << 32) | (i + 1); keys[m++] = ((i + 1) << 32) | i; }
      if (y + 1 < N) { keys[m++] = (i << 32) | (i + N); keys[m++] = ((i + N) << 32) | i; }
    }
  if (k > 0) {
    /* choose k distinct nodes: the k smallest hashes (seeded sampling without
       replacement), ties broken by id */
    uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    uint64_t key4 = rkey(seed, 4);
    int nb = bits_for(n);
#pragma omp parallel for
    for (int64_t i = 0; i < n; i++) h[i] = ((ru64(key4, (uint64_t)i) >> nb) << nb) | (uint64_t)i;
    uint64_t *srt = radix_sort_u64(h, t, n, 64);
    /* shortcut set for duplicate detection: open addressing hash */
    int64_t cap = 1;
    while (cap < 4 * k) cap <<= 1;
    uint64_t *tab = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)cap);
    for (int64_t i = 0; i < cap; i++) tab[i] = ~0ull;
    uint64_t keyd = rkey(seed, 4 ^ 0x100);
    for (int64_t j = 0; j < k; j++) {
      int64_t u = (int64_t)(srt[j] & (((uint64_t)1 << nb) - 1));
      for (uint64_t att = 0;; att++) {
        int64_t v = (int64_t)(ru64(keyd, ((uint64_t)j << 20) | att) % (uint64_t)n);
        if (v == u) continue;
        int64_t ux = u % N, uy = u / N, vx = v % N, vy = v / N;
        int64_t dx = ux > vx ? ux - vx : vx - ux, dy = uy > vy ? uy - vy : vy - uy;
        if (dx + dy == 1) continue; /* duplicate of a grid edge */
        uint64_t a = (uint64_t)(u < v ? u : v), b = (uint64_t)(u < v ? v : u);
        uint64_t e = (a << 32) | b;
        uint64_t hh = sm64(e) & (uint64_t)(cap - 1);
        int dup = 0;
        while (tab[hh] != ~0ull) {
          if (tab[hh] == e) { dup = 1; break; }
          hh = (hh + 1) & (uint64_t)(cap - 1);
        }
        if (dup) continue;
        tab[hh] = e;
        keys[m++] = ((uint64_t)u << 32) | (uint64_t)v;
        keys[m++] = ((uint64_t)v << 32) | (uint64_t)u;
        break;
      }
    }
    free(tab);
    free(h);
    free(t);
  }
  return finish(n, keys, m, out);
}

/* ---------------------------------------------------------- attributes */

/* a_uv = 1 - U(seed, 2, (u<<32)|v) in (0,1], rounded once to fp32.  Derived
   from a hash of the arc so deduplication cannot depend on draw order (R12).
   The CSR is in-CSR: row v, column u. */
void fjgen_weights(int64_t n, const int64_t *row_ptr, const int32_t *col, uint64_t seed,
                   float *w) {
  uint64_t key = rkey(seed, 2);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; v++)
    for (int64_t e = row_ptr[v]; e < row_ptr[v + 1]; e++) {
      uint64_t u = (uint64_t)col[e];
      double x = 1.0 - ru01(key, (u << 32) | (uint64_t)v);
      w[e] = (float)x;
    }
}

/* kind: 0 uniform [lo,hi); 1 Beta(2,5) as the 2nd order statistic of 6
   uniforms; 2 step 1[x < N/2] + N(0, sd^2) on an N-wide grid (lo = N, hi = sd);
   3 exponential x_min + Exp(1), max-normalised (lo = x_min);
   4 Pareto x_min (1-U)^(-1/(alpha-1)), max-normalised (lo = x_min, hi = alpha). */
void fjgen_opinions(int64_t n, int kind, double lo, double hi, uint64_t seed, float *s) {
  uint64_t k1 = rkey(seed, 1), k5 = rkey(seed, 5);
  if (kind == 0) {
#pragma omp parallel for
    for (int64_t i = 0; i < n; i++) s[i] = (float)(lo + (hi - lo) * ru01(k1, (uint64_t)i));
  } else if (kind == 1) {
#pragma omp parallel for
    for (int64_t i = 0; i < n; i++) {
      double u[6];
      for (int j = 0; j < 6; j++) u[j] = ru01(k1, (uint64_t)i * 6 + (uint64_t)j);
      /* 2nd smallest of six uniforms ~ Beta(2,5) */
      double m1 = 2, m2 = 2;
      for (int j = 0; j < 6; j++) {
        if (u[j] < m1) { m2 = m1; m1 = u[j]; }
        else if (u[j] < m2) m2 = u[j];
      }
      s[i] = (float)m2;
    }
  } else if (kind == 2) {
    int64_t N = (int64_t)lo;
    double sd = hi;
#pragma omp parallel for
    for (int64_t i = 0; i < n; i++) {
      int64_t x = i % N;
      double u1 = ru01(k5, 2 * (uint64_t)i), u2 = ru01(k5, 2 * (uint64_t)i + 1);
      double g = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2); /* Box–Muller */
      s[i] = (float)((x < N / 2 ? 1.0 : 0.0) + sd * g);
    }
  } else if (kind == 3 || kind == 4) {
    double *x = (double *)malloc(sizeof(double) * (size_t)n), mx = 0;
    for (int64_t i = 0; i < n; i++) {
      double u = ru01(k1, (uint64_t)i);
      x[i] = kind == 3 ? lo - log(1.0 - u) : lo * pow(1.0 - u, -1.0 / (hi - 1.0));
      if (x[i] > mx) mx = x[i];
    }
    for (int64_t i = 0; i < n; i++) s[i] = (float)(x[i] / mx);
    free(x);
  }
}

/* Set exactly `count` seeded entries of s to 0.0: the `count` nodes with the
   smallest hash U(seed,3,i) (sampling without replacement, reading R19). */
void fjgen_zero_mask(int64_t n, int64_t count, uint64_t seed, float *s) {
  uint64_t key = rkey(seed, 3);
  uint64_t *h = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  uint64_t *t = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
  int nb = bits_for(n);
#pragma omp parallel for
  for (int64_t i = 0; i < n; i++) h[i] = ((ru64(key, (uint64_t)i) >> nb) << nb) | (uint64_t)i;
  uint64_t *srt = radix_sort_u64(h, t, n, 64);
  for (int64_t j = 0; j < count && j < n; j++) s[srt[j] & (((uint64_t)1 << nb) - 1)] = 0.0f;
  free(h);
  free(t);
}

int fjgen_num_threads(void) { return nthreads(); }
