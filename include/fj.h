/*
 * fj.h — C-ABI of the B200-native Friedkin–Johnsen equilibrium library
 * (paper_2507_14864_b200/libfj.so, sm_100a).
 *
 * What it computes (PAPER.md, cited P:line):
 *   z = (I + L)^{-1} s                        Lemma 1, P:87–89 (§3.3)
 * with the paper's residual-threshold local iteration run to its ε rule:
 *   ImprovedBLI     = Alg. 2 around Alg. 1
 *   ImprovedBLISOR  = Alg. 2 around Alg. 3
 * executed in the Gauss–Seidel form that Theorem 3 proves
 * equivalent: every row i whose residual |r_i| exceeds its threshold h_i is
 * relaxed, ẑ_i += ω r_i/(1+d_i) (equ:sor1), until no row exceeds its
 * threshold (the paper's "while Q ≠ ∅", P:216 / P:448).  Then
 *   polarization  P(G) = Σ_i z̃_i²            Table tab:measures P:106
 *   disagreement  D(G) = Σ_{(i,j)∈E} a_ij (z_i − z_j)²
 *
 * Orientation (reading R1/R2): an arc u→v means "u listens to v"
 * (a_uv > 0); d_u = Σ_v a_uv is u's weighted out-degree.  The graph is
 * passed as an in-CSR: row v lists the u with an arc u→v.  For an undirected
 * graph both arcs of every edge are present with equal weights.
 *
 * Memory: every pointer argument may be a HOST pointer (pageable or pinned)
 * or a DEVICE pointer of the current CUDA context; the library detects which
 * (cudaPointerGetAttributes) and stages host data through device memory.
 * All device work is ordered on the graph's stream; every call returns after
 * that work has completed (it synchronises the stream).
 *
 * Errors: every call returns an fj_status; on a non-OK status
 * fj_last_error() returns a thread-local message.  Status classes follow the
 * SPEC exit codes: 2 invalid input, 3 numeric (watchdog/divergence),
 * 4 CUDA / allocation failure.
 */
#ifndef FJ_H
#define FJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FJ_ABI_VERSION 1

typedef struct fj_graph *fj_graph_t;

typedef enum {
  FJ_OK = 0,
  FJ_ERR_INVALID = 2, /* bad argument or malformed graph; nothing computed */
  FJ_ERR_NUMERIC = 3, /* watchdog or divergence sentinel; z_out holds last iterate */
  FJ_ERR_CUDA = 4     /* CUDA runtime or allocation failure */
} fj_status;

/* Sweep schedule.  All of them relax only rows with |r_i| > h_i and stop on
   the same certified rule; they differ in the order of relaxations, which
   Lemma 3 allows to be arbitrary. */
typedef enum {
  FJ_METHOD_AUTO = 0,    /* ASYNC at ω = 1 or on directed graphs, else COLORED  */
  FJ_METHOD_ASYNC = 1,   /* in-place asynchronous sweeps (chaotic Gauss–Seidel) */
  FJ_METHOD_COLORED = 2, /* multicolor Gauss–Seidel/SOR: rows of one color are
                            mutually non-adjacent, colors run in sequence, so
                            every sweep equals a sequential SOR sweep (Thm 3) */
  FJ_METHOD_PUSH = 3     /* frontier push (Alg. 1/3 data-parallel: active rows
                            scatter ω r_v a_uv/(1+d_v) to in-neighbours)        */
} fj_method;

typedef struct {
  double sigma;      /* σ of Alg. 2; <= 0 → 1e-5                        */
  double c;          /* shift c of Alg. 2; <= 0 → σ + max(0, −min s) (R5)       */
  int method;        /* fj_method                                                       */
  int max_sweeps;    /* watchdog; <= 0 → 1,000,000                              */
  int cert_rounds;   /* fp64 certificate resumes; < 0 → 3                               */
  int certify;       /* 1 (default): run the compensated fp64 residual certificate     */
  double *zprime_out;/* optional fp64[n] ẑ' = ẑ + c in node order (host or device), for
                        an independent certificate by the caller; NULL = not written    */
  const double *z_init; /* optional fp64[n] warm start (unshifted estimate of z, node
                        order, host or device), e.g. the z of an earlier solve: resume /
                        checkpoint.  Any start is valid (Lemma 3: the residual is
                        recomputed from ẑ); the ε rule and certificate are unchanged.
                        ASYNC/COLORED only (FJ_ERR_INVALID with PUSH).  NULL = start at 0
                        as Alg. 1 does                                           */
} fj_opts;

typedef struct {
  int64_t sweeps;        /* full sweeps over the active graph                           */
  int64_t phases;        /* color phases executed (= sweeps for ASYNC)                  */
  int64_t relaxations;   /* row relaxations ("number of updates")               */
  int64_t edge_updates;  /* Σ over relaxations of the row's arc count          */
  int64_t rows_read;     /* rows whose residual was evaluated                          */
  int64_t arcs_read;     /* arcs streamed by the sweep kernel                          */
  int64_t cert_rounds;   /* certificate-driven resumes                                  */
  double cert_ratio;     /* final max_v |R_v|/h_v of the fp64 certificate (≤ 1 = met)  */
  double c, eps_prime;   /* shift and ε' = σε/(c+σ) used                                */
  int colors;            /* number of color phases per sweep                            */
  int status;            /* fj_status of the solve                                      */
  int reason;            /* 0 converged, 1 watchdog, 2 divergence sentinel             */
  double solve_ms;       /* device time of the whole solve (CUDA events, graph stream) */
  double sweep_ms;       /* device time inside the sweep kernel launches               */
  double cert_ms;        /* device time inside the certificate kernel                  */
} fj_stats;

typedef struct {
  int64_t n, m;          /* nodes, stored arcs                                          */
  int directed, weighted;
  int64_t max_out_degree, empty_rows;
  int64_t tasks;         /* work items of the sweep layout                              */
  int colors;            /* 0 until a colored solve built the coloring                 */
  int num_sms;
} fj_graph_info;

typedef struct {
  double polarization;   /* P(G) = Σ z̃²                                    */
  double disagreement;   /* D(G) = Σ_E a (z_i − z_j)² (R13/R14)                  */
  double internal_conflict; /* I(G) = Σ (z − s)²; 0 if s == NULL               */
  double controversy;    /* C(G) = Σ z²                                   */
} fj_measures_t;

/* Fill *o with the defaults above. */
void fj_opts_default(fj_opts *o);

/*
 * Build a device graph (§8 row a1).  in_row_ptr: int64[n+1] with
 * in_row_ptr[0] = 0, non-decreasing, in_row_ptr[n] = nnz; in_col: int32[nnz]
 * node ids in [0, n); in_w: fp32[nnz] weights a_uv > 0 and finite, or NULL
 * for unit weights.  Rows need not be sorted.  directed = 0 requires the arc
 * set to be symmetric with equal weights.  cuda_stream: cudaStream_t (NULL =
 * legacy default stream) on which all work of this graph is ordered.
 * The library copies the arrays; the caller may free them on return.
 * FJ_ERR_INVALID: n < 1, nnz < 0, n ≥ 2^31, bad row_ptr, column out of
 * range, self-loop, duplicate arc, non-positive / non-finite weight,
 * asymmetric undirected input.
 */
fj_status fj_graph_create(int64_t n, int64_t nnz, const int64_t *in_row_ptr,
                          const int32_t *in_col, const float *in_w, int directed,
                          void *cuda_stream, fj_graph_t *out);

/* Free every device buffer of g (NULL is a no-op). */
fj_status fj_graph_destroy(fj_graph_t g);

fj_status fj_graph_get_info(fj_graph_t g, fj_graph_info *info);

/*
 * Solve for z (§8 rows a2–a6).  s: fp32[n] internal opinions (any sign; the
 * paper assumes [0,1], and Alg. 2's shift covers the rest, reading R5).
 * eps ∈ (0,1): relative error parameter.  omega ∈ (0,2): relaxation factor
 * (1 = BLI).  z_out: caller-owned fp32[n].
 * Guarantee on FJ_OK: the fp64 residual certificate holds, so
 *   |z_out_v − z_v| ≤ eps·max(|z_v|, σ) + fp32 rounding   for every v
 * (Lemma 5 P:345 / Lemma 6 P:467 with reading R5).
 * FJ_ERR_NUMERIC: watchdog or divergence (ω > 1 on a directed graph can
 * diverge; P:484 covers only the symmetric case); z_out holds the last iterate.
 */
fj_status fj_solve(fj_graph_t g, const float *s, double eps, double omega, float *z_out);

/* Extended solve: o may be NULL (defaults); st may be NULL. */
fj_status fj_solve_ex(fj_graph_t g, const float *s, double eps, double omega,
                      const fj_opts *o, float *z_out, fj_stats *st);

/*
 * Batched solve: k ∈ [1, 4] opinion vectors on one graph
 * in one set of sweeps; ẑ is kept node-major so every gathered cache line and
 * every CSR stream serves all k right-hand sides.  S and Z_out: fp32[n·k],
 * node-major (S[v·k + r]).  Every right-hand side r gets its own Alg. 2 shift
 * c_r and thresholds (reading R5), its own relax decisions, and its own fp64
 * certificate; st (nullable) reports the worst certificate ratio, the sum of
 * relaxations / edge updates over the right-hand sides, and the c of r = 0.
 * Schedule: ASYNC only (o->method AUTO or ASYNC).
 */
fj_status fj_solve_batch(fj_graph_t g, const float *S, int k, double eps, double omega,
                         const fj_opts *o, float *Z_out, fj_stats *st);

/*
 * ω selection.
 * fj_omega_opt: μ = ρ((I+D)^{-1}A) by power iteration from the
 * all-ones vector (at most max_iters SpMV sweeps, stop when the estimate moves
 * by ≤ tol relatively), then ω_opt = 1 + (μ/(1+√(1−μ²)))² (Eq. optimal-omega,
 * P:486).  The formula is the consistently-ordered SPD optimum; on directed
 * graphs it is only a guide.  Outputs are host doubles.
 */
fj_status fj_omega_opt(fj_graph_t g, int max_iters, double tol, double *mu, double *omega);

/*
 * fj_omega_sweep: the paper's heuristic: solve at ω = hi, hi − step,
 * …, down to lo, and return in *best_omega the ω with the fewest relaxations
 * ("minimum number of updates"); diverging points cost +∞, ties go to the
 * smaller ω.  table (nullable, host, 3·(*npts) doubles on entry =
 * capacity): rows (ω, relaxations, status).  *npts returns the point count.
 * method: fj_method for every solve.
 */
fj_status fj_omega_sweep(fj_graph_t g, const float *s, double eps, double lo, double hi,
                         double step, int method, double *best_omega, double *table, int *npts);

/* Polarization and disagreement of z (fp32[n]) on g (§8 row a7), fp64
   accumulation; results written to host doubles. */
fj_status fj_measures(fj_graph_t g, const float *z, double *polarization,
                      double *disagreement);

/* All four measures of tab:measures; s (fp32[n]) may be NULL. */
fj_status fj_measures_ex(fj_graph_t g, const float *z, const float *s, fj_measures_t *out);

/* Thread-local message for the last non-OK status of this thread. */
const char *fj_last_error(void);

int fj_abi_version(void);

/* Number of kernels this library has launched in this process (its own
   kernels; the CUB sort/scan/reduce primitives used by graph build and the
   opinion min/max are not counted).  Diagnostics for benchmarks. */
int64_t fj_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* FJ_H */
