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
 * Threads: different graph handles may be used from different threads at
 * once (each owns its stream and workspace).  One handle must not be used by
 * two threads at the same time: a COLORED or PUSH solve builds its layout
 * lazily inside the handle.
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

#define FJ_ABI_VERSION 4

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
  /* Schedule options (defaults from fj_opts_default; none changes what is computed,
     only the order of relaxations, which Lemma 3 leaves free): */
  double tail_frac;  /* COLORED: colors after the first K whose rows total ≤ tail_frac·n
                        are merged into one bounded asynchronous phase (reading R23);
                        < 0 → 0.01, 0 → no merge (exact multicolor SOR)                 */
  int coloring;      /* COLORED: 0 = speculative first-fit in largest-first degree
                        buckets (default), 1 = Jones–Plassmann (degree priority)        */
  int push_compact;  /* PUSH: 1 = compacted frontier (ballot + slots), 0 = dense (default)*/
  int push_sparse_div; /* PUSH compacted: walk the list once the last sweep relaxed
                        < n / push_sparse_div rows; <= 0 → 8                            */
  /* The coloring and tail merge are built at the first COLORED solve of a graph and
     rebuilt if a later solve asks for a different coloring or tail_frac. */
  int shadow;        /* ASYNC/COLORED: 1 = the sweeps gather from a 32-bit fixed-point
                        shadow of ẑ' (4 B per gather) until a sweep relaxes
                        nothing or only the shadow's rounding noise, then fp64 sweeps from
                        the same ẑ' finish the ε rule (Lemma 3) and the fp64
                        certificate decides as always; 0 = fp64 sweeps only; < 0
                        (default) → 1 on hub-dominated graphs (rows above 256 arcs hold
                        over half the arcs), else 0                                     */
  int slices;        /* ASYNC/COLORED: how a sweep walks rows of ≤ 256 arcs.  1: row slices
                        — 32 rows per warp, one lane per row, arcs stored slice by slice
                        (sliced ELL), sums in registers; 0: warp tiles — a warp per ≤ 256
                        contiguous CSR arcs, products staged in shared memory; < 0
                        (default): slices, except on colored layouts that have rows above
                        32 arcs.  Same relaxations either way (the order of a row's sum
                        differs in rounding only)                                       */
  int frontier;      /* ASYNC/COLORED: the frontier phase (the paper's queue, Alg. 1
                        P:216-226, on the thin tail of a solve).  Once a sweep relaxes fewer
                        than T rows, every row's residual is written once and the push form
                        runs on the rows above threshold only: pop, scatter a·Δ to the rows
                        that gather them (fp64 atomics), list the rows that cross their
                        threshold, until the list is empty (after COLORED sweeps the pops
                        use ω = 1: the rounds are Jacobi-ordered, for which SOR carries no
                        guarantee, and Lemma 3 allows any amount).  0 = off; > 0: T; < 0
                        (default): T = non-empty rows / 256                              */
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
  int64_t shadow_sweeps; /* of `sweeps`: those that gathered from the shadow           */
  double shadow_ms;      /* of `sweep_ms`: device time of the shadow sweep launch      */
  int64_t frontier_rounds; /* pop + scatter rounds of the frontier phase                */
  int64_t frontier_pushes; /* scatter entries of those rounds (≤ 256 in-arcs each)      */
  double frontier_ms;    /* of `sweep_ms`: device time of the frontier launches        */
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
 * Batched solve (the paper runs three opinion
 * distributions per graph): k ∈ [1, 8] opinion vectors on one graph in
 * one set of sweeps (padded to K = 2, 4 or 8 internally); ẑ is kept node-major
 * so every gathered cache line and every CSR stream serves all k right-hand
 * sides.  S and Z_out: fp32[n·k], node-major (S[v·k + r]).  Every right-hand
 * side r gets its own Alg. 2 shift c_r and thresholds (reading R5), its own
 * relax decisions, and its own fp64 certificate; st (nullable) reports the
 * worst certificate ratio, the sum of relaxations / edge updates over the k
 * real right-hand sides (padding excluded), and the c of r = 0.
 * Schedule (o->method): AUTO = ASYNC at ω = 1 or on directed graphs, COLORED
 * (multicolor SOR, tail merge per o->tail_frac) for ω ≠ 1 on undirected
 * graphs, as fj_solve; ASYNC or COLORED explicitly; PUSH and z_init →
 * FJ_ERR_INVALID.  The loop stops after a sweep in which no right-hand side
 * relaxed any row; FJ_ERR_NUMERIC as fj_solve_ex.  With o->frontier != 0
 * (default) a batched sweep that relaxes fewer than T·k rows hands over to
 * the frontier phase, which finishes every right-hand side on its own (see
 * fj_opts.frontier); st->frontier_rounds / frontier_pushes sum over them.
 */
fj_status fj_solve_batch(fj_graph_t g, const float *S, int k, double eps, double omega,
                         const fj_opts *o, float *Z_out, fj_stats *st);

/*
 * ω batch (rows f1/f2): ONE opinion vector s (fp32[n]) solved at k ∈ [1, 8]
 * relaxation factors omegas[r] ∈ (0, 2) (host array) in one set of sweeps —
 * the paper's ω heuristic evaluates many ω on the same problem.
 * Z_out: fp32[n·k] node-major, column r = z at omegas[r].  A column whose
 * residual trips the divergence sentinel is frozen (no longer
 * relaxed) instead of stopping the batch: status_out[r] (nullable, host int[k])
 * = FJ_OK if column r met its certificate, FJ_ERR_NUMERIC if it diverged or
 * failed it; relax_out[r] (nullable, host int64[k]) = its relaxations (the
 * paper's "number of updates").  Schedule as fj_solve_batch (AUTO: ASYNC if all
 * ω are 1 or the graph is directed, COLORED otherwise).  Returns FJ_OK if at
 * least one column converged, FJ_ERR_NUMERIC if none did.
 */
fj_status fj_solve_batch_omega(fj_graph_t g, const float *s, int k, const double *omegas,
                               double eps, const fj_opts *o, float *Z_out, fj_stats *st,
                               int64_t *relax_out, int *status_out);

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
 * method: fj_method of the schedule (AUTO, ASYNC or COLORED; PUSH →
 * FJ_ERR_INVALID).  The grid runs as ω batches of up to 8 points
 * (fj_solve_batch_omega): every ω of one call shares one schedule (AUTO: ASYNC
 * on directed graphs, COLORED on undirected ones), so the relaxation counts
 * compare like with like.
 */
fj_status fj_omega_sweep(fj_graph_t g, const float *s, double eps, double lo, double hi,
                         double step, int method, double *best_omega, double *table, int *npts);

/* Polarization and disagreement of z (fp32[n]) on g (§8 row a7), fp64
   accumulation; results written to host doubles. */
fj_status fj_measures(fj_graph_t g, const float *z, double *polarization,
                      double *disagreement);

/* All four measures of tab:measures; s (fp32[n]) may be NULL. */
fj_status fj_measures_ex(fj_graph_t g, const float *z, const float *s, fj_measures_t *out);

/*
 * ---------------------------------------------------------------------------
 * Sharded solve: one graph split over ranks by a
 * 1-D node partition begin[0] = 0 ≤ begin[1] ≤ … ≤ begin[world] = n.  Rank r
 * owns the equations of its nodes u ∈ [begin[r], begin[r+1]) — row u of
 * (I+L)z = s (Lemma 1) reads a_uv along u's OUT-arcs u→v — and the
 * estimate ẑ_u.  Every sweep each rank relaxes its own rows exactly as
 * fj_solve's ASYNC schedule does (|r_u| > h_u), reading the other
 * ranks' ẑ from the last exchange; then every rank receives the current ẑ of
 * exactly the remote nodes its rows read (its halo) and the ranks reduce
 * (relaxations, divergence flag).  A sweep in which no rank
 * relaxes anything read only final values, so the loop ends on the paper's
 * rule (Q = ∅) exactly as on one GPU; the fp64 certificate (Lemma 3,
 * P:231) then runs on every rank and its maximum decides, with the same
 * resume rule (reading R21).  Across ranks the schedule is block-Jacobi with
 * in-place Gauss–Seidel inside each block: convergent at ω = 1 (I+L is an
 * M-matrix); ω ≠ 1 is allowed and, as with directed ASYNC, the sentinel and
 * the certificate decide.
 *
 * Transport (fj_comm): NCCL (one rank per process and GPU; ranks exchange
 * halos with grouped ncclSend/ncclRecv and reduce with ncclAllReduce over
 * NVLink/NVSwitch; libnccl.so.2 is loaded on first use), or an in-process
 * transport that holds all `world` shards of one process on the current
 * device and exchanges with device copies (single-GPU use and tests).
 */
typedef struct fj_comm *fj_comm_t;
typedef struct fj_shard *fj_shard_t;

/* Arc-balanced 1-D partition (host only, no device work).  row_ptr: HOST
   int64[n+1] of the out-CSR (row u = u's out-arcs, i.e. its work per sweep).
   Writes begin[0..world]: begin[0] = 0, begin[world] = n, every part
   non-empty (needs n ≥ world), part r ends at the first row boundary at or
   after r·(m + n)/world in units of (arcs + 1 per row).  FJ_ERR_INVALID on
   bad arguments. */
fj_status fj_shard_plan(int64_t n, const int64_t *row_ptr, int world, int64_t *begin);

/* 128-byte NCCL unique id, created on one rank and passed by the caller to
   every rank (e.g. torch.distributed broadcast of the bytes). */
fj_status fj_comm_unique_id(void *id128);
/* NCCL communicator: this process is `rank` of `world`, on the current CUDA
   device.  All work of the shards of this comm is ordered on one stream the
   comm owns. */
fj_status fj_comm_create(const void *id128, int rank, int world, fj_comm_t *out);
/* In-process transport: all `world` ranks are shards of this process on the
   current device. */
fj_status fj_comm_create_local(int world, fj_comm_t *out);
/* As fj_comm_create_local, but the exchange runs the NCCL path's own bookkeeping
   (count matrix, send lists, pack kernel, per-peer segments) and only replaces
   each ncclSend/ncclRecv pair by a device copy: the multi-rank path minus NCCL
   itself, testable on one GPU. */
fj_status fj_comm_create_loopback(int world, fj_comm_t *out);
/* Destroy a comm after every shard created on it. */
fj_status fj_comm_destroy(fj_comm_t c);

/*
 * Shard `rank` of an n-node graph: out_row_ptr int64[n_local + 1] (starting at
 * 0, n_local = begin[rank+1] − begin[rank] ≥ 1), out_col int32[nnz_local]
 * GLOBAL ids v of the arcs u→v of the owned rows (row i = node begin[rank]+i),
 * each row strictly increasing; out_w fp32 weights (> 0, finite) or NULL.
 * begin: host int64[world+1].  directed: as in fj_graph_create (an undirected
 * graph stores both arcs of every edge; symmetry across ranks is the caller's
 * contract and is not checked).  Host or device pointers; copied.
 * FJ_ERR_INVALID: bad begin / rank, empty part, bad row_ptr, id out of range,
 * self-loop, unsorted or duplicate column, bad weight, n ≥ 2^30.
 */
fj_status fj_shard_create(fj_comm_t comm, int rank, int64_t n, const int64_t *begin,
                          const int64_t *out_row_ptr, const int32_t *out_col,
                          const float *out_w, int directed, fj_shard_t *out);

/* Collective over the shards this process owns — one with an NCCL comm, all
   `world` in rank order with a local comm: exchange the sweep layouts' node
   orders and relabel remote columns.  Required once before solve/measures. */
fj_status fj_shard_connect(fj_shard_t *shards, int count);

/*
 * Collective solve over the shards this process owns (as in connect).
 * s[i]: fp32[n_local(i)] opinions of shard i's nodes; z_out[i]: fp32[n_local(i)]
 * results; zprime_out (nullable array, entries nullable): fp64 ẑ' = ẑ + c per
 * shard.  o: as fj_solve_ex (method must be AUTO/ASYNC; z_init and
 * zprime_out of o must be NULL).  st (nullable): sweeps, relaxations and edge
 * updates summed over all ranks, worst certificate ratio, device times of
 * this process.  Guarantee and statuses as fj_solve.
 */
fj_status fj_shard_solve(fj_shard_t *shards, int count, const float *const *s, double eps,
                         double omega, const fj_opts *o, float *const *z_out,
                         double *const *zprime_out, fj_stats *st);

/* Collective measures of a sharded z (fp32 slices as z_out above); s nullable
   (then I = 0).  Same definitions as fj_measures_ex. */
fj_status fj_shard_measures(fj_shard_t *shards, int count, const float *const *z,
                            const float *const *s, fj_measures_t *out);

/* Rows owned by s and, after fj_shard_connect, its halo: the number of
   distinct remote nodes its rows read, i.e. the fp64 values it receives per
   sweep (0 before connect).  Host outputs. */
fj_status fj_shard_info(fj_shard_t s, int64_t *n_local, int64_t *halo);

/* Free a shard (NULL is a no-op). */
fj_status fj_shard_destroy(fj_shard_t s);

/*
 * Practical roofline of a sweep (diagnostics): one pass over g's
 * sweep layout that streams every arc's column (and weight) and gathers one
 * fp64 value per arc at the column's index — the memory pattern of a sweep
 * without its row structure or arithmetic.  Writes the mean device time of
 * `reps` ≥ 1 passes (CUDA events on g's stream, after one warm-up pass) to
 * *ms_per_pass.  Touches no solver state.
 */
fj_status fj_gather_probe(fj_graph_t g, int reps, double *ms_per_pass);

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
