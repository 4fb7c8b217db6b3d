// batch.cu — batched right-hand sides: k ≤ 8 opinion
// vectors share every CSR stream and every gathered ẑ line, under the ASYNC
// schedule (ω = 1, directed graphs) or the COLORED one (ω ≠ 1 on undirected
// graphs: multicolor SOR with the merged tail of reading R23, as fj_solve).
#include "sweep_common.cuh"

namespace fj {

// ------------------------------------------------- batched RHS
// K opinion vectors solved together: ẑ is stored node-major [n][K] so one
// gathered 16–32-byte line serves all K right-hand sides, and the CSR stream
// is read once per sweep for all of them.  Each RHS has its own shift c_r and
// thresholds (Alg. 2, reading R5) and its own relax decision per row.
template <int K>
__device__ __forceinline__ void gatherK(const double *__restrict__ z, int j, double (&v)[K]) {
  const double2 *q = reinterpret_cast<const double2 *>(z + (int64_t)j * K);
#pragma unroll
  for (int h = 0; h < K / 2; h++) {
    const double2 a = q[h];
    v[2 * h] = a.x;
    v[2 * h + 1] = a.y;
  }
}

// per-CTA shared state of a batched sweep: every column's shift/thresholds,
// its relaxation factor, and — for the ω batch (k values of ω for one opinion
// vector, fj_solve_batch_omega) — its divergence flag and relaxation count
struct BCtx {
  Scalars sk[8];
  double om[8];
  int bad[8];          // column diverged (ω batch): frozen, no longer relaxed
  unsigned cupd[8];    // relaxations of this CTA in the current sweep (ω batch)
  int omb;             // ω batch mode
};

template <int K>
__device__ __forceinline__ void relax_rowK(const KP &p, BCtx *bc, int row, int len,
                                           dd (&tot)[K], const float (&sv)[K],
                                           const double (&zi)[K], double d1, TAcc &t) {
  double out[K];
#pragma unroll
  for (int r = 0; r < K; r++) {
    const Scalars &S = bc->sk[r];
    const double sp = (double)sv[r] + S.c;
    const double h = threshold(S, sp);
    const double rho = residual_dd(tot[r], sp, d1, zi[r]);
    const double ar = fabs(rho);
    out[r] = zi[r];
    if (ar > p.theta * h && !bc->bad[r]) {
      // tail phase (R23): ω_i = min(ω, 1.98/(1+β_i)), as relax_row_pre
      double om = bc->om[r];
      if (row >= p.tail_row0 && row < p.tail_row1)
        om = fmin(om, 1.98 / (1.0 + (double)p.tail_beta[row - p.tail_row0]));
      out[r] = zi[r] + om * rho / d1;
      if (r < p.kreal) {  // padded right-hand sides relax but do not count
        t.upd++;
        t.eu += (unsigned long long)len;
        if (bc->omb) atomicAdd(&bc->cupd[r], 1u);
      }
    }
    if (!(ar <= S.sentinel)) {  // divergence sentinel
      if (bc->omb) atomicOr(p.colbad + r, 1);  // ω batch: this column only
      else t.bad = 1;
    }
  }
  double2 *q = reinterpret_cast<double2 *>(p.z + (int64_t)row * K);
#pragma unroll
  for (int h = 0; h < K / 2; h++) __stcg(q + h, make_double2(out[2 * h], out[2 * h + 1]));
}

// warp unit (row > kWarpTileArcs arcs, or a piece of one), K right-hand sides;
// U·K gathered values in flight per lane (U = 4, 2, 1 arcs for K = 2, 4, 8)
// Arcs in flight per lane (warp units FJ_BU*, tiles FJ_BT*) and CTAs per SM at
// K = 4; build-time knobs of the batched kernel, defaults measured on C4/C5
// (profiles/r02_batch_ab.txt: K = 8 at 2 arcs 6.69 vs 8.07 ms per C4 sweep at
// 1; K = 4 at 3 CTAs/SM 3.75, at 2 (no spills) 3.71 but +22 % sweeps, at 4 3.67).
#ifndef FJ_BU4
#define FJ_BU4 2
#endif
#ifndef FJ_BU8
#define FJ_BU8 2
#endif
#ifndef FJ_BT4
#define FJ_BT4 2
#endif
#ifndef FJ_BT8
#define FJ_BT8 2
#endif
#ifndef FJ_BMIN4
#define FJ_BMIN4 3
#endif
template <bool W, int K>
__device__ __forceinline__ void do_warpK(const KP &p, BCtx *bc, const Task &tk, TAcc &t) {
  constexpr int U = K >= 8 ? FJ_BU8 : (K >= 4 ? FJ_BU4 : 4);
  const int lane = threadIdx.x & 31;
  const int row = tk.a, piece = tk.b, np = tk.kind >> 8, slot = tk.slot;
  const int64_t a0 = tk.a0, a1 = tk.a1;
  // row state on lanes: 1..K s, K+1..2K ẑ, 2K+1 d1, 2K+2/2K+3 row_ptr
  double pre = 0.0;
  if (lane >= 1 && lane <= K) pre = (double)__ldg(p.s + (int64_t)row * K + lane - 1);
  else if (lane > K && lane <= 2 * K) pre = __ldcg(p.z + (int64_t)row * K + lane - K - 1);
  else if (lane == 2 * K + 1 && W) pre = __ldg(p.d1 + row);
  else if (lane == 2 * K + 2) pre = (double)__ldg(p.rp + row);
  else if (lane == 2 * K + 3) pre = (double)__ldg(p.rp + row + 1);
  dd a[K];
#pragma unroll
  for (int r = 0; r < K; r++) a[r] = dd{0.0, 0.0};
  for (int64_t k0 = a0 + lane; k0 < a1; k0 += 32 * U) {
    int j[U];
    float wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t k = k0 + 32 * u;
      const bool ok = k < a1;
      j[u] = ld_stream(p.col + (ok ? k : a0));
      wv[u] = W ? ld_stream(p.w + (ok ? k : a0)) : 1.0f;  // clamped: never speculate past the row
      if (!ok) wv[u] = 0.0f;
    }
    double zj[U][K];
#pragma unroll
    for (int u = 0; u < U; u++) gatherK<K>(p.z, j[u], zj[u]);
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int r = 0; r < K; r++) dd_addprod(a[r], (double)wv[u], zj[u][r]);
  }
#pragma unroll
  for (int r = 0; r < K; r++)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc_merge(a[r], acc_shfl(a[r], 0xffffffffu, off));
  float sv[K];
  double zi[K];
#pragma unroll
  for (int r = 0; r < K; r++) {
    sv[r] = (float)__shfl_sync(0xffffffffu, pre, 1 + r);
    zi[r] = __shfl_sync(0xffffffffu, pre, 1 + K + r);
  }
  const double rbv = __shfl_sync(0xffffffffu, pre, 2 * K + 2);
  const double rev = __shfl_sync(0xffffffffu, pre, 2 * K + 3);
  const int len = (int)(rev - rbv);
  const double d1 = W ? __shfl_sync(0xffffffffu, pre, 2 * K + 1) : (double)(len + 1);
  if (lane != 0) return;
  if (np > 1) {
#pragma unroll
    for (int r = 0; r < K; r++)
      __stcg(p.partial + ((int64_t)slot + piece) * K + r, make_double2(a[r].hi, a[r].lo));
    const int old = arrive_release(p.arrive + slot);  // no L1 flush (sweep_common.cuh)
    if ((old + 1) % np != 0) return;
#pragma unroll
    for (int r = 0; r < K; r++) a[r] = dd{0.0, 0.0};
    for (int q = 0; q < np; q++)
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 x = ld_partial(p.partial + ((int64_t)slot + q) * K + r);
        acc_merge(a[r], dd{x.x, x.y});
      }
  }
  relax_rowK<K>(p, bc, row, len, a, sv, zi, d1, t);
}

// warp tile (short rows), K right-hand sides: G lanes per row accumulate
// directly in registers (no shared memory), two row steps
template <bool W, int K>
__device__ __forceinline__ void tileK(const KP &p, BCtx *bc, const Task &tk, TAcc &t) {
  const int lane = threadIdx.x & 31;
  const int cls = tk.kind & 0xff;
  const int G = 1 << cls;
  const int gl = lane & (G - 1);
  const int ng = 32 >> cls;
#pragma unroll 1
  for (int q = 0; q < 2; q++) {
    const int row = tk.a + q * ng + (lane >> cls);
    const bool has = row < tk.b;
    int64_t rb = 0, re = 0;
    float sv[K];
    double zi[K], d1 = 0.0;
#pragma unroll
    for (int r = 0; r < K; r++) {
      sv[r] = 0.f;
      zi[r] = 0.0;
    }
    if (has) {
      rb = __ldg(p.rp + row);
      re = __ldg(p.rp + row + 1);
      if (gl == 0) {
#pragma unroll
        for (int r = 0; r < K; r++) {
          sv[r] = __ldg(p.s + (int64_t)row * K + r);
          zi[r] = __ldcg(p.z + (int64_t)row * K + r);
        }
        if (W) d1 = __ldg(p.d1 + row);
      }
    }
    double a[K];
#pragma unroll
    for (int r = 0; r < K; r++) a[r] = 0.0;
    // arcs in flight per lane (K gathered values each)
    constexpr int TU = K >= 8 ? FJ_BT8 : (K >= 4 ? FJ_BT4 : 4);
#pragma unroll TU
    for (int64_t k = rb + gl; k < re; k += G) {
      const int j = ld_stream(p.col + k);
      const double wk = W ? (double)ld_stream(p.w + k) : 1.0;
      double v[K];
      gatherK<K>(p.z, j, v);
#pragma unroll
      for (int r = 0; r < K; r++) a[r] = fma(wk, v[r], a[r]);
    }
#pragma unroll
    for (int r = 0; r < K; r++)
      for (int off = G >> 1; off > 0; off >>= 1) a[r] += __shfl_xor_sync(0xffffffffu, a[r], off);
    if (has && gl == 0) {
      const int len = (int)(re - rb);
      dd tot[K];
#pragma unroll
      for (int r = 0; r < K; r++) tot[r] = dd{a[r], 0.0};
      relax_rowK<K>(p, bc, row, len, tot, sv, zi, W ? d1 : (double)(len + 1), t);
    }
  }
}

// Barrier-synchronised persistent sweeps for K right-hand sides: k_sweep's
// loop (static round-robin over each phase's list, next item prefetched, one
// grid barrier per color phase and per sweep, counters reduced on the device)
// around the K-wide units and tiles above.  The loop ends after a sweep in
// which no right-hand side relaxed any row (Q = ∅ for all of them).
// CTAs per SM: 4 at K = 2, 3 at K = 4, 2 at K = 8 (registers for the K-wide
// accumulators without spills).
template <bool W, int K>
__global__ void __launch_bounds__(kBlock, K >= 8 ? 2 : (K >= 4 ? FJ_BMIN4 : 4)) k_sweep_batch_bar(KP p) {
  __shared__ BCtx bc;
  __shared__ unsigned long long s_dec[3];
  __shared__ int s_nbad;
  if (threadIdx.x < K) {
    bc.sk[threadIdx.x] = p.sc[threadIdx.x];
    bc.om[threadIdx.x] = p.omegas ? p.omegas[threadIdx.x] : p.omega;
    bc.bad[threadIdx.x] = 0;
    bc.cupd[threadIdx.x] = 0u;
  }
  if (threadIdx.x == 0) bc.omb = p.colbad != nullptr;
  __syncthreads();
  const int stride = gridDim.x * (kBlock / 32);
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1;
  if (p.skip_if_done) {
    // second launch of a solve with the frontier phase: nothing to do if every column's
    // k_front (or the sweeps before it) ended converged — prev holds their out[] blocks
    bool all0 = true;
    for (int r = 0; r < p.kreal; r++) all0 = all0 && __ldcg(p.prev + 8 * r + 3) == 0ull;
    if (all0) {
      sweep_result(p.out, 0, 0ull, 0ull, 0);
      return;
    }
  }
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k) {
      const int r0 = p.rphase_begin[k], nr = p.rphase_begin[k + 1] - r0;
      int wi = warp_id;
      Task nxt;
      if (wi < nr) nxt = p.rtasks[r0 + wi];
      while (wi < nr) {
        const Task cur = nxt;
        const int wn = wi + stride;
        if (wn < nr) nxt = p.rtasks[r0 + wn];
        if ((cur.kind & 0xff) == kWarp) do_warpK<W, K>(p, &bc, cur, t);
        else tileK<W, K>(p, &bc, cur, t);
        wi = wn;
      }
      if (k + 1 < p.ncolors) grid_sync(p.bar);
    }
    if (bc.omb) {  // ω batch: this CTA's per-column relaxations of the sweep
      __syncthreads();
      if (threadIdx.x < K && bc.cupd[threadIdx.x]) {
        atomicAdd(p.colupd + threadIdx.x, (unsigned long long)bc.cupd[threadIdx.x]);
        bc.cupd[threadIdx.x] = 0u;
      }
    }
    unsigned long long dec[3];
    sweep_totals(p.cnt, p.bar, sw, t, s_dec, dec);
    tot_upd += dec[0];
    tot_eu += dec[1];
    sweeps = sw + 1;
    if (bc.omb) {  // columns that diverged anywhere are frozen from now on
      if (threadIdx.x == 0) s_nbad = 0;
      __syncthreads();
      if (threadIdx.x < K) {
        bc.bad[threadIdx.x] = __ldcg(p.colbad + threadIdx.x);
        if (bc.bad[threadIdx.x] && threadIdx.x < p.kreal) atomicAdd(&s_nbad, 1);
      }
      __syncthreads();
    }
    const bool bad = dec[2] != 0 || (bc.omb && s_nbad == p.kreal), done = dec[0] == 0;
    if (bad) { reason = 2; break; }
    if (done) { reason = 0; break; }
    if (dec[0] < p.thin) { reason = 3; break; }  // thin sweep: the frontier phase takes over
  }
  sweep_result(p.out, sweeps, tot_upd, tot_eu, reason);
}

template <bool W>
static const void *batch_kernel(int K) {
  return K == 2 ? (const void *)k_sweep_batch_bar<W, 2>
                : (K == 4 ? (const void *)k_sweep_batch_bar<W, 4> : (const void *)k_sweep_batch_bar<W, 8>);
}

// s (node order, k columns) → layout order, K padded columns (pad = last)
__global__ void k_init_batch(int64_t n, int k, int K, const int32_t *__restrict__ perm,
                             const int64_t *__restrict__ rp, const float *__restrict__ S,
                             Scalars *__restrict__ SK, float *__restrict__ sK,
                             double *__restrict__ zK) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t u = perm[i];
  const bool empty = rp[i + 1] == rp[i];
  for (int r = 0; r < K; r++) {
    const float si = S[u * k + (r < k ? r : k - 1)];
    if (!isfinite(si)) atomicOr(&SK[0].bad_input, 1);
    sK[i * K + r] = si;
    zK[i * K + r] = empty ? (double)si + SK[r].c : 0.0;  // d = 0 rows: exact
  }
}
// column r of S (node order) → contiguous fp32 (for the per-RHS min/max)
__global__ void k_column(int64_t n, int k, int r, const float *__restrict__ S, float *__restrict__ out) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n) out[u] = S[u * k + r];
}
// column r of the layout-order state → contiguous (for the per-RHS certificate)
__global__ void k_columnL(int64_t n, int K, int r, const float *__restrict__ sK,
                          const double *__restrict__ zK, float *__restrict__ s1,
                          double *__restrict__ z1) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  s1[i] = sK[i * K + r];
  z1[i] = zK[i * K + r];
}
// frontier phase: a column's ẑ' back into the K-wide state (the last real column also into
// the padding columns, which duplicate it)
__global__ void k_column_back(int64_t n, int K, int r0, int r1, const double *__restrict__ z1,
                              double *__restrict__ zK) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = z1[i];
  for (int r = r0; r < r1; r++) zK[i * K + r] = v;
}
__global__ void k_finalize_batch(int64_t n, int k, int K, const int32_t *__restrict__ iperm,
                                 const double *__restrict__ zK, const Scalars *__restrict__ SK,
                                 float *__restrict__ Z) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t i = iperm[u];
  for (int r = 0; r < k; r++) Z[u * k + r] = (float)(zK[i * K + r] - SK[r].c);
}

// k ≤ 8 right-hand sides per solve (padded to K = 2, 4, 8), ASYNC
// or COLORED schedule, one certificate per right-hand side
// replicate one opinion vector into k node-major columns (the ω batch)
__global__ void k_replicate(int64_t n, int k, const float *__restrict__ s, float *__restrict__ S) {
  const int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u < n)
    for (int r = 0; r < k; r++) S[u * k + r] = s[u];
}

// omegas == nullptr: k opinion vectors at one ω (fj_solve_batch).  Otherwise
// the ω batch (fj_solve_batch_omega): S_in is ONE vector, column r runs at
// omegas[r] (host), a column whose residual trips the sentinel is frozen and
// reported in status_out[r]; relax_out[r] = its relaxations.
fj_status batch_solve_impl(fj_graph *g, const float *S_in, int k, double eps, double omega,
                           const fj_opts *o, float *Z_out, fj_stats *st_out,
                           const double *omegas, int64_t *relax_out, int *status_out) {
  NvtxRange nv("fj_solve_batch");
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  const int K = k <= 2 ? 2 : (k <= 4 ? 4 : 8);
  // AUTO as fj_solve: multicolor SOR for ω ≠ 1 on undirected graphs
  bool all_one = omega == 1.0;
  if (omegas)
    for (int r = 0; r < k; r++) all_one = all_one && omegas[r] == 1.0;
  int method = o->method;
  if (method == FJ_METHOD_AUTO)
    method = (all_one || g->directed) ? FJ_METHOD_ASYNC : FJ_METHOD_COLORED;
  if (method == FJ_METHOD_COLORED) FJ_TRY(build_coloring(g, o));
  const Layout &L = method == FJ_METHOD_COLORED ? g->color_layout : g->async_layout;
  const bool W = g->weighted != 0;
  fj_stats stats{};
  stats.colors = L.ncolors;
  Workspace ws(st);
  cudaEvent_t e0, e1, es0, es1;
  for (cudaEvent_t *e : {&e0, &e1, &es0, &es1}) FJ_CUDA(ws.event(e));
  FJ_CUDA(cudaEventRecord(e0, st));
  const float *S = S_in;
  float *S_owned = nullptr;
  const int64_t s_len = omegas ? n : n * k;
  if (!is_device_ptr(S_in)) {
    FJ_CUDA(ws.alloc(&S_owned, s_len));
    FJ_CUDA(cudaMemcpyAsync(S_owned, S_in, sizeof(float) * s_len, cudaMemcpyHostToDevice, st));
    S = S_owned;
  }
  double *d_om = nullptr;
  int *colbad = nullptr;
  unsigned long long *colupd = nullptr;
  if (omegas) {  // one vector → k columns; per-column ω, flags and counts
    float *Srep = nullptr;
    FJ_CUDA(ws.alloc(&Srep, n * k));
    fj::count_launch();
    k_replicate<<<gridn(n), kBlock, 0, st>>>(n, k, S, Srep);
    S = Srep;
    double hom[8];
    for (int r = 0; r < K; r++) hom[r] = omegas[r < k ? r : k - 1];
    FJ_CUDA(ws.alloc(&d_om, 8));
    FJ_CUDA(cudaMemcpyAsync(d_om, hom, sizeof(double) * 8, cudaMemcpyHostToDevice, st));
    FJ_CUDA(ws.alloc(&colbad, 8));
    FJ_CUDA(cudaMemsetAsync(colbad, 0, sizeof(int) * 8, st));
    FJ_CUDA(ws.alloc(&colupd, 8));
    FJ_CUDA(cudaMemsetAsync(colupd, 0, sizeof(unsigned long long) * 8, st));
    FJ_CUDA(cudaStreamSynchronize(st));  // hom is stack-owned
  }
  const bool zdev = is_device_ptr(Z_out);
  float *sK = nullptr, *col = nullptr, *mm = nullptr, *s1 = nullptr, *Zd = nullptr;
  double *zK = nullptr, *z1 = nullptr;
  double2 *partial = nullptr;
  int *arrive = nullptr, *arrive2 = nullptr;
  Scalars *SK = nullptr;
  unsigned long long *outv = nullptr;
  unsigned *ctl = nullptr, *ctlb = nullptr;
  SweepCounters *cnt = nullptr;
  const size_t np = (size_t)std::max(1, L.npartials);
  FJ_CUDA(ws.alloc(&sK, n * K));
  FJ_CUDA(ws.alloc(&zK, n * K));
  FJ_CUDA(ws.alloc(&col, n));
  FJ_CUDA(ws.alloc(&mm, 2));
  FJ_CUDA(ws.alloc(&s1, n));
  FJ_CUDA(ws.alloc(&z1, n));
  FJ_CUDA(ws.alloc(&partial, np * K));
  FJ_CUDA(ws.alloc(&arrive, np));
  FJ_CUDA(ws.alloc(&arrive2, np));
  FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * np, st));
  FJ_CUDA(ws.alloc(&SK, K));
  FJ_CUDA(ws.alloc(&outv, 8 + 16 + 8 * 8));  // sweeps, certificate, second launch, k_front per column
  FJ_CUDA(ws.alloc(&ctl, 8));
  FJ_CUDA(ws.alloc(&ctlb, kCtlWords));
  FJ_CUDA(ws.alloc(&cnt, 3));
  if (!zdev) FJ_CUDA(ws.alloc(&Zd, n * k));
  // a2 per right-hand side: shift and thresholds (Alg. 2, reading R5)
  for (int r = 0; r < K; r++) {
    fj::count_launch();
    k_column<<<gridn(n), kBlock, 0, st>>>(n, k, r < k ? r : k - 1, S, col);
    FJ_TRY(minmax_f32(col, n, mm, ws, g->num_sms));
    fj::count_launch();
    k_scalars<<<1, 1, 0, st>>>(mm, mm + 1, eps, o->sigma, o->c, SK + r);
  }
  fj::count_launch();
  k_init_batch<<<gridn(n), kBlock, 0, st>>>(n, k, K, L.perm, L.rp, S, SK, sK, zK);
  KP p = make_kp(g, L);
  p.s = sK;
  p.z = zK;
  p.sc = SK;
  p.omega = omega;
  p.theta = 1.0;
  p.partial = partial;
  p.arrive = arrive;
  p.max_sweeps = o->max_sweeps;
  p.kreal = k;
  p.omegas = d_om;
  p.colbad = colbad;
  p.colupd = colupd;
  // barrier-synchronised persistent sweeps (an epoch-claim barrier-free
  // variant measured slower: C4 k = 4 1065 vs 1010 ms, C5 124 vs 99 ms)
  const void *fb = W ? batch_kernel<true>(K) : batch_kernel<false>(K);
  const int bgrid = persistent_grid(fb, g->num_sms);
  const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
  const int cgrid = persistent_grid(cf, g->num_sms);
  float ms_sweep = 0;
  int rounds = 0;
  p.ctr = ctlb;
  p.bar = ctlb + 8;
  p.cnt = cnt;
  p.out = outv;
  // Frontier phase (fj_opts.frontier, solve.cu k_front): once a batched sweep relaxes fewer
  // than T·k rows over all right-hand sides, every column finishes on its own in the push
  // form (column extracted to contiguous s1 / z1, compensated residuals, pop / scatter
  // rounds, column written back); a second launch of the batched sweeps follows and
  // returns at once when every column converged.  Not for the ω batch (its per-column
  // relaxation counts and divergence flags belong to the sweeps).
  const bool use_front = o->frontier != 0 && !omegas && L.active_rows > 0;
  const void *ffn = front_kernel(W);
  unsigned long long *outB = outv + 16, *outF = outv + 24, *scratch_max = outv + 5;
  KP pf = make_kp(g, L);
  int fgrid = 0;
  unsigned long long thin = 0;
  if (use_front) {
    const int64_t act = std::max<int64_t>(1, L.active_rows);
    const int64_t T = o->frontier > 0 ? (int64_t)o->frontier : std::max<int64_t>(32, act / FJ_THIN_DIV);
    thin = (unsigned long long)(T * k);
    pf.fr_cap = (int)std::min<int64_t>(std::max<int64_t>(4096, act / 4), 1 << 30);
    pf.fr_pcap = (int)std::min<int64_t>((int64_t)pf.fr_cap + L.m / kDepChunk, 1 << 30);
    FJ_CUDA(ws.alloc(&pf.fr_r, (size_t)n));
    FJ_CUDA(ws.alloc(&pf.fr_rows, 2 * (size_t)pf.fr_cap));
    FJ_CUDA(ws.alloc(&pf.fr_push, (size_t)pf.fr_pcap));
    FJ_CUDA(ws.alloc(&pf.fr_cnt, 4));
    pf.in_rp = g->in_rp;
    pf.in_col = g->in_col;
    pf.in_w = g->in_w;
    pf.perm = L.perm;
    pf.iperm = L.iperm;
    pf.fr_max_rounds = 100000;
    pf.s = s1;
    pf.z = z1;
    pf.partial = partial;
    pf.arrive = arrive2;
    pf.ctr = ctl;
    pf.bar = ctlb + 8;
    pf.cnt = cnt;
    pf.cert_max = scratch_max;
    pf.omega = L.ncolors > 1 ? 1.0 : omega;  // after colored sweeps: plain pops (solve.cu)
    FJ_CUDA(cudaFuncSetAttribute(ffn, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    fgrid = persistent_grid(ffn, g->num_sms, 0);
  }
  auto rest = [&]() -> fj_status {
    FJ_CUDA(cudaMemsetAsync(ctlb, 0, sizeof(unsigned) * kCtlWords, st));
    FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(SweepCounters) * 3, st));
    return FJ_OK;
  };
  for (;;) {
    FJ_CUDA(cudaMemsetAsync(outv, 0, sizeof(unsigned long long) * (8 + 16 + 8 * 8), st));
    FJ_TRY(rest());
    FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * np, st));
    FJ_CUDA(cudaEventRecord(es0, st));
    p.thin = thin;
    p.skip_if_done = 0;
    p.prev = nullptr;
    p.out = outv;
    {
      void *args[] = {&p};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fb, bgrid, kBlock, args, 0, st));
    }
    if (use_front) {
      pf.theta = p.theta;
      for (int r = 0; r < k; r++) {
        fj::count_launch();
        k_columnL<<<gridn(n), kBlock, 0, st>>>(n, K, r, sK, zK, s1, z1);
        KP q = pf;
        q.sc = SK + r;
        q.prev = outv;
        q.out = outF + 8 * r;
        FJ_TRY(rest());
        FJ_CUDA(cudaMemsetAsync(arrive2, 0, sizeof(int) * np, st));
        FJ_CUDA(cudaMemsetAsync(pf.fr_cnt, 0, sizeof(unsigned) * 4, st));
        {  // residuals of the column (runs only after a thin exit)
          KP qr = q;
          qr.rout = pf.fr_r;
          void *rargs[] = {&qr};
          fj::count_launch();
          FJ_CUDA(cudaLaunchKernel(cf, cgrid, kBlock, rargs, 0, st));
        }
        FJ_TRY(rest());
        void *fargs[] = {&q};
        fj::count_launch();
        FJ_CUDA(cudaLaunchCooperativeKernel(ffn, fgrid, kBlock, fargs, 0, st));
        fj::count_launch();
        k_column_back<<<gridn(n), kBlock, 0, st>>>(n, K, r, r + 1 == k ? K : r + 1, z1, zK);
      }
      // the batched sweeps again: at once done if every column converged, else they carry on
      FJ_TRY(rest());
      FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * np, st));
      KP q = p;
      q.thin = 0;
      q.skip_if_done = 1;
      q.prev = outF;
      q.out = outB;
      void *args[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fb, bgrid, kBlock, args, 0, st));
    }
    FJ_CUDA(cudaEventRecord(es1, st));
    unsigned long long h[8], hx[8 + 64];
    FJ_CUDA(cudaMemcpyAsync(h, outv, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaMemcpyAsync(hx, outB, sizeof(hx), cudaMemcpyDeviceToHost, st));
    // compensated certificate of every right-hand side (ω batch: of every
    // column that did not diverge)
    double worst = 0.0;
    int hbad[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (colbad) {
      FJ_CUDA(cudaMemcpyAsync(hbad, colbad, sizeof(int) * 8, cudaMemcpyDeviceToHost, st));
      FJ_CUDA(cudaStreamSynchronize(st));
    }
    for (int r = 0; r < k; r++) {
      if (hbad[r]) {
        if (status_out) status_out[r] = FJ_ERR_NUMERIC;
        continue;
      }
      fj::count_launch();
      k_columnL<<<gridn(n), kBlock, 0, st>>>(n, K, r, sK, zK, s1, z1);
      KP q = make_kp(g, L);
      q.s = s1;
      q.z = z1;
      q.sc = SK + r;
      q.partial = partial;
      q.arrive = arrive2;
      q.ctr = ctl;
      q.cert_max = outv + 4;
      FJ_CUDA(cudaMemsetAsync(arrive2, 0, sizeof(int) * np, st));
      FJ_CUDA(cudaMemsetAsync(outv + 4, 0, sizeof(unsigned long long), st));
      void *cargs[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchKernel(cf, cgrid, kBlock, cargs, 0, st));
      unsigned long long bits = 0;
      FJ_CUDA(cudaMemcpyAsync(&bits, outv + 4, sizeof(bits), cudaMemcpyDeviceToHost, st));
      FJ_CUDA(cudaStreamSynchronize(st));
      const double ratio = __builtin_bit_cast(double, bits);
      if (!(ratio <= worst)) worst = ratio;
      if (status_out) status_out[r] = ratio <= 1.0 ? FJ_OK : FJ_ERR_NUMERIC;
    }
    FJ_CUDA(cudaStreamSynchronize(st));
    float a = 0;
    FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
    ms_sweep += a;
    stats.sweeps += (int64_t)h[0];
    stats.relaxations += (int64_t)h[1];
    stats.edge_updates += (int64_t)h[2];
    stats.reason = (int)h[3];
    if (use_front) {
      // every column's k_front continued the first launch's totals: its own part on top,
      // then the second launch of the sweeps (whose reason is the round's)
      for (int r = 0; r < k; r++) {
        const unsigned long long *f = hx + 8 + 8 * r;
        stats.relaxations += (int64_t)(f[1] - h[1]);
        stats.edge_updates += (int64_t)(f[2] - h[2]);
        stats.frontier_rounds += (int64_t)f[4];
        stats.frontier_pushes += (int64_t)f[5];
      }
      stats.sweeps += (int64_t)hx[0];
      stats.relaxations += (int64_t)hx[1];
      stats.edge_updates += (int64_t)hx[2];
      stats.reason = (int)hx[3];
    }
    stats.cert_ratio = worst;
    if (stats.reason != 0 || stats.cert_ratio <= 1.0 || rounds >= o->cert_rounds) break;
    rounds++;
    p.theta *= 0.5;
    p.max_sweeps = std::min(o->max_sweeps, 2000);
  }
  stats.cert_rounds = rounds;
  stats.phases = stats.sweeps * L.ncolors;
  stats.rows_read = stats.sweeps * L.active_rows;
  stats.arcs_read = stats.sweeps * L.m;
  stats.relaxations += L.empty_rows * k;
  if (relax_out) {  // ω batch: relaxations per column (rows solved at init included)
    unsigned long long hu[8];
    FJ_CUDA(cudaMemcpyAsync(hu, colupd, sizeof(hu), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    for (int r = 0; r < k; r++) relax_out[r] = (int64_t)hu[r] + L.empty_rows;
  }
  fj::count_launch();
  k_finalize_batch<<<gridn(n), kBlock, 0, st>>>(n, k, K, L.iperm, zK, SK, zdev ? Z_out : Zd);
  if (!zdev) FJ_CUDA(cudaMemcpyAsync(Z_out, Zd, sizeof(float) * n * k, cudaMemcpyDeviceToHost, st));
  Scalars hs{};
  FJ_CUDA(cudaMemcpyAsync(&hs, SK, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaEventRecord(e1, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  float ms = 0;
  FJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  stats.solve_ms = ms;
  stats.sweep_ms = ms_sweep;
  stats.c = hs.c;
  stats.eps_prime = hs.eps_p;
  FJ_CUDA(cudaGetLastError());
  fj_status rc = finish_status(hs, stats, o, omega);
  if (st_out) *st_out = stats;
  return rc;
}

}  // namespace fj

extern "C" {

fj_status fj_solve_batch(fj_graph_t g, const float *S, int k, double eps, double omega,
                         const fj_opts *o, float *Z_out, fj_stats *st) {
  fj_opts d;
  fj_opts_default(&d);
  if (o) {
    d = *o;
    if (!(d.sigma > 0)) d.sigma = 1e-5;
    if (d.max_sweeps <= 0) d.max_sweeps = 1000000;
    if (d.cert_rounds < 0) d.cert_rounds = 3;
  }
  if (!g || !S || !Z_out || k < 1 || k > 8) {
    fj::set_error("fj_solve_batch: need non-null arguments and 1 <= k <= 8");
    return FJ_ERR_INVALID;
  }
  if (!(eps > 0.0 && eps < 1.0) || !(omega > 0.0 && omega < 2.0)) {
    fj::set_error("fj_solve_batch: eps in (0,1) and omega in (0,2) required");
    return FJ_ERR_INVALID;
  }
  if (d.method != FJ_METHOD_AUTO && d.method != FJ_METHOD_ASYNC && d.method != FJ_METHOD_COLORED) {
    fj::set_error("fj_solve_batch: the ASYNC and COLORED schedules are batched, not PUSH");
    return FJ_ERR_INVALID;
  }
  if (d.z_init) {
    fj::set_error("fj_solve_batch: z_init (warm start) is not supported for batches");
    return FJ_ERR_INVALID;
  }
  return fj::batch_solve_impl(g, S, k, eps, omega, &d, Z_out, st, nullptr, nullptr, nullptr);
}

fj_status fj_solve_batch_omega(fj_graph_t g, const float *s, int k, const double *omegas,
                               double eps, const fj_opts *o, float *Z_out, fj_stats *st,
                               int64_t *relax_out, int *status_out) {
  fj_opts d;
  fj_opts_default(&d);
  if (o) {
    d = *o;
    if (!(d.sigma > 0)) d.sigma = 1e-5;
    if (d.max_sweeps <= 0) d.max_sweeps = 1000000;
    if (d.cert_rounds < 0) d.cert_rounds = 3;
  }
  if (!g || !s || !Z_out || !omegas || k < 1 || k > 8) {
    fj::set_error("fj_solve_batch_omega: need non-null arguments and 1 <= k <= 8");
    return FJ_ERR_INVALID;
  }
  for (int r = 0; r < k; r++)
    if (!(omegas[r] > 0.0 && omegas[r] < 2.0)) {
      fj::set_error("fj_solve_batch_omega: omega[%d] = %g outside (0, 2)", r, omegas[r]);
      return FJ_ERR_INVALID;
    }
  if (!(eps > 0.0 && eps < 1.0)) {
    fj::set_error("fj_solve_batch_omega: eps in (0,1) required");
    return FJ_ERR_INVALID;
  }
  if (d.method != FJ_METHOD_AUTO && d.method != FJ_METHOD_ASYNC && d.method != FJ_METHOD_COLORED) {
    fj::set_error("fj_solve_batch_omega: the ASYNC and COLORED schedules are batched, not PUSH");
    return FJ_ERR_INVALID;
  }
  if (d.z_init) {
    fj::set_error("fj_solve_batch_omega: z_init (warm start) is not supported for batches");
    return FJ_ERR_INVALID;
  }
  int stat[8];
  fj_status rc = fj::batch_solve_impl(g, s, k, eps, omegas[0], &d, Z_out, st, omegas, relax_out,
                                      stat);
  if (status_out)
    for (int r = 0; r < k; r++) status_out[r] = stat[r];
  if (rc == FJ_ERR_NUMERIC) {  // per-column outcomes are in status_out
    bool any_ok = false;
    for (int r = 0; r < k; r++) any_ok = any_ok || stat[r] == FJ_OK;
    if (any_ok) rc = FJ_OK;
  }
  return rc;
}


}  // extern "C"
