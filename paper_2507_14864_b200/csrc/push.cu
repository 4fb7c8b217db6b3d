// push.cu — FJ_METHOD_PUSH (§8 row a3 in its literal form): Alg. 1/3 made data
// parallel — a pop phase and an fp64-atomic scatter phase per color — with the
// certificate on the pull layout and residual replacement on resume.
#include "sweep_common.cuh"

namespace fj {

// ------------------------------------------------------------ frontier push
// FJ_METHOD_PUSH: Alg. 1 / Alg. 3 in data-parallel form on the push layout
// (rows = in-rows: row v lists the u with an arc u→v, i.e. v's scatter list).
// Per color phase:
//   A (pop):  every v of the color with |r_v| > θ h_v takes q_v = ω r_v/(1+d_v),
//             ẑ_v += q_v (equ:sor1), r_v ← (1−ω) r_v (equ:sor2); else q_v = 0;
//   B (push): every popped v adds a_uv q_v to r_u for u ∈ N_v (equ:sor3)
//             with fp64 atomics.
// Rows of one color share no arc, so a phase equals popping its frontier one
// node after another (Lemma 3 holds for any order).
struct PP {
  const int64_t *__restrict__ rp;
  const int32_t *__restrict__ col;
  const float *__restrict__ w;
  const double *__restrict__ d1;
  const Task *__restrict__ tasks;
  const Task *__restrict__ wtasks;
  const int *phase_begin, *wphase_begin;
  const int64_t *crow;
  int ncolors;
  int tail_phase;  // colored: merged tail colors relaxed with ω = 1 (reading R23)
  int64_t n;
  const float *__restrict__ s;
  double *z, *r, *q;
  const Scalars *sc;
  double omega, theta;
  int max_sweeps;
  unsigned *bar;
  SweepCounters *cnt;
  unsigned long long *out;
  int32_t *front;                 // compacted frontier of the current phase
  unsigned long long *fcount;     // [3] frontier sizes (ring over phases)
  int sparse_div;                 // sparse scatter when |frontier|·div < rows of the phase
};

// pop one row: q_v = ω r_v/(1+d_v) if |r_v| > h_v; returns whether v has a
// scatter list to walk
__device__ __forceinline__ bool pop_row(const PP &p, const Scalars &S, int64_t v, TAcc &t,
                                        double om) {
  const double sp = (double)p.s[v] + S.c;
  const double h = threshold(S, sp);
  const double rv = p.r[v];
  double qv = 0.0;
  bool act = false;
  if (fabs(rv) > p.theta * h) {                       // |r_v| > h_v
    qv = om * rv / p.d1[v];                           // ω r_v/(1+d_v)
    p.z[v] += qv;                                     // equ:sor1
    p.r[v] = rv - om * rv;                            // equ:sor2: (1−ω) r_v
    t.upd++;
    t.eu += (unsigned long long)(p.rp[v + 1] - p.rp[v]);
    act = p.rp[v + 1] > p.rp[v];
  }
  if (!(fabs(rv) <= S.sentinel)) t.bad = 1;
  p.q[v] = qv;
  return act;
}

// pop phase over rows [b, e): dense (q_v marks the frontier)
__device__ __forceinline__ void push_pop(const PP &p, const Scalars &S, int64_t b, int64_t e,
                                         TAcc &t, double om) {
  for (int64_t v = b + blockIdx.x * (int64_t)kBlock + threadIdx.x; v < e;
       v += (int64_t)gridDim.x * kBlock)
    pop_row(p, S, v, t, om);
}

// pop phase with frontier compaction: ballot per warp, one atomic per warp
// with active rows, popcount prefix for the slots
__device__ __forceinline__ void push_pop_compact(const PP &p, const Scalars &S, int64_t b,
                                                 int64_t e, TAcc &t, double om,
                                                 unsigned long long *fcount) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = b + blockIdx.x * (int64_t)kBlock + (threadIdx.x & ~31); base < e;
       base += (int64_t)gridDim.x * kBlock) {
    const int64_t v = base + lane;
    const bool act = v < e && pop_row(p, S, v, t, om);
    const unsigned m = __ballot_sync(0xffffffffu, act);
    if (m) {
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(fcount, (unsigned long long)__popc(m));
      off = __shfl_sync(0xffffffffu, off, 0);
      if (act) p.front[off + __popc(m & ((1u << lane) - 1u))] = (int32_t)v;
    }
  }
}

template <bool W>
__device__ __forceinline__ void push_scatter_arcs(const PP &p, int64_t k0, int64_t k1, int step,
                                                  double qv) {
  for (int64_t k = k0; k < k1; k += step) {
    const int u = ld_stream(p.col + k);
    const double a = W ? (double)ld_stream(p.w + k) : 1.0;
    atomicAdd(p.r + u, a * qv);                          // equ:sor3
  }
}

// scatter of a compacted frontier: warp per active row
template <bool W>
__device__ __forceinline__ void scatter_sparse(const PP &p, long long F) {
  const int lane = threadIdx.x & 31;
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  for (long long fi = warp_id; fi < F; fi += (long long)gridDim.x * (kBlock / 32)) {
    const int v = p.front[fi];
    push_scatter_arcs<W>(p, p.rp[v] + lane, p.rp[v + 1], 32, p.q[v]);
  }
}

// CF: frontier compaction (FJ_PUSH_COMPACT=1).  Measured slower than the
// dense frontier (q_v ≠ 0 marks) on C2/C4/C5 (DESIGN.md §8 tuning log), so
// the default instantiation keeps the dense loop only.
template <bool W, bool CF>
__global__ void __launch_bounds__(kBlock, 4) k_push(PP p) {
  __shared__ unsigned long long s_dec[3];
  const Scalars S = *p.sc;
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1, phase = 0;
  unsigned long long last_upd = (unsigned long long)p.n;  // relaxations of the last sweep
  const int lane = threadIdx.x & 31;
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k, ++phase) {
      const double om = k == p.tail_phase ? 1.0 : p.omega;
      unsigned long long *fc = p.fcount + phase % 3;
      if (CF && blockIdx.x == 0 && threadIdx.x == 0) p.fcount[(phase + 1) % 3] = 0ull;  // next
      // compact only when the last sweep relaxed few rows: early sweeps relax
      // most rows, and there the dense task walk needs no atomics at all
      const long long rows = (long long)(p.crow[k + 1] - p.crow[k]);
      const bool compact = CF && (long long)last_upd * p.sparse_div < (long long)p.n;
      if (CF && compact) {
        push_pop_compact(p, S, p.crow[k], p.crow[k + 1], t, om, fc);
        if (k == p.ncolors - 1) push_pop_compact(p, S, p.crow[p.ncolors], p.n, t, om, fc);
      } else {
        push_pop(p, S, p.crow[k], p.crow[k + 1], t, om);
        if (k == p.ncolors - 1) push_pop(p, S, p.crow[p.ncolors], p.n, t, om);  // no in-arcs
      }
      grid_sync(p.bar);
      // B: scatter.  A small frontier is walked as the compacted list (warp
      // per active row); a large one by the layout's tasks (q = 0 rows skip)
      const long long F = compact ? (long long)__ldcg(fc) : rows;
      if (CF && compact && F * p.sparse_div < rows) {
        scatter_sparse<W>(p, F);
        grid_sync(p.bar);
        continue;
      }
      // dense: warp units (long scatter lists), then tile tasks (group per row)
      const int w0 = p.wphase_begin[k], nw = p.wphase_begin[k + 1] - w0;
      for (int wi = warp_id; wi < nw; wi += gridDim.x * (kBlock / 32)) {
        const Task tk = p.wtasks[w0 + wi];
        const double qv = p.q[tk.a];
        if (qv != 0.0) push_scatter_arcs<W>(p, tk.a0 + lane, tk.a1, 32, qv);
      }
      const int t0 = p.phase_begin[k], nt = p.phase_begin[k + 1] - t0;
      for (int ti = blockIdx.x; ti < nt; ti += gridDim.x) {
        const Task tk = p.tasks[t0 + ti];
        const int cls = tk.kind & 0xff;
        const int G = 1 << cls;
        const int row = tk.a + (threadIdx.x >> cls);
        if (row < tk.b) {
          const double qv = p.q[row];
          if (qv != 0.0)
            push_scatter_arcs<W>(p, p.rp[row] + (threadIdx.x & (G - 1)), p.rp[row + 1], G, qv);
        }
      }
      grid_sync(p.bar);
    }
    unsigned long long dec[3];
    sweep_totals(p.cnt, p.bar, sw, t, s_dec, dec);
    tot_upd += dec[0];
    tot_eu += dec[1];
    last_upd = dec[0];
    sweeps = sw + 1;
    const bool bad = dec[2] != 0, done = dec[0] == 0;
    if (bad) { reason = 2; break; }
    if (done) { reason = 0; break; }
  }
  sweep_result(p.out, sweeps, tot_upd, tot_eu, reason);
}

// push-layout init: s in push order, ẑ' = 0, r = s' (Alg. 1 init)
__global__ void k_push_init(int64_t n, const int32_t *__restrict__ perm, const float *__restrict__ s,
                            Scalars *__restrict__ S, float *__restrict__ s_l, double *__restrict__ z,
                            double *__restrict__ r) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float si = s[perm[i]];
  if (!isfinite(si)) atomicOr(&S->bad_input, 1);
  s_l[i] = si;
  z[i] = 0.0;
  r[i] = (double)si + S->c;
}

// dst[i] = src[idx[i]]
__global__ void k_gather64(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ src,
                           double *__restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
// dst[idx[i]] = src[i]
__global__ void k_scatter64(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ src,
                            double *__restrict__ dst) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[idx[i]] = src[i];
}

// FJ_METHOD_PUSH: frontier push on the in-row layout; certificate on the pull
// layout (the residual needs out-rows); residual replacement on resume.
fj_status push_solve_impl(fj_graph *g, const float *s_in, double eps, double omega,
                                 const fj_opts *o, float *z_out, fj_stats *st_out) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  const bool colored = omega != 1.0;
  if (colored) FJ_TRY(build_coloring(g, o));
  Layout &P = colored ? g->push_color_layout : g->push_layout;
  if (!P.tasks) {
    FJ_TRY(build_layout_from_out(g, g->in_rp, g->in_col, g->in_w, colored ? g->colors : nullptr,
                                 colored ? g->ncolors : 1, &P, true));
    P.tail_phase = colored ? g->tail_color : -1;
  }
  const Layout &L = g->async_layout;
  const bool W = g->weighted != 0;
  fj_stats stats{};
  stats.colors = P.ncolors;

  Workspace ws(st);
  cudaEvent_t e0, e1, es0, es1;
  for (cudaEvent_t *e : {&e0, &e1, &es0, &es1}) FJ_CUDA(ws.event(e));
  FJ_CUDA(cudaEventRecord(e0, st));
  Staged s{};
  FJ_TRY(stage_in(s_in, n, ws, s));
  const bool zdev = is_device_ptr(z_out);
  const bool zpdev = o->zprime_out && is_device_ptr(o->zprime_out);
  float *sP = nullptr, *sL = nullptr, *smin = nullptr, *zo = nullptr;
  double *zP = nullptr, *rP = nullptr, *qP = nullptr, *zL = nullptr, *tmp = nullptr, *zp = nullptr;
  double *RL = nullptr;
  Scalars *S = nullptr;
  unsigned *ctl = nullptr;
  SweepCounters *cnt = nullptr;
  unsigned long long *outv = nullptr;
  FJ_CUDA(ws.alloc(&sP, n));
  FJ_CUDA(ws.alloc(&sL, n));
  FJ_CUDA(ws.alloc(&zP, n));
  FJ_CUDA(ws.alloc(&rP, n));
  FJ_CUDA(ws.alloc(&qP, n));
  FJ_CUDA(ws.alloc(&zL, n));
  FJ_CUDA(ws.alloc(&tmp, n));
  FJ_CUDA(ws.alloc(&RL, n));
  FJ_CUDA(ws.alloc(&smin, 2));
  FJ_CUDA(ws.alloc(&S, 1));
  FJ_CUDA(ws.alloc(&ctl, kCtlWords));
  FJ_CUDA(ws.alloc(&cnt, 3));
  FJ_CUDA(ws.alloc(&outv, 8));
  if (!zdev) FJ_CUDA(ws.alloc(&zo, n));
  if (o->zprime_out && !zpdev) FJ_CUDA(ws.alloc(&zp, n));
  FJ_TRY(minmax_f32(s.dev, n, smin, ws, g->num_sms));
  fj::count_launch();
  k_scalars<<<1, 1, 0, st>>>(smin, smin + 1, eps, o->sigma, o->c, S);
  fj::count_launch();
  k_push_init<<<gridn(n), kBlock, 0, st>>>(n, P.perm, s.dev, S, sP, zP, rP);
  fj::count_launch();
  k_init<<<gridn(n), kBlock, 0, st>>>(n, L.perm, L.rp, s.dev, S, sL, zL);

  PP pp{};
  pp.rp = P.rp;
  pp.col = P.col;
  pp.w = P.w;
  pp.d1 = P.d1;
  pp.tasks = P.tasks;
  pp.wtasks = P.wtasks;
  pp.phase_begin = P.d_phase_begin;
  pp.wphase_begin = P.d_wphase_begin;
  pp.crow = P.d_crow;
  pp.ncolors = P.ncolors;
  pp.tail_phase = P.tail_phase;
  pp.n = n;
  pp.s = sP;
  pp.z = zP;
  pp.r = rP;
  pp.q = qP;
  pp.sc = S;
  pp.omega = omega;
  pp.theta = 1.0;
  pp.max_sweeps = o->max_sweeps;
  pp.bar = ctl + 8;
  pp.cnt = cnt;
  pp.out = outv;
  int32_t *front = nullptr;
  FJ_CUDA(ws.alloc(&front, n));
  pp.front = front;
  pp.fcount = reinterpret_cast<unsigned long long *>(ctl + 16);  // zeroed with ctl
  pp.sparse_div = o->push_sparse_div > 0 ? o->push_sparse_div : 8;
  KP kq = make_kp(g, L);
  kq.s = sL;
  kq.z = zL;
  kq.sc = S;
  kq.ctr = ctl + 5;
  kq.cert_max = outv + 4;
  kq.rout = RL;
  double2 *partial = nullptr;  // long-row partials of the pull layout (certificate)
  int *arrive = nullptr;
  FJ_CUDA(ws.alloc(&partial, std::max(1, L.npartials)));
  FJ_CUDA(ws.alloc(&arrive, std::max(1, L.npartials)));
  FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
  kq.partial = partial;
  kq.arrive = arrive;

  const bool compact = o->push_compact != 0;
  const void *fn = W ? (compact ? (const void *)k_push<true, true> : (const void *)k_push<true, false>)
                     : (compact ? (const void *)k_push<false, true> : (const void *)k_push<false, false>);
  const int grid = persistent_grid(fn, g->num_sms);
  const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
  float ms_sweep = 0;
  int rounds = 0;
  for (;;) {
    FJ_CUDA(cudaMemsetAsync(ctl, 0, sizeof(unsigned) * kCtlWords, st));
    FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(SweepCounters) * 3, st));
    FJ_CUDA(cudaMemsetAsync(outv, 0, sizeof(unsigned long long) * 8, st));
    void *args[] = {&pp};
    FJ_CUDA(cudaEventRecord(es0, st));
    fj::count_launch();
    FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, 0, st));
    FJ_CUDA(cudaEventRecord(es1, st));
    // certificate on the pull layout: ẑ' push order → node order → pull order
    fj::count_launch();
    k_scatter64<<<gridn(n), kBlock, 0, st>>>(n, P.perm, zP, tmp);
    fj::count_launch();
    k_gather64<<<gridn(n), kBlock, 0, st>>>(n, L.perm, tmp, zL);
    void *cargs[] = {&kq};
    fj::count_launch();
    FJ_CUDA(cudaLaunchKernel(cf, persistent_grid(cf, g->num_sms), kBlock, cargs, 0, st));
    unsigned long long h[8];
    FJ_CUDA(cudaMemcpyAsync(h, outv, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    float a = 0;
    FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
    ms_sweep += a;
    stats.sweeps += (int64_t)h[0];
    stats.relaxations += (int64_t)h[1];
    stats.edge_updates += (int64_t)h[2];
    stats.reason = (int)h[3];
    stats.cert_ratio = __builtin_bit_cast(double, h[4]);
    if (stats.reason != 0) break;
    if (stats.cert_ratio <= 1.0 || rounds >= o->cert_rounds) break;
    rounds++;
    // residual replacement (Lemma 3: r = s' − (I+L)ẑ'), pull order → push order
    fj::count_launch();
    k_scatter64<<<gridn(n), kBlock, 0, st>>>(n, L.perm, RL, tmp);
    fj::count_launch();
    k_gather64<<<gridn(n), kBlock, 0, st>>>(n, P.perm, tmp, rP);
    pp.theta *= 0.5;
    pp.max_sweeps = std::min(o->max_sweeps, 2000);
  }
  stats.cert_rounds = rounds;
  stats.phases = stats.sweeps * P.ncolors * 2;
  stats.rows_read = stats.sweeps * n;
  stats.arcs_read = stats.edge_updates;
  fj::count_launch();
  k_finalize<<<gridn(n), kBlock, 0, st>>>(n, P.iperm, zP, S, zdev ? z_out : zo,
                                          o->zprime_out ? (zpdev ? o->zprime_out : zp) : nullptr);
  if (!zdev) FJ_CUDA(cudaMemcpyAsync(z_out, zo, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
  if (o->zprime_out && !zpdev)
    FJ_CUDA(cudaMemcpyAsync(o->zprime_out, zp, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  Scalars hs{};
  FJ_CUDA(cudaMemcpyAsync(&hs, S, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
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
