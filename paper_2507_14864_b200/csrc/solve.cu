// solve.cu — the hot path (§8 rows a2–a7): shift/init, persistent sweep
// kernel with on-device loop control, fp64 residual certificate, unshift,
// and the measures.
//
// Method.  The paper's push loop (Alg. 1/3, P:204–228,
// P:436–463) relaxes one queued node at a time; Theorem 3 shows
// each relaxation is a Gauss–Seidel update of row v of (I+L)ẑ = s with the
// residual r_v = s_v − ((I+L)ẑ)_v, and Lemma 3 shows the estimate is
// correct for any order and amount of relaxation.  A sweep here evaluates the
// residual of every non-empty row from the current ẑ (a pull over the row's
// arcs, fp64 accumulation) and relaxes exactly the rows the paper would have
// queued, |r_v| > h_v (P:221/453/458):
//        ẑ_v ← ẑ_v + ω r_v / (1 + d_v)                      (equ:sor1)
// ASYNC: one phase per sweep, rows updated in place (later rows see earlier
// updates, as in Gauss–Seidel).  COLORED: one phase per color; rows of one
// color share no arc, so each phase equals sequential SOR over that color.
// The loop ends on the first sweep that relaxes nothing: every residual was
// then evaluated on the final ẑ and is ≤ h — the paper's "Q = ∅".
// A separate compensated fp64 pass (certificate) re-checks max |r_v|/h_v.
#include <stdlib.h>

#include <cuda/atomic>
#include <type_traits>
#include <cub/cub.cuh>

#include <nvtx3/nvToolsExt.h>

#include "fj_internal.cuh"

namespace fj {

struct NvtxRange {  // tracing: one NVTX range per library phase (nsys/ncu timelines)
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

enum Mode { RELAX = 0, CERT = 1, DIS = 2, SPMV = 3 };
constexpr int kClaim = 16;  // work items per dynamic claim
constexpr int kCtlWords = 256;  // control block: [0..2] claim counters, [5] cert counter, [8..] barrier

struct Scalars {
  double c;        // shift (Alg. 2; reading R5)
  double eps_p;    // ε' = σε/(c+σ)
  double hs;       // h = hs·s'            (s_min ≥ 0)
  double heps;     // h = heps·max(hs·s', σ) (s_min < 0, floored, R5)
  double sigma;
  double sentinel; // divergence sentinel 1e6·max|s'|
  int floored;
  int bad_input;
};

struct SweepCounters {
  unsigned long long upd, eu;
  unsigned long long bad, pad;
};

struct KP {
  const int64_t *__restrict__ rp;
  const int32_t *__restrict__ col;
  const float *__restrict__ w;
  const double *__restrict__ d1;
  const Task *__restrict__ tasks;
  const Task *__restrict__ wtasks;
  const Task *__restrict__ rtasks;
  const int *rphase_begin;
  const float *__restrict__ s;  // layout order
  double *z;                    // ẑ' (RELAX/CERT) or z (DIS), layout order
  const Scalars *sc;
  double omega;
  double theta;  // sweep relaxes |r| > θ·h: θ = 1 first, < 1 on certificate resumes
  double2 *partial;
  int *arrive;
  const int *phase_begin;
  const int *wphase_begin;
  int ncolors;
  int ntasks_all;
  int nwtasks_all;
  int max_sweeps;
  unsigned *ctr;          // [3]
  SweepCounters *cnt;     // [3]
  unsigned *bar;          // [2]
  unsigned long long *out;  // [4] sweeps, relaxations, edge updates, reason
  unsigned long long *cert_max;  // double bits
  double *dis;
  double *rout;                  // CERT: optional residual output (layout order)
  int dbg;                       // diagnostics (env FJ_DBG_SKIP): 1 skip warp units, 2 skip tiles
  int dyn;                       // dynamic work claiming in k_sweep (env FJ_DYN)
  int symm;                      // alternate sweep direction (env FJ_SYMM)
};

// CSR streams are read once per sweep: read-only path, no L1 allocation, so
// L1 keeps the gathered ẑ values (hub rows are hit by many arcs)
__device__ __forceinline__ int ld_stream(const int *q) {
  int v;
  asm("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(q));
  return v;
}
__device__ __forceinline__ float ld_stream(const float *q) {
  float v;
  asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(q));
  return v;
}
// ẑ gathers: L1-cached.  ẑ is written during the sweep kernel, so an SM may
// read a value another SM has since replaced; asynchronous relaxation allows
// that (Lemma 3 holds for any order).  Every grid barrier executes a
// gpu-scope fence, which invalidates L1, so the certifying zero-update sweep
// and every color phase read current values.
// (weak loads: the compiler may batch them; __ldca compiles to a strong load)
__device__ __forceinline__ double ld_z(const double *q) { return *q; }

struct dd {
  double hi, lo;
};
__device__ __forceinline__ void dd_add(dd &a, double x) {
  double s = a.hi + x;
  double bb = s - a.hi;
  a.lo += (a.hi - (s - bb)) + (x - bb);
  a.hi = s;
}
__device__ __forceinline__ void dd_addprod(dd &a, double x, double y) {
  double p = x * y;
  double e = fma(x, y, -p);
  dd_add(a, p);
  a.lo += e;
}

template <int MODE>
struct AccT {
  using T = double;
};
template <>
struct AccT<CERT> {
  using T = dd;
};

__device__ __forceinline__ void acc_zero(double &a) { a = 0.0; }
__device__ __forceinline__ void acc_zero(dd &a) { a.hi = a.lo = 0.0; }
__device__ __forceinline__ double acc_shfl(double a, unsigned mask, int off) {
  return __shfl_xor_sync(mask, a, off);
}
__device__ __forceinline__ dd acc_shfl(dd a, unsigned mask, int off) {
  dd b;
  b.hi = __shfl_xor_sync(mask, a.hi, off);
  b.lo = __shfl_xor_sync(mask, a.lo, off);
  return b;
}
__device__ __forceinline__ void acc_merge(double &a, double b) { a += b; }
__device__ __forceinline__ void acc_merge(dd &a, dd b) {
  dd_add(a, b.hi);
  a.lo += b.lo;
}

struct TAcc {
  unsigned long long upd, eu, bad;
  double certmax, dis;
};

// ---------------------------------------------------------- per-row finish
__device__ __forceinline__ double threshold(const Scalars &S, double sp) {
  // h_v (reading R5): ε' s'_v, or (ε/2)·max(σ s'_v/(c+σ), σ) for signed s
  return S.floored ? S.heps * fmax(S.hs * sp, S.sigma) : S.hs * sp;
}

// residual r_i = s'_i − (1+d_i) ẑ_i + Σ_j a_ij ẑ_j combined in double-double:
// at hub rows (d ~ 1e4–1e5) the two large terms cancel to ~h ≈ 5e-12, below
// the rounding noise of a plain fp64 combination
__device__ __forceinline__ double residual_dd(dd sum, double sp, double d1, double zi) {
  dd_add(sum, sp);
  dd_addprod(sum, -d1, zi);
  return sum.hi + sum.lo;
}

template <bool W>
__device__ __forceinline__ void relax_row(const KP &p, const Scalars &S, int row, int len,
                                          dd total, TAcc &t) {
  const double sp = (double)p.s[row] + S.c;              // s' = s + c
  const double h = threshold(S, sp);
  const double zi = __ldcg(p.z + row);
  const double d1 = W ? p.d1[row] : (double)(len + 1);   // a_ii = 1 + d_i (Thm 3)
  const double rho = residual_dd(total, sp, d1, zi);      // r_i = s'_i − ((I+L)ẑ)_i
  const double ar = fabs(rho);
  if (ar > p.theta * h) {                                 // |r_i| > h_i
    __stcg(p.z + row, zi + p.omega * rho / d1);           // equ:sor1
    t.upd++;
    t.eu += (unsigned long long)len;
  }
  if (!(ar <= S.sentinel)) t.bad = 1;
}

// same as relax_row, with the row state loaded by the caller (prefetched)
__device__ __forceinline__ void relax_row_pre(const KP &p, const Scalars &S, int row, int len,
                                              dd total, float sv, double zi, double d1, TAcc &t) {
  const double sp = (double)sv + S.c;
  const double h = threshold(S, sp);
  const double rho = residual_dd(total, sp, d1, zi);
  const double ar = fabs(rho);
  if (ar > p.theta * h) {
    __stcg(p.z + row, zi + p.omega * rho / d1);
    t.upd++;
    t.eu += (unsigned long long)len;
  }
  if (!(ar <= S.sentinel)) t.bad = 1;
}

template <bool W>
__device__ __forceinline__ void cert_row(const KP &p, const Scalars &S, int row, int len, dd total,
                                         TAcc &t) {
  const double sp = (double)p.s[row] + S.c;
  const double h = threshold(S, sp);
  const double zi = p.z[row];
  const double d1 = W ? p.d1[row] : (double)(len + 1);
  const double R = residual_dd(total, sp, d1, zi);
  if (p.rout) p.rout[row] = R;
  const double ratio = fabs(R) / h;
  if (!(ratio <= t.certmax)) t.certmax = ratio;  // NaN sticks
}

// arc accumulation
template <int MODE, bool W>
__device__ __forceinline__ void arc_acc(typename AccT<MODE>::T &a, const KP &p, int64_t k,
                                        double zr) {
  const int j = ld_stream(p.col + k);
  const double wk = W ? (double)ld_stream(p.w + k) : 1.0;
  if constexpr (MODE == RELAX) {
    a = fma(wk, ld_z(p.z + j), a);
  } else if constexpr (MODE == CERT) {
    if (W) dd_addprod(a, wk, p.z[j]);
    else dd_add(a, p.z[j]);
  } else if constexpr (MODE == SPMV) {
    a = fma(wk, p.z[j], a);
  } else {
    const double dz = zr - p.z[j];
    a = fma(wk * dz, dz, a);
  }
}

template <int MODE, int G, bool W>
__device__ __forceinline__ void do_group(const KP &p, const Scalars &S, int rb, int re, TAcc &t) {
  using A = typename AccT<MODE>::T;
  const int lane = threadIdx.x & (G - 1);
  const int grp = threadIdx.x / G;
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
  for (int row = rb + grp; row < re; row += kBlock / G) {
    const int64_t beg = p.rp[row], end = p.rp[row + 1];
    const double zr = (MODE == DIS) ? p.z[row] : 0.0;
    A a;
    acc_zero(a);
#pragma unroll 4
    for (int64_t k = beg + lane; k < end; k += G) arc_acc<MODE, W>(a, p, k, zr);
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) acc_merge(a, acc_shfl(a, gmask, off));
    if (lane == 0) {
      const int len = (int)(end - beg);
      if constexpr (MODE == RELAX) relax_row<W>(p, S, row, len, dd{a, 0.0}, t);
      else if constexpr (MODE == CERT) cert_row<W>(p, S, row, len, a, t);
      else if constexpr (MODE == SPMV) p.rout[row] = a;
      else t.dis += a;
    }
  }
}

// block-wide deterministic reduction; result valid in thread 0
template <class A>
__device__ __forceinline__ A block_reduce(A a, A *sm) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc_merge(a, acc_shfl(a, 0xffffffffu, off));
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sm[w] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kBlock / 32; i++) acc_merge(a, sm[i]);
  }
  __syncthreads();
  return a;
}

// Warp unit (rows above 256 arcs): one warp accumulates a whole row or one
// kWarpPiece-arc piece of it in registers — 8 independent col/w loads, then 8
// ẑ gathers per lane per step — and reduces with shuffles (no block barrier).
// Pieces of one row are combined by the last-arriving warp in piece order
// (deterministic).
template <int MODE, bool W>
__device__ __forceinline__ void do_warp(const KP &p, const Scalars &S, const Task &tk, TAcc &t) {
  // rows above 256 arcs accumulate in double-double for RELAX and CERT
  using A = typename std::conditional<MODE == DIS || MODE == SPMV, double, dd>::type;
#ifndef FJ_WU
#define FJ_WU 8
#endif
  constexpr int U = FJ_WU;  // arcs per lane per step (loads in flight)
  const int lane = threadIdx.x & 31;
  const int row = tk.a, piece = tk.b, np = tk.kind >> 8, slot = tk.slot;
  const int64_t a0 = tk.a0, a1 = tk.a1;
  const double zr = (MODE == DIS) ? p.z[row] : 0.0;
  // RELAX: lanes 1..5 fetch the row state now so that the final relax does
  // not wait on another round trip (s, ẑ_row, 1+d, row_ptr pair)
  double pre = 0.0;
  if constexpr (MODE == RELAX) {
    if (lane == 1) pre = (double)__ldg(p.s + row);
    else if (lane == 2) pre = __ldcg(p.z + row);
    else if (lane == 3 && W) pre = __ldg(p.d1 + row);
    else if (lane == 4) pre = (double)__ldg(p.rp + row);
    else if (lane == 5) pre = (double)__ldg(p.rp + row + 1);
  }
  A a;
  acc_zero(a);
  for (int64_t k0 = a0 + lane; k0 < a1; k0 += 32 * U) {
    // stage 1: all column / weight loads of this step (out-of-range lanes
    // read a valid dummy slot and contribute weight 0)
    int j[U];
    float wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t k = k0 + 32 * u;
      const bool ok = k < a1;
      j[u] = ld_stream(p.col + (ok ? k : a0));
      wv[u] = W ? ld_stream(p.w + (ok ? k : a0)) : 1.0f;
      if (!ok) wv[u] = 0.0f;
    }
    // stage 2: all gathers
    double zj[U];
#pragma unroll
    for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
    // stage 3: accumulate
#pragma unroll
    for (int u = 0; u < U; u++) {
      if constexpr (MODE == SPMV) {
        a = fma((double)wv[u], zj[u], a);
      } else if constexpr (MODE != DIS) {
#ifdef FJ_PLAIN_WARP
        a.hi = fma((double)wv[u], zj[u], a.hi);  // diagnostics only
#else
        dd_addprod(a, (double)wv[u], zj[u]);
#endif
      } else {
        const double dz = zr - zj[u];
        a = fma((double)wv[u] * dz, dz, a);
      }
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc_merge(a, acc_shfl(a, 0xffffffffu, off));
  float sv = 0.f;
  double zi = 0.0, d1 = 0.0;
  int len = 0;
  if constexpr (MODE == RELAX) {
    sv = (float)__shfl_sync(0xffffffffu, pre, 1);
    zi = __shfl_sync(0xffffffffu, pre, 2);
    const double rb = __shfl_sync(0xffffffffu, pre, 4), re = __shfl_sync(0xffffffffu, pre, 5);
    len = (int)(re - rb);
    d1 = W ? __shfl_sync(0xffffffffu, pre, 3) : (double)(len + 1);
  }
  if (lane != 0) return;
  if constexpr (MODE == DIS) {
    t.dis += a;
    return;
  } else if constexpr (MODE == SPMV) {
    atomicAdd(p.rout + row, a);  // pieces of one row add up (y zeroed first)
    return;
  } else {
    if (np > 1) {
      __stcg(p.partial + slot + piece, make_double2(a.hi, a.lo));
      __threadfence();
      // cumulative arrival count: the np-th, 2np-th, ... arrival finishes the
      // row (no reset, so overlapping sweeps of the barrier-free kernel can
      // never lose an arrival; mixing partials of two sweeps is still a
      // valid relaxation amount by Lemma 3 and the certificate decides)
      const int old = atomicAdd(p.arrive + slot, 1);
      if ((old + 1) % np != 0) return;
      __threadfence();
      acc_zero(a);
      for (int q = 0; q < np; q++) {  // fixed order ⇒ deterministic row sum
        const double2 x = __ldcg(p.partial + slot + q);
        acc_merge(a, dd{x.x, x.y});
      }
    }
    if constexpr (MODE == RELAX) {
      // a non-final piece returned above; a multi-piece row is finished by
      // the last-arriving warp, whose prefetched ẑ_row is still current (only
      // this row's finisher writes it, once per phase)
      relax_row_pre(p, S, row, len, a, sv, zi, d1, t);
    } else {
      const int lenc = (int)(__ldg(p.rp + row + 1) - __ldg(p.rp + row));
      cert_row<W>(p, S, row, lenc, a, t);
    }
  }
}

// RELAX on a GROUP task, smem-staged (the hot loop).  All global loads of
// the task are issued up front for memory-level parallelism:
//   row state of the task's rows (rp pair, s, ẑ, 1+d) — one G-lane group per row;
//   phase 1: the task's contiguous arc range, ≤ kTileArcs = 8 per thread:
//            col + w loads, then the ẑ gathers, products a_ij ẑ_j → smem;
//   phase 2: each group sums its row's products from smem, lane 0 relaxes.
// One __syncthreads per task (smem double-buffered across tasks).
template <bool W>
__device__ __forceinline__ void relax_tile(const KP &p, const Scalars &S, const Task &tk, TAcc &t,
                                           double *prod) {
  const int cls = tk.kind & 0xff;
  const int G = 1 << cls;
  const int lane = threadIdx.x & (G - 1);
  const int row = tk.a + (threadIdx.x >> cls);
  const bool has = row < tk.b;
  int64_t beg = 0, end = 0;
  float sv = 0.f;
  double zi = 0.0, d1 = 0.0;
  if (has) {
    beg = __ldg(p.rp + row);
    end = __ldg(p.rp + row + 1);
    if (lane == 0) {
      sv = __ldg(p.s + row);
      zi = __ldcg(p.z + row);
      if (W) d1 = __ldg(p.d1 + row);
    }
  }
  const int64_t a0 = tk.a0;
  const int na = (int)(tk.a1 - a0);
  constexpr int U = kTileArcs / kBlock;
  int j[U];
  float wv[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * kBlock + threadIdx.x;
    const bool ok = e < na;
    j[u] = ld_stream(p.col + a0 + (ok ? e : 0));
    wv[u] = W ? ld_stream(p.w + a0 + (ok ? e : 0)) : 1.0f;
  }
  double zj[U];
#pragma unroll
  for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * kBlock + threadIdx.x;
    if (e < na) prod[e] = (double)wv[u] * zj[u];
  }
  __syncthreads();
  double a = 0.0;
  if (has) {
    const int kb = (int)(beg - a0), ke = (int)(end - a0);
    for (int k = kb + lane; k < ke; k += G) a += prod[k];
  }
  for (int off = G >> 1; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
  if (has && lane == 0) {
    const int len = (int)(end - beg);
    const double sp = (double)sv + S.c;                       // s' = s + c
    const double h = threshold(S, sp);
    if (!W) d1 = (double)(len + 1);                           // a_ii = 1 + d_i
    const double rho = residual_dd(dd{a, 0.0}, sp, d1, zi);  // r_i = s'_i − ((I+L)ẑ)_i
    const double ar = fabs(rho);
    if (ar > p.theta * h) {                                   // |r_i| > h_i
      __stcg(p.z + row, zi + p.omega * rho / d1);             // equ:sor1
      t.upd++;
      t.eu += (unsigned long long)len;
    }
    if (!(ar <= S.sentinel)) t.bad = 1;
  }
}

// RELAX on a warp tile (rows of ≤ 256 arcs, ≤ kWarpTileArcs arcs per tile):
// one warp, no block barrier.  Row state and the tile's arcs are loaded up
// front (≤ 8 column/weight loads then ≤ 8 ẑ gathers per lane), products go to
// the warp's smem slice, then G-lane groups sum their rows (≤ 2 row steps)
// and the group leader relaxes.
template <bool W>
__device__ __forceinline__ void relax_warp_tile(const KP &p, const Scalars &S, const Task &tk,
                                                TAcc &t, double *wprod) {
  constexpr int U = kWarpTileArcs / 32;
  const int lane = threadIdx.x & 31;
  const int cls = tk.kind & 0xff;
  const int G = 1 << cls;
  const int gl = lane & (G - 1);
  const int ng = 32 >> cls;  // groups per warp = rows per step
  // row state is loaded per step in phase 2: loading both steps up front
  // spilled (148 B/thread) and was 9 % slower on C4, 16 % on C5
  int64_t rb[2], re[2];
  float sv[2];
  double zi[2], d1[2];
  const int64_t a0 = tk.a0;
  const int na = (int)(tk.a1 - a0);
  int j[U];
  float wv[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * 32 + lane;
    const bool ok = e < na;
    j[u] = ld_stream(p.col + a0 + (ok ? e : 0));
    wv[u] = W ? ld_stream(p.w + a0 + (ok ? e : 0)) : 1.0f;
  }
  double zj[U];
#pragma unroll
  for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * 32 + lane;
    if (e < na) wprod[e] = (double)wv[u] * zj[u];
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; q++) {
    {
      const int row = tk.a + q * ng + (lane >> cls);
      rb[q] = re[q] = 0;
      sv[q] = 0.f;
      zi[q] = d1[q] = 0.0;
      if (row < tk.b) {
        rb[q] = __ldg(p.rp + row);
        re[q] = __ldg(p.rp + row + 1);
        if (gl == 0) {
          sv[q] = __ldg(p.s + row);
          zi[q] = __ldcg(p.z + row);
          if (W) d1[q] = __ldg(p.d1 + row);
        }
      }
    }
    double a = 0.0;
    const int kb = (int)(rb[q] - a0), ke = (int)(re[q] - a0);
    for (int k = kb + gl; k < ke; k += G) a += wprod[k];
    for (int off = G >> 1; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    const int row = tk.a + q * ng + (lane >> cls);
    if (row < tk.b && gl == 0) {
      const int len = (int)(re[q] - rb[q]);
      relax_row_pre(p, S, row, len, dd{a, 0.0}, sv[q], zi[q], W ? d1[q] : (double)(len + 1), t);
    }
  }
  __syncwarp();  // the slice is reused by this warp's next task
}

// ------------------------------------------------ TMA-pipelined warp stream
// Each warp walks its work items (hub-row warp units, then short-row warp
// tiles) as a stream of <= 256-arc chunks.  The column indices (and weights)
// of chunk i+1 are fetched into the warp's shared-memory stage by a TMA bulk
// copy (cp.async.bulk, completion on an mbarrier) while chunk i is gathered and
// reduced, so the HBM stream runs behind the dependent ẑ gathers without
// holding registers.
constexpr int kChunk = kWarpTileArcs;                       // arcs per chunk
constexpr int kStageElems = kChunk + 8;                     // + 16-byte alignment slack
struct WarpSmem {
  int32_t col[2][kStageElems];
  float w[2][kStageElems];
  double prod[kChunk];
  unsigned long long bar[2];
};

__device__ __forceinline__ uint32_t smem_u32(const void *q) {
  return (uint32_t)__cvta_generic_to_shared(q);
}
__device__ __forceinline__ void mbar_init(unsigned long long *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            unsigned long long *b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}

// lane 0: fetch arcs [c0, c1) of the layout CSR into stage st (16-byte
// aligned superset; the arrays are padded by >= 8 elements)
template <bool W>
__device__ __forceinline__ void chunk_issue(const KP &p, WarpSmem *ws, int st, int64_t c0,
                                            int64_t c1) {
  const int64_t al = c0 & ~(int64_t)3;
  const uint32_t nb = (uint32_t)((((c1 + 3) & ~(int64_t)3) - al) * 4);
  // the stage was last read through the generic proxy (after __syncwarp)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect(&ws->bar[st], W ? 2 * nb : nb);
  tma_load_1d(ws->col[st], p.col + al, nb, &ws->bar[st]);
  if (W) tma_load_1d(ws->w[st], p.w + al, nb, &ws->bar[st]);
}

// relax the rows of a warp tile from a staged chunk
template <bool W>
__device__ __forceinline__ void tile_from_stage(const KP &p, const Scalars &S, const Task &tk,
                                                TAcc &t, WarpSmem *ws, int st, uint32_t par) {
  constexpr int U = kChunk / 32;
  const int lane = threadIdx.x & 31;
  const int cls = tk.kind & 0xff;
  const int G = 1 << cls;
  const int gl = lane & (G - 1);
  const int ng = 32 >> cls;
  int64_t rb[2], re[2];
  float sv[2];
  double zi[2], d1[2];
#pragma unroll
  for (int q = 0; q < 2; q++) {  // row state first: independent of the chunk
    const int row = tk.a + q * ng + (lane >> cls);
    rb[q] = re[q] = 0;
    sv[q] = 0.f;
    zi[q] = d1[q] = 0.0;
    if (row < tk.b) {
      rb[q] = __ldg(p.rp + row);
      re[q] = __ldg(p.rp + row + 1);
      if (gl == 0) {
        sv[q] = __ldg(p.s + row);
        zi[q] = __ldcg(p.z + row);
        if (W) d1[q] = __ldg(p.d1 + row);
      }
    }
  }
  const int64_t a0 = tk.a0;
  const int na = (int)(tk.a1 - a0);
  const int off = (int)(a0 & 3);
  mbar_wait(&ws->bar[st], par);
  int j[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * 32 + lane;
    j[u] = e < na ? ws->col[st][off + e] : -1;
  }
  double zj[U];
#pragma unroll
  for (int u = 0; u < U; u++) zj[u] = j[u] >= 0 ? ld_z(p.z + j[u]) : 0.0;
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * 32 + lane;
    if (e < na) ws->prod[e] = (W ? (double)ws->w[st][off + e] : 1.0) * zj[u];
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; q++) {
    double a = 0.0;
    const int kb = (int)(rb[q] - a0), ke = (int)(re[q] - a0);
    for (int k = kb + gl; k < ke; k += G) a += ws->prod[k];
    for (int o = G >> 1; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    const int row = tk.a + q * ng + (lane >> cls);
    if (row < tk.b && gl == 0) {
      const int len = (int)(re[q] - rb[q]);
      relax_row_pre(p, S, row, len, dd{a, 0.0}, sv[q], zi[q], W ? d1[q] : (double)(len + 1), t);
    }
  }
}

// one warp's work items of a phase, as a TMA-pipelined chunk stream
template <bool W>
__device__ __forceinline__ void relax_stream(const KP &p, const Scalars &S, int r0, int nr,
                                             TAcc &t, WarpSmem *ws, uint32_t &phase_bits) {
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * (kBlock / 32);
  int ti = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  if (ti >= nr) return;
  Task T = p.rtasks[r0 + ti];
  int64_t c0 = T.a0;
  int st = 0;
  if (lane == 0) chunk_issue<W>(p, ws, 0, c0, min(T.a1, c0 + (int64_t)kChunk));
  dd acc{0.0, 0.0};   // warp-unit accumulator (per lane)
  double pre = 0.0;   // warp-unit row state (lanes 1..5)
  bool unit_start = true;
  while (true) {
    const bool unit = (T.kind & 0xff) == kWarp;
    const int64_t c1 = unit ? min(T.a1, c0 + (int64_t)kChunk) : T.a1;
    // next chunk (same unit, or the next work item)
    Task N = T;
    int nti = ti;
    int64_t n0 = c1;
    if (!unit || c1 >= T.a1) {
      nti = ti + stride;
      if (nti < nr) {
        N = p.rtasks[r0 + nti];
        n0 = N.a0;
      }
    }
    const bool has_next = nti < nr;
    if (has_next && lane == 0)
      chunk_issue<W>(p, ws, st ^ 1, n0,
                     (N.kind & 0xff) == kWarp ? min(N.a1, n0 + (int64_t)kChunk) : N.a1);
    const uint32_t par = (phase_bits >> st) & 1u;
    phase_bits ^= 1u << st;
    if (!unit) {
      tile_from_stage<W>(p, S, T, t, ws, st, par);
    } else {
      const int row = T.a;
      if (unit_start) {
        acc = dd{0.0, 0.0};
        pre = 0.0;
        if (lane == 1) pre = (double)__ldg(p.s + row);
        else if (lane == 2) pre = __ldcg(p.z + row);
        else if (lane == 3 && W) pre = __ldg(p.d1 + row);
        else if (lane == 4) pre = (double)__ldg(p.rp + row);
        else if (lane == 5) pre = (double)__ldg(p.rp + row + 1);
      }
      const int off = (int)(c0 & 3);
      const int na = (int)(c1 - c0);
      mbar_wait(&ws->bar[st], par);
      constexpr int U = kChunk / 32;
      int j[U];
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int e = u * 32 + lane;
        j[u] = e < na ? ws->col[st][off + e] : -1;
      }
      double zj[U];
#pragma unroll
      for (int u = 0; u < U; u++) zj[u] = j[u] >= 0 ? ld_z(p.z + j[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; u++) {
        const int e = u * 32 + lane;
        if (e < na) {
          if (W) dd_addprod(acc, (double)ws->w[st][off + e], zj[u]);
          else dd_add(acc, zj[u]);
        }
      }
      if (c1 >= T.a1) {  // unit done: reduce and finish the row (or its piece)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc_merge(acc, acc_shfl(acc, 0xffffffffu, o));
        const float sv = (float)__shfl_sync(0xffffffffu, pre, 1);
        const double zi = __shfl_sync(0xffffffffu, pre, 2);
        const double rbv = __shfl_sync(0xffffffffu, pre, 4), rev = __shfl_sync(0xffffffffu, pre, 5);
        const int len = (int)(rev - rbv);
        const double d1 = W ? __shfl_sync(0xffffffffu, pre, 3) : (double)(len + 1);
        if (lane == 0) {
          const int np = T.kind >> 8;
          bool finish = true;
          if (np > 1) {
            __stcg(p.partial + T.slot + T.b, make_double2(acc.hi, acc.lo));
            __threadfence();
            finish = (atomicAdd(p.arrive + T.slot, 1) + 1) % np == 0;
            if (finish) {
              __threadfence();
              acc = dd{0.0, 0.0};
              for (int q = 0; q < np; q++) {
                const double2 x = __ldcg(p.partial + T.slot + q);
                acc_merge(acc, dd{x.x, x.y});
              }
            }
          }
          if (finish) relax_row_pre(p, S, row, len, acc, sv, zi, d1, t);
        }
      }
    }
    __syncwarp();  // stage st and the product slice are free again
    if (!has_next) break;
    unit_start = !unit || c1 >= T.a1;
    st ^= 1;
    T = N;
    c0 = n0;
    ti = nti;
  }
}

template <int MODE, bool W>
__device__ __forceinline__ void dispatch_tile(const KP &p, const Scalars &S, const Task &tk, TAcc &t) {
  switch (tk.kind & 0xff) {
    case kG1: do_group<MODE, 1, W>(p, S, tk.a, tk.b, t); break;
    case kG2: do_group<MODE, 2, W>(p, S, tk.a, tk.b, t); break;
    case kG4: do_group<MODE, 4, W>(p, S, tk.a, tk.b, t); break;
    case kG8: do_group<MODE, 8, W>(p, S, tk.a, tk.b, t); break;
    case kG16: do_group<MODE, 16, W>(p, S, tk.a, tk.b, t); break;
    default: do_group<MODE, 32, W>(p, S, tk.a, tk.b, t); break;
  }
}

// Grid-wide barrier of a cooperative launch (all CTAs co-resident): one
// arrival counter and a generation word (sense reversal).  The gpu-scope
// fences order every CTA's prior writes (bar.sync makes them cumulative) and
// invalidate L1, so plain ẑ loads after the barrier see current values.
// (A two-level tree measured slower: 6.7 vs 4.5 µs per barrier on 592 CTAs.)
// bar layout: [0] count, [1] generation
__device__ __forceinline__ void grid_sync(unsigned *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(bar[0]), gen(bar[1]);
    const unsigned g = gen.load(cuda::memory_order_relaxed);
    __threadfence();
    if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == gridDim.x - 1) {
      cnt.store(0u, cuda::memory_order_relaxed);
      gen.store(g + 1u, cuda::memory_order_release);
    } else {
      while (gen.load(cuda::memory_order_acquire) == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------ persistent sweeps
#ifndef FJ_MINB
#define FJ_MINB 4
#endif
template <bool W, bool TMA>
__global__ void __launch_bounds__(kBlock, FJ_MINB) k_sweep(KP p) {
  extern __shared__ double s_prod[];  // per warp: a WarpSmem (TMA stages + products)
  __shared__ unsigned long long s_dec[3];
  const Scalars S = *p.sc;
  WarpSmem *ws = reinterpret_cast<WarpSmem *>(s_prod) + (threadIdx.x >> 5);
  uint32_t phase_bits = 0;
  if (TMA && (threadIdx.x & 31) == 0) {
    mbar_init(&ws->bar[0]);
    mbar_init(&ws->bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1;
  int phase = 0;
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k, ++phase) {
      // static round-robin (tasks are balanced by construction; no claim
      // atomics on the hot loop): warp units first (hub rows), then tiles
      const int w0 = p.wphase_begin[k], nw = p.wphase_begin[k + 1] - w0;
      const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
      if (TMA) {
        relax_stream<W>(p, S, p.rphase_begin[k], p.rphase_begin[k + 1] - p.rphase_begin[k], t,
                        ws, phase_bits);
      } else if (p.dyn) {  // dynamic: warps claim kClaim items at a time
        const int r0 = p.rphase_begin[k], nr = p.rphase_begin[k + 1] - r0;
        double *wprod = s_prod + (threadIdx.x >> 5) * kWarpTileArcs;
        const int lane = threadIdx.x & 31;
        if (blockIdx.x == 0 && threadIdx.x == 0) p.ctr[(phase + 2) % 3] = 0u;
        for (;;) {
          int base = 0;
          if (lane == 0) base = (int)atomicAdd(p.ctr + phase % 3, (unsigned)kClaim);
          base = __shfl_sync(0xffffffffu, base, 0);
          if (base >= nr) break;
          const int end = min(nr, base + kClaim);
          for (int wi = base; wi < end; wi++) {
            const Task cur = p.rtasks[r0 + wi];
            if ((cur.kind & 0xff) == kWarp) do_warp<RELAX, W>(p, S, cur, t);
            else relax_warp_tile<W>(p, S, cur, t, wprod);
          }
        }
      } else {  // static round-robin: one warp per work item, next item prefetched
        const int r0 = p.rphase_begin[k], nr = p.rphase_begin[k + 1] - r0;
        const int stride = gridDim.x * (kBlock / 32);
        double *wprod = s_prod + (threadIdx.x >> 5) * kWarpTileArcs;
        // FJ_SYMM: odd sweeps walk the work list backwards (symmetric ordering)
        const bool rev = p.symm && (sw & 1);
        int wi = warp_id;
        Task nxt;
        if (wi < nr) nxt = p.rtasks[r0 + (rev ? nr - 1 - wi : wi)];
        while (wi < nr) {
          const Task cur = nxt;
          const int wn = wi + stride;
          if (wn < nr) nxt = p.rtasks[r0 + (rev ? nr - 1 - wn : wn)];
          if ((cur.kind & 0xff) == kWarp) {
            if (!(p.dbg & 1)) do_warp<RELAX, W>(p, S, cur, t);
          } else if (!(p.dbg & 2)) {
            relax_warp_tile<W>(p, S, cur, t, wprod);
          }
          wi = wn;
        }
      }
      if (k + 1 < p.ncolors) grid_sync(p.bar);
    }
    // commit this sweep's counters (warp-aggregated atomics)
    unsigned long long u = t.upd, e = t.eu, b = t.bad;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, off);
      e += __shfl_xor_sync(0xffffffffu, e, off);
      b |= __shfl_xor_sync(0xffffffffu, b, off);
    }
    SweepCounters *c = p.cnt + sw % 3;
    if ((threadIdx.x & 31) == 0 && (u | e | b)) {
      atomicAdd(&c->upd, u);
      atomicAdd(&c->eu, e);
      if (b) atomicOr(&c->bad, b);
    }
    t.upd = t.eu = t.bad = 0;
    grid_sync(p.bar);
    if (threadIdx.x == 0) {
      s_dec[0] = __ldcg(&c->upd);
      s_dec[1] = __ldcg(&c->eu);
      s_dec[2] = __ldcg(&c->bad);
      if (blockIdx.x == 0) {
        SweepCounters *z = p.cnt + (sw + 2) % 3;
        z->upd = z->eu = z->bad = 0;
      }
    }
    __syncthreads();
    tot_upd += s_dec[0];
    tot_eu += s_dec[1];
    sweeps = sw + 1;
    const bool bad = s_dec[2] != 0, done = s_dec[0] == 0;
    __syncthreads();
    if (bad) { reason = 2; break; }
    if (done) { reason = 0; break; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.out[0] = (unsigned long long)sweeps;
    p.out[1] = tot_upd;
    p.out[2] = tot_eu;
    p.out[3] = (unsigned long long)reason;
  }
}

// ------------------------------------------- barrier-free asynchronous sweeps
// ASYNC with one phase: warps claim batches of work items from one monotonic
// counter; item c belongs to epoch (sweep) c / nr.  Epochs therefore run back
// to back without a grid barrier, and the claim order balances the load.  The
// warp that completes an epoch checks its update count: zero updates (no row
// had |r| > h when evaluated) stops the loop — the paper's Q = ∅ — and the
// host-side compensated certificate decides (resuming if a row slipped).
constexpr int kRing = 8;     // per-epoch counter slots
struct AsyncCtl {
  unsigned long long next;                 // claim counter (items)
  unsigned long long upd[kRing], eu[kRing], done[kRing];
  unsigned long long tot_upd, tot_eu;
  unsigned int stop, bad, epochs, pad;
};

// settle one warp's counts for an epoch part: warp-reduce, then lane 0 adds
// them; the warp that completes the epoch decides whether to stop
__device__ __forceinline__ void async_settle(AsyncCtl *c, unsigned long long ep,
                                             unsigned long long nr, TAcc &t,
                                             unsigned long long cnt) {
  unsigned long long u = t.upd, e2 = t.eu, b = t.bad;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, off);
    e2 += __shfl_xor_sync(0xffffffffu, e2, off);
    b |= __shfl_xor_sync(0xffffffffu, b, off);
  }
  t = TAcc{};
  if ((threadIdx.x & 31) != 0 || cnt == 0) return;
  const int slot = (int)(ep % kRing);
  if (u) atomicAdd(&c->upd[slot], u);
  atomicAdd(&c->tot_upd, u);
  atomicAdd(&c->tot_eu, e2);
  if (b) atomicOr(&c->bad, 1u);
  __threadfence();
  if (atomicAdd(&c->done[slot], cnt) + cnt == nr) {  // epoch ep complete
    __threadfence();
    const unsigned long long uu = atomicAdd(&c->upd[slot], 0ull);
    atomicMax(&c->epochs, (unsigned int)(ep + 1));
    if (uu == 0 || atomicAdd(&c->bad, 0u)) atomicExch(&c->stop, 1u);
    const int z = (int)((ep + kRing / 2) % kRing);  // recycle a slot well ahead
    c->upd[z] = 0;
    c->done[z] = 0;
  }
}

// out[0..3] = sweeps, relaxations, edge updates, reason (as k_sweep writes)
__global__ void k_async_result(const AsyncCtl *c, unsigned long long *out,
                               unsigned long long max_sweeps) {
  out[0] = c->epochs;
  out[1] = c->tot_upd;
  out[2] = c->tot_eu;
  out[3] = c->bad ? 2ull : (c->stop ? 0ull : 1ull);
}

template <bool W>
__global__ void __launch_bounds__(kBlock, FJ_MINB) k_sweep_async(KP p, AsyncCtl *c) {
  extern __shared__ double s_prod[];
  const Scalars S = *p.sc;
  const int lane = threadIdx.x & 31;
  double *wprod = s_prod + (threadIdx.x >> 5) * kWarpTileArcs;
  const unsigned long long nr = (unsigned long long)(p.rphase_begin[1] - p.rphase_begin[0]);
  const Task *items = p.rtasks + p.rphase_begin[0];
  const unsigned long long limit = nr * (unsigned long long)p.max_sweeps;
  unsigned long long my_epoch = ~0ull;
  TAcc t{};
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&c->next, (unsigned long long)kClaim);
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned int stop = *(volatile unsigned int *)&c->stop;
    if (stop || base >= limit || nr == 0) break;
    unsigned long long ep = base / nr, cnt = 0;
    // bounded staleness: a warp may run at most kRing/2 - 1 sweeps ahead of
    // the oldest unfinished one (keeps the per-sweep counter slots distinct;
    // the oldest sweep's holders are never blocked, so this cannot deadlock)
    if (lane == 0)
      while (ep >= (unsigned long long)*(volatile unsigned int *)&c->epochs + kRing / 2 - 1 &&
             !*(volatile unsigned int *)&c->stop)
        __nanosleep(256);
    __syncwarp();
    for (int q = 0; q < kClaim; q++) {
      const unsigned long long it = base + q;
      if (it >= limit) break;
      const unsigned long long e = it / nr;
      if (e != ep) {  // the batch straddles two epochs: settle the first part
        async_settle(c, ep, nr, t, cnt);
        cnt = 0;
        ep = e;
      }
      if (e != my_epoch) {  // a new sweep for this warp: drop stale L1 lines of ẑ
        __threadfence();
        my_epoch = e;
      }
      const Task tk = items[it - e * nr];
      if ((tk.kind & 0xff) == kWarp) do_warp<RELAX, W>(p, S, tk, t);
      else relax_warp_tile<W>(p, S, tk, t, wprod);
      cnt++;
    }
    async_settle(c, ep, nr, t, cnt);
  }
}

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

template <int K>
__device__ __forceinline__ void relax_rowK(const KP &p, const Scalars *SK, int row, int len,
                                           dd (&tot)[K], const float (&sv)[K],
                                           const double (&zi)[K], double d1, TAcc &t) {
  double out[K];
#pragma unroll
  for (int r = 0; r < K; r++) {
    const Scalars &S = SK[r];
    const double sp = (double)sv[r] + S.c;
    const double h = threshold(S, sp);
    const double rho = residual_dd(tot[r], sp, d1, zi[r]);
    const double ar = fabs(rho);
    out[r] = zi[r];
    if (ar > p.theta * h) {
      out[r] = zi[r] + p.omega * rho / d1;
      t.upd++;
      t.eu += (unsigned long long)len;
    }
    if (!(ar <= S.sentinel)) t.bad = 1;
  }
  double2 *q = reinterpret_cast<double2 *>(p.z + (int64_t)row * K);
#pragma unroll
  for (int h = 0; h < K / 2; h++) __stcg(q + h, make_double2(out[2 * h], out[2 * h + 1]));
}

// warp unit (row > kWarpTileArcs arcs, or a piece of one), K right-hand sides
template <bool W, int K>
__device__ __forceinline__ void do_warpK(const KP &p, const Scalars *SK, const Task &tk, TAcc &t) {
  constexpr int U = 4;
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
      wv[u] = ok ? (W ? ld_stream(p.w + k) : 1.0f) : 0.0f;
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
    __threadfence();
    const int old = atomicAdd(p.arrive + slot, 1);
    if ((old + 1) % np != 0) return;
    __threadfence();
#pragma unroll
    for (int r = 0; r < K; r++) a[r] = dd{0.0, 0.0};
    for (int q = 0; q < np; q++)
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 x = __ldcg(p.partial + ((int64_t)slot + q) * K + r);
        acc_merge(a[r], dd{x.x, x.y});
      }
  }
  relax_rowK<K>(p, SK, row, len, a, sv, zi, d1, t);
}

// warp tile (short rows), K right-hand sides: G lanes per row accumulate
// directly in registers (no shared memory), two row steps
template <bool W, int K>
__device__ __forceinline__ void tileK(const KP &p, const Scalars *SK, const Task &tk, TAcc &t) {
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
#pragma unroll 4
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
      relax_rowK<K>(p, SK, row, len, tot, sv, zi, W ? d1 : (double)(len + 1), t);
    }
  }
}

template <bool W, int K>
__global__ void __launch_bounds__(kBlock, 4) k_sweep_batch(KP p, AsyncCtl *c) {
  __shared__ Scalars sk[K];
  if (threadIdx.x < K) sk[threadIdx.x] = p.sc[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const unsigned long long nr = (unsigned long long)(p.rphase_begin[1] - p.rphase_begin[0]);
  const Task *items = p.rtasks + p.rphase_begin[0];
  const unsigned long long limit = nr * (unsigned long long)p.max_sweeps;
  unsigned long long my_epoch = ~0ull;
  TAcc t{};
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&c->next, (unsigned long long)kClaim);
    base = __shfl_sync(0xffffffffu, base, 0);
    const unsigned int stop = *(volatile unsigned int *)&c->stop;
    if (stop || base >= limit || nr == 0) break;
    unsigned long long ep = base / nr, cnt = 0;
    // bounded staleness: a warp may run at most kRing/2 - 1 sweeps ahead of
    // the oldest unfinished one (keeps the per-sweep counter slots distinct;
    // the oldest sweep's holders are never blocked, so this cannot deadlock)
    if (lane == 0)
      while (ep >= (unsigned long long)*(volatile unsigned int *)&c->epochs + kRing / 2 - 1 &&
             !*(volatile unsigned int *)&c->stop)
        __nanosleep(256);
    __syncwarp();
    for (int q = 0; q < kClaim; q++) {
      const unsigned long long it = base + q;
      if (it >= limit) break;
      const unsigned long long e = it / nr;
      if (e != ep) {
        async_settle(c, ep, nr, t, cnt);
        cnt = 0;
        ep = e;
      }
      if (e != my_epoch) {
        __threadfence();
        my_epoch = e;
      }
      const Task tk = items[it - e * nr];
      if ((tk.kind & 0xff) == kWarp) do_warpK<W, K>(p, sk, tk, t);
      else tileK<W, K>(p, sk, tk, t);
      cnt++;
    }
    async_settle(c, ep, nr, t, cnt);
  }
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
__global__ void k_finalize_batch(int64_t n, int k, int K, const int32_t *__restrict__ iperm,
                                 const double *__restrict__ zK, const Scalars *__restrict__ SK,
                                 float *__restrict__ Z) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t i = iperm[u];
  for (int r = 0; r < k; r++) Z[u * k + r] = (float)(zK[i * K + r] - SK[r].c);
}

// ------------------------------------------ one pass over all tasks (CERT/DIS)
template <int MODE, bool W>
__global__ void __launch_bounds__(kBlock, 4) k_pass(KP p) {
  Scalars S{};
  if (MODE == CERT) S = *p.sc;
  TAcc t{};
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  for (int wi = warp_id; wi < p.nwtasks_all; wi += gridDim.x * (kBlock / 32))
    do_warp<MODE, W>(p, S, p.wtasks[wi], t);
  for (int ti = blockIdx.x; ti < p.ntasks_all; ti += gridDim.x)
    dispatch_tile<MODE, W>(p, S, p.tasks[ti], t);
  if constexpr (MODE == CERT) {
    double m = t.certmax;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (isnan(t.certmax)) m = t.certmax;
    if ((threadIdx.x & 31) == 0 && m != 0.0)
      atomicMax(p.cert_max, (unsigned long long)__double_as_longlong(m));
  } else if constexpr (MODE == DIS) {
    double sdis = t.dis;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sdis += __shfl_xor_sync(0xffffffffu, sdis, off);
    if ((threadIdx.x & 31) == 0 && sdis != 0.0) atomicAdd(p.dis, sdis);
  }
}

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
  int64_t n;
  const float *__restrict__ s;
  double *z, *r, *q;
  const Scalars *sc;
  double omega, theta;
  int max_sweeps;
  unsigned *bar;
  SweepCounters *cnt;
  unsigned long long *out;
};

__device__ __forceinline__ void push_pop(const PP &p, const Scalars &S, int64_t b, int64_t e,
                                         TAcc &t) {
  for (int64_t v = b + blockIdx.x * (int64_t)kBlock + threadIdx.x; v < e;
       v += (int64_t)gridDim.x * kBlock) {
    const double sp = (double)p.s[v] + S.c;
    const double h = threshold(S, sp);
    const double rv = p.r[v];
    double qv = 0.0;
    if (fabs(rv) > p.theta * h) {                       // |r_v| > h_v
      qv = p.omega * rv / p.d1[v];                      // ω r_v/(1+d_v)
      p.z[v] += qv;                                     // equ:sor1
      p.r[v] = rv - p.omega * rv;                       // equ:sor2: (1−ω) r_v
      t.upd++;
      t.eu += (unsigned long long)(p.rp[v + 1] - p.rp[v]);
    }
    if (!(fabs(rv) <= S.sentinel)) t.bad = 1;
    p.q[v] = qv;
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

template <bool W>
__global__ void __launch_bounds__(kBlock, 4) k_push(PP p) {
  __shared__ unsigned long long s_dec[3];
  const Scalars S = *p.sc;
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1;
  const int lane = threadIdx.x & 31;
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k) {
      push_pop(p, S, p.crow[k], p.crow[k + 1], t);
      if (k == p.ncolors - 1) push_pop(p, S, p.crow[p.ncolors], p.n, t);  // rows with no in-arcs
      grid_sync(p.bar);
      // B: warp units (long scatter lists), then tile tasks (group per row)
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
    unsigned long long u = t.upd, e = t.eu, b = t.bad;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      u += __shfl_xor_sync(0xffffffffu, u, off);
      e += __shfl_xor_sync(0xffffffffu, e, off);
      b |= __shfl_xor_sync(0xffffffffu, b, off);
    }
    SweepCounters *c = p.cnt + sw % 3;
    if (lane == 0 && (u | e | b)) {
      atomicAdd(&c->upd, u);
      atomicAdd(&c->eu, e);
      if (b) atomicOr(&c->bad, b);
    }
    t.upd = t.eu = t.bad = 0;
    grid_sync(p.bar);
    if (threadIdx.x == 0) {
      s_dec[0] = __ldcg(&c->upd);
      s_dec[1] = __ldcg(&c->eu);
      s_dec[2] = __ldcg(&c->bad);
      if (blockIdx.x == 0) {
        SweepCounters *zc = p.cnt + (sw + 2) % 3;
        zc->upd = zc->eu = zc->bad = 0;
      }
    }
    __syncthreads();
    tot_upd += s_dec[0];
    tot_eu += s_dec[1];
    sweeps = sw + 1;
    const bool bad = s_dec[2] != 0, done = s_dec[0] == 0;
    __syncthreads();
    if (bad) { reason = 2; break; }
    if (done) { reason = 0; break; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.out[0] = (unsigned long long)sweeps;
    p.out[1] = tot_upd;
    p.out[2] = tot_eu;
    p.out[3] = (unsigned long long)reason;
  }
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

// ----------------------------------------------------------- node kernels
__global__ void k_scalars(const float *__restrict__ smin, const float *__restrict__ smax,
                          double eps, double sigma, double c_override, Scalars *S) {
  const double lo = (double)*smin, hi = (double)*smax;
  Scalars s{};
  s.bad_input = !(isfinite(lo) && isfinite(hi));
  s.sigma = sigma;
  s.c = c_override > 0 ? c_override : sigma + fmax(0.0, -lo);   // reading R5
  s.eps_p = sigma / (s.c + sigma) * eps;
  s.floored = lo < 0.0;
  s.hs = s.floored ? sigma / (s.c + sigma) : s.eps_p;
  s.heps = 0.5 * eps;
  s.sentinel = 1e6 * fmax(fabs(hi + s.c), fabs(lo + s.c));
  *S = s;
}

// s into layout order; ẑ' = 0 (Alg. 1 init) except rows with no arcs,
// whose equation is (1 + 0) z_v = s'_v: solved exactly (ẑ'_v = s'_v)
__global__ void k_init(int64_t n, const int32_t *__restrict__ perm, const int64_t *__restrict__ rp,
                       const float *__restrict__ s, Scalars *__restrict__ S,
                       float *__restrict__ s_l, double *__restrict__ z,
                       const double *__restrict__ z_init = nullptr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float si = s[perm[i]];
  if (!isfinite(si)) atomicOr(&S->bad_input, 1);  // min/max reductions skip NaN
  s_l[i] = si;
  if (rp[i + 1] == rp[i]) z[i] = (double)si + S->c;          // d = 0: exact
  else if (z_init) {                                          // warm start (Lemma 3)
    const double v = z_init[perm[i]] + S->c;
    if (!isfinite(v)) atomicOr(&S->bad_input, 2);
    z[i] = v;
  } else z[i] = 0.0;                                          // Alg. 1 init
}

__global__ void k_finalize(int64_t n, const int32_t *__restrict__ iperm, const double *__restrict__ z,
                           const Scalars *__restrict__ S, float *__restrict__ zout,
                           double *__restrict__ zprime) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const double zp = z[iperm[u]];
  zout[u] = (float)(zp - S->c);  // ẑ_v − c
  if (zprime) zprime[u] = zp;
}

// measures node pass: z into layout order (fp64) + Σz
__global__ void k_meas_nodes1(int64_t n, const int32_t *__restrict__ perm,
                              const float *__restrict__ z, double *__restrict__ zl,
                              double *__restrict__ sums) {
  __shared__ double sm[kBlock / 32];
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    v = (double)z[perm[i]];
    zl[i] = v;
  }
  v = block_reduce<double>(v, sm);
  if (threadIdx.x == 0) atomicAdd(sums, v);
}

// Σ (z − mean)², Σ (z − s)², Σ z²  (two-pass mean, reading R15)
__global__ void k_meas_nodes2(int64_t n, const float *__restrict__ z, const float *__restrict__ s,
                              double *__restrict__ sums) {
  __shared__ double sm[kBlock / 32];
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double mean = sums[0] / (double)n;
  double P = 0, I = 0, C = 0;
  if (i < n) {
    const double zi = (double)z[i];
    P = (zi - mean) * (zi - mean);
    C = zi * zi;
    if (s) I = (zi - (double)s[i]) * (zi - (double)s[i]);
  }
  P = block_reduce<double>(P, sm);
  I = block_reduce<double>(I, sm);
  C = block_reduce<double>(C, sm);
  if (threadIdx.x == 0) {
    atomicAdd(sums + 1, P);
    atomicAdd(sums + 2, I);
    atomicAdd(sums + 3, C);
  }
}

// ------------------------------------------------------------- host side
static unsigned gridn(int64_t work) {
  int64_t b = (work + kBlock - 1) / kBlock;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 1 << 30));
}

static int persistent_grid(const void *fn, int num_sms, size_t smem = 0) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kBlock, smem);
  if (per_sm < 1) per_sm = 1;
  return per_sm * num_sms;
}

struct Staged {
  const float *dev = nullptr;
  float *owned = nullptr;
};

static fj_status stage_in(const float *src, int64_t n, cudaStream_t st, Staged &out) {
  if (is_device_ptr(src)) {
    out.dev = src;
    return FJ_OK;
  }
  FJ_CUDA(cudaMallocAsync(&out.owned, sizeof(float) * n, st));
  FJ_CUDA(cudaMemcpyAsync(out.owned, src, sizeof(float) * n, cudaMemcpyHostToDevice, st));
  out.dev = out.owned;
  return FJ_OK;
}

static KP make_kp(const fj_graph *g, const Layout &L) {
  KP p{};
  p.rp = L.rp;
  p.col = L.col;
  p.w = L.w;
  p.d1 = L.d1;
  p.tasks = L.tasks;
  p.wtasks = L.wtasks;
  p.rtasks = L.rtasks;
  p.rphase_begin = L.d_rphase_begin;
  p.phase_begin = L.d_phase_begin;
  p.wphase_begin = L.d_wphase_begin;
  p.ncolors = L.ncolors;
  p.ntasks_all = L.ntasks;
  p.nwtasks_all = L.nwtasks;
  return p;
}

static fj_status finish_status(const Scalars &hs, fj_stats &stats, const fj_opts *o,
                               double omega) {
  fj_status rc = FJ_OK;
  if (hs.bad_input) {
    set_error("fj_solve: s (or z_init) contains a non-finite value");
    rc = FJ_ERR_INVALID;
  } else if (stats.reason == 1) {
    set_error("fj_solve: watchdog, %lld sweeps without convergence", (long long)stats.sweeps);
    rc = FJ_ERR_NUMERIC;
  } else if (stats.reason == 2) {
    set_error("fj_solve: divergence sentinel |r| > 1e6 max|s'| (omega = %g)", omega);
    rc = FJ_ERR_NUMERIC;
  } else if (o->certify && !(stats.cert_ratio <= 1.0)) {
    set_error("fj_solve: fp64 residual certificate failed (max |r|/h = %g)", stats.cert_ratio);
    rc = FJ_ERR_NUMERIC;
  }
  stats.status = rc;
  return rc;
}

// FJ_METHOD_PUSH: frontier push on the in-row layout; certificate on the pull
// layout (the residual needs out-rows); residual replacement on resume.
static fj_status push_solve_impl(fj_graph *g, const float *s_in, double eps, double omega,
                                 const fj_opts *o, float *z_out, fj_stats *st_out) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  const bool colored = omega != 1.0;
  if (colored && !g->colors) FJ_TRY(build_coloring(g));
  Layout &P = colored ? g->push_color_layout : g->push_layout;
  if (!P.tasks)
    FJ_TRY(build_layout_from_out(g, g->in_rp, g->in_col, g->in_w, colored ? g->colors : nullptr,
                                 colored ? g->ncolors : 1, &P, true));
  const Layout &L = g->async_layout;
  const bool W = g->weighted != 0;
  fj_stats stats{};
  stats.colors = P.ncolors;

  cudaEvent_t e0, e1, es0, es1;
  FJ_CUDA(cudaEventCreate(&e0));
  FJ_CUDA(cudaEventCreate(&e1));
  FJ_CUDA(cudaEventCreate(&es0));
  FJ_CUDA(cudaEventCreate(&es1));
  FJ_CUDA(cudaEventRecord(e0, st));
  Staged s{};
  FJ_TRY(stage_in(s_in, n, st, s));
  const bool zdev = is_device_ptr(z_out);
  const bool zpdev = o->zprime_out && is_device_ptr(o->zprime_out);
  float *sP = nullptr, *sL = nullptr, *smin = nullptr, *zo = nullptr;
  double *zP = nullptr, *rP = nullptr, *qP = nullptr, *zL = nullptr, *tmp = nullptr, *zp = nullptr;
  double *RL = nullptr;
  Scalars *S = nullptr;
  unsigned *ctl = nullptr;
  SweepCounters *cnt = nullptr;
  unsigned long long *outv = nullptr;
  FJ_CUDA(cudaMallocAsync(&sP, sizeof(float) * n, st));
  FJ_CUDA(cudaMallocAsync(&sL, sizeof(float) * n, st));
  FJ_CUDA(cudaMallocAsync(&zP, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&rP, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&qP, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&zL, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&tmp, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&RL, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&smin, sizeof(float) * 2, st));
  FJ_CUDA(cudaMallocAsync(&S, sizeof(Scalars), st));
  FJ_CUDA(cudaMallocAsync(&ctl, sizeof(unsigned) * kCtlWords, st));
  FJ_CUDA(cudaMallocAsync(&cnt, sizeof(SweepCounters) * 3, st));
  FJ_CUDA(cudaMallocAsync(&outv, sizeof(unsigned long long) * 8, st));
  if (!zdev) FJ_CUDA(cudaMallocAsync(&zo, sizeof(float) * n, st));
  if (o->zprime_out && !zpdev) FJ_CUDA(cudaMallocAsync(&zp, sizeof(double) * n, st));
  {
    size_t t1 = 0, t2 = 0;
    FJ_CUDA(cub::DeviceReduce::Min(nullptr, t1, s.dev, smin, n, st));
    FJ_CUDA(cub::DeviceReduce::Max(nullptr, t2, s.dev, smin + 1, n, st));
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, std::max(t1, t2), st));
    FJ_CUDA(cub::DeviceReduce::Min(t, t1, s.dev, smin, n, st));
    FJ_CUDA(cub::DeviceReduce::Max(t, t2, s.dev, smin + 1, n, st));
    FJ_CUDA(cudaFreeAsync(t, st));
  }
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
  KP kq = make_kp(g, L);
  kq.s = sL;
  kq.z = zL;
  kq.sc = S;
  kq.ctr = ctl + 5;
  kq.cert_max = outv + 4;
  kq.rout = RL;
  double2 *partial = nullptr;  // long-row partials of the pull layout (certificate)
  int *arrive = nullptr;
  FJ_CUDA(cudaMallocAsync(&partial, sizeof(double2) * std::max(1, L.npartials), st));
  FJ_CUDA(cudaMallocAsync(&arrive, sizeof(int) * std::max(1, L.npartials), st));
  FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
  kq.partial = partial;
  kq.arrive = arrive;

  const void *fn = W ? (const void *)k_push<true> : (const void *)k_push<false>;
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
  for (void *q : {(void *)sP, (void *)sL, (void *)zP, (void *)rP, (void *)qP, (void *)zL,
                  (void *)tmp, (void *)RL, (void *)smin, (void *)S, (void *)ctl, (void *)cnt,
                  (void *)outv, (void *)zo, (void *)zp, (void *)s.owned, (void *)partial,
                  (void *)arrive})
    if (q) cudaFreeAsync(q, st);
  for (cudaEvent_t e : {e0, e1, es0, es1}) cudaEventDestroy(e);
  FJ_CUDA(cudaGetLastError());
  fj_status rc = finish_status(hs, stats, o, omega);
  if (st_out) *st_out = stats;
  return rc;
}

// k ≤ 4 right-hand sides per solve, ASYNC schedule, one
// certificate per right-hand side
static fj_status batch_solve_impl(fj_graph *g, const float *S_in, int k, double eps, double omega,
                                  const fj_opts *o, float *Z_out, fj_stats *st_out) {
  NvtxRange nv("fj_solve_batch");
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  const int K = k <= 2 ? 2 : 4;
  const Layout &L = g->async_layout;
  const bool W = g->weighted != 0;
  fj_stats stats{};
  stats.colors = 1;
  cudaEvent_t e0, e1, es0, es1;
  FJ_CUDA(cudaEventCreate(&e0));
  FJ_CUDA(cudaEventCreate(&e1));
  FJ_CUDA(cudaEventCreate(&es0));
  FJ_CUDA(cudaEventCreate(&es1));
  FJ_CUDA(cudaEventRecord(e0, st));
  const float *S = S_in;
  float *S_owned = nullptr;
  if (!is_device_ptr(S_in)) {
    FJ_CUDA(cudaMallocAsync(&S_owned, sizeof(float) * n * k, st));
    FJ_CUDA(cudaMemcpyAsync(S_owned, S_in, sizeof(float) * n * k, cudaMemcpyHostToDevice, st));
    S = S_owned;
  }
  const bool zdev = is_device_ptr(Z_out);
  float *sK = nullptr, *col = nullptr, *mm = nullptr, *s1 = nullptr, *Zd = nullptr;
  double *zK = nullptr, *z1 = nullptr;
  double2 *partial = nullptr;
  int *arrive = nullptr, *arrive2 = nullptr;
  Scalars *SK = nullptr;
  AsyncCtl *actl = nullptr;
  unsigned long long *outv = nullptr;
  unsigned *ctl = nullptr;
  const size_t np = (size_t)std::max(1, L.npartials);
  FJ_CUDA(cudaMallocAsync(&sK, sizeof(float) * n * K, st));
  FJ_CUDA(cudaMallocAsync(&zK, sizeof(double) * n * K, st));
  FJ_CUDA(cudaMallocAsync(&col, sizeof(float) * n, st));
  FJ_CUDA(cudaMallocAsync(&mm, sizeof(float) * 2, st));
  FJ_CUDA(cudaMallocAsync(&s1, sizeof(float) * n, st));
  FJ_CUDA(cudaMallocAsync(&z1, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&partial, sizeof(double2) * np * K, st));
  FJ_CUDA(cudaMallocAsync(&arrive, sizeof(int) * np, st));
  FJ_CUDA(cudaMallocAsync(&arrive2, sizeof(int) * np, st));
  FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * np, st));
  FJ_CUDA(cudaMallocAsync(&SK, sizeof(Scalars) * K, st));
  FJ_CUDA(cudaMallocAsync(&actl, sizeof(AsyncCtl), st));
  FJ_CUDA(cudaMallocAsync(&outv, sizeof(unsigned long long) * 8, st));
  FJ_CUDA(cudaMallocAsync(&ctl, sizeof(unsigned) * 8, st));
  if (!zdev) FJ_CUDA(cudaMallocAsync(&Zd, sizeof(float) * n * k, st));
  // a2 per right-hand side: shift and thresholds (Alg. 2, reading R5)
  {
    size_t t1 = 0, t2 = 0;
    FJ_CUDA(cub::DeviceReduce::Min(nullptr, t1, col, mm, n, st));
    FJ_CUDA(cub::DeviceReduce::Max(nullptr, t2, col, mm + 1, n, st));
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, std::max(t1, t2), st));
    for (int r = 0; r < K; r++) {
      fj::count_launch();
      k_column<<<gridn(n), kBlock, 0, st>>>(n, k, r < k ? r : k - 1, S, col);
      FJ_CUDA(cub::DeviceReduce::Min(t, t1, col, mm, n, st));
      FJ_CUDA(cub::DeviceReduce::Max(t, t2, col, mm + 1, n, st));
      fj::count_launch();
      k_scalars<<<1, 1, 0, st>>>(mm, mm + 1, eps, o->sigma, o->c, SK + r);
    }
    FJ_CUDA(cudaFreeAsync(t, st));
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
  const void *fn = K == 2 ? (W ? (const void *)k_sweep_batch<true, 2> : (const void *)k_sweep_batch<false, 2>)
                          : (W ? (const void *)k_sweep_batch<true, 4> : (const void *)k_sweep_batch<false, 4>);
  const int grid = persistent_grid(fn, g->num_sms);
  const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
  const int cgrid = persistent_grid(cf, g->num_sms);
  float ms_sweep = 0;
  int rounds = 0;
  for (;;) {
    FJ_CUDA(cudaMemsetAsync(actl, 0, sizeof(AsyncCtl), st));
    FJ_CUDA(cudaMemsetAsync(outv, 0, sizeof(unsigned long long) * 8, st));
    FJ_CUDA(cudaEventRecord(es0, st));
    void *args[] = {&p, &actl};
    fj::count_launch();
    FJ_CUDA(cudaLaunchKernel(fn, grid, kBlock, args, 0, st));
    fj::count_launch();
    k_async_result<<<1, 1, 0, st>>>(actl, outv, (unsigned long long)p.max_sweeps);
    FJ_CUDA(cudaEventRecord(es1, st));
    unsigned long long h[8];
    FJ_CUDA(cudaMemcpyAsync(h, outv, sizeof(h), cudaMemcpyDeviceToHost, st));
    // compensated certificate of every right-hand side
    double worst = 0.0;
    for (int r = 0; r < k; r++) {
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
    }
    FJ_CUDA(cudaStreamSynchronize(st));
    float a = 0;
    FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
    ms_sweep += a;
    stats.sweeps += (int64_t)h[0];
    stats.relaxations += (int64_t)h[1];
    stats.edge_updates += (int64_t)h[2];
    stats.reason = (int)h[3];
    stats.cert_ratio = worst;
    if (stats.reason != 0 || stats.cert_ratio <= 1.0 || rounds >= o->cert_rounds) break;
    rounds++;
    p.theta *= 0.5;
    p.max_sweeps = std::min(o->max_sweeps, 2000);
  }
  stats.cert_rounds = rounds;
  stats.phases = stats.sweeps;
  stats.rows_read = stats.sweeps * L.active_rows;
  stats.arcs_read = stats.sweeps * L.m;
  stats.relaxations += L.empty_rows * k;
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
  for (void *q : {(void *)sK, (void *)zK, (void *)col, (void *)mm, (void *)s1, (void *)z1,
                  (void *)partial, (void *)arrive, (void *)arrive2, (void *)SK, (void *)actl,
                  (void *)outv, (void *)ctl, (void *)Zd, (void *)S_owned})
    if (q) cudaFreeAsync(q, st);
  for (cudaEvent_t e : {e0, e1, es0, es1}) cudaEventDestroy(e);
  FJ_CUDA(cudaGetLastError());
  fj_status rc = finish_status(hs, stats, o, omega);
  if (st_out) *st_out = stats;
  return rc;
}

fj_status solve_impl(fj_graph *g, const float *s_in, double eps, double omega, const fj_opts *o,
                     float *z_out, fj_stats *st_out) {
  NvtxRange nv("fj_solve");
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  fj_stats stats{};
  int method = o->method;
  // AUTO: BLI (ω = 1) runs asynchronous sweeps, provably convergent for the
  // M-matrix I + L in any order.  BLISOR (ω ≠ 1) on an undirected graph runs
  // multicolor sweeps (sequential SOR on an SPD matrix converges for every
  // ω ∈ (0,2)); on a directed graph, where no ordering carries a
  // guarantee, asynchronous sweeps (the certificate and the divergence
  // sentinel still decide the outcome).
  if (method == FJ_METHOD_AUTO)
    method = (omega == 1.0 || g->directed) ? FJ_METHOD_ASYNC : FJ_METHOD_COLORED;
  if (method == FJ_METHOD_COLORED && !g->colors) FJ_TRY(build_coloring(g));
  if (method == FJ_METHOD_PUSH) {
    if (o->z_init) {
      set_error("fj_solve: z_init (warm start) is supported by ASYNC/COLORED, not PUSH");
      return FJ_ERR_INVALID;
    }
    return push_solve_impl(g, s_in, eps, omega, o, z_out, st_out);
  }
  const Layout &L = (method == FJ_METHOD_COLORED) ? g->color_layout : g->async_layout;
  const bool W = g->weighted != 0;

  cudaEvent_t e0, e1, es0, es1, ec0, ec1;
  FJ_CUDA(cudaEventCreate(&e0));
  FJ_CUDA(cudaEventCreate(&e1));
  FJ_CUDA(cudaEventCreate(&es0));
  FJ_CUDA(cudaEventCreate(&es1));
  FJ_CUDA(cudaEventCreate(&ec0));
  FJ_CUDA(cudaEventCreate(&ec1));
  FJ_CUDA(cudaEventRecord(e0, st));

  Staged s{};
  FJ_TRY(stage_in(s_in, n, st, s));
  const bool zdev = is_device_ptr(z_out);
  const bool zpdev = o->zprime_out && is_device_ptr(o->zprime_out);

  // workspace (stream-ordered pool allocations)
  float *s_l = nullptr, *smin = nullptr, *smax = nullptr, *zo = nullptr;
  double *z = nullptr, *zp = nullptr;
  double2 *partial = nullptr;
  int *arrive = nullptr;
  Scalars *S = nullptr;
  unsigned *ctl = nullptr;  // ctr[3] + bar[2]
  SweepCounters *cnt = nullptr;
  unsigned long long *outv = nullptr, *certbits = nullptr;
  FJ_CUDA(cudaMallocAsync(&s_l, sizeof(float) * n, st));
  FJ_CUDA(cudaMallocAsync(&z, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&smin, sizeof(float) * 2, st));
  smax = smin + 1;
  FJ_CUDA(cudaMallocAsync(&S, sizeof(Scalars), st));
  FJ_CUDA(cudaMallocAsync(&partial, sizeof(double2) * std::max(1, L.npartials), st));
  FJ_CUDA(cudaMallocAsync(&arrive, sizeof(int) * std::max(1, L.npartials), st));
  FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
  FJ_CUDA(cudaMallocAsync(&ctl, sizeof(unsigned) * kCtlWords, st));
  FJ_CUDA(cudaMallocAsync(&cnt, sizeof(SweepCounters) * 3, st));
  FJ_CUDA(cudaMallocAsync(&outv, sizeof(unsigned long long) * 8, st));
  certbits = outv + 4;
  if (!zdev) FJ_CUDA(cudaMallocAsync(&zo, sizeof(float) * n, st));
  if (o->zprime_out && !zpdev) FJ_CUDA(cudaMallocAsync(&zp, sizeof(double) * n, st));

  // a2: shift and init (Alg. 2)
  {
    size_t tmp = 0;
    FJ_CUDA(cub::DeviceReduce::Min(nullptr, tmp, s.dev, smin, n, st));
    size_t tmp2 = 0;
    FJ_CUDA(cub::DeviceReduce::Max(nullptr, tmp2, s.dev, smax, n, st));
    tmp = std::max(tmp, tmp2);
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, tmp, st));
    FJ_CUDA(cub::DeviceReduce::Min(t, tmp, s.dev, smin, n, st));
    FJ_CUDA(cub::DeviceReduce::Max(t, tmp, s.dev, smax, n, st));
    FJ_CUDA(cudaFreeAsync(t, st));
  }
  fj::count_launch();
  k_scalars<<<1, 1, 0, st>>>(smin, smax, eps, o->sigma, o->c, S);
  const double *zinit = nullptr;
  double *zinit_owned = nullptr;
  if (o->z_init) {
    if (is_device_ptr(o->z_init)) {
      zinit = o->z_init;
    } else {
      FJ_CUDA(cudaMallocAsync(&zinit_owned, sizeof(double) * n, st));
      FJ_CUDA(cudaMemcpyAsync(zinit_owned, o->z_init, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      zinit = zinit_owned;
    }
  }
  fj::count_launch();
  k_init<<<gridn(n), kBlock, 0, st>>>(n, L.perm, L.rp, s.dev, S, s_l, z, zinit);
  if (zinit_owned) FJ_CUDA(cudaFreeAsync(zinit_owned, st));

  KP p = make_kp(g, L);
  p.s = s_l;
  p.z = z;
  p.sc = S;
  p.omega = omega;
  p.theta = 1.0;
  p.dbg = getenv("FJ_DBG_SKIP") ? atoi(getenv("FJ_DBG_SKIP")) : 0;
  p.dyn = getenv("FJ_DYN") ? atoi(getenv("FJ_DYN")) : 0;
  p.symm = getenv("FJ_SYMM") ? atoi(getenv("FJ_SYMM")) : 0;
  p.partial = partial;
  p.arrive = arrive;
  p.max_sweeps = o->max_sweeps;
  p.ctr = ctl;
  p.bar = ctl + 8;
  p.cnt = cnt;
  p.out = outv;
  p.cert_max = certbits;

  // TMA-streamed chunks pay off when the arc stream dominates (short rows,
  // local gathers: lattice, ER); hub-dominated graphs keep the shared memory
  // as L1 for their gathers and load the stream directly
  const bool tma = getenv("FJ_TMA") ? atoi(getenv("FJ_TMA")) != 0 : L.stream_tma;
  const void *fn = W ? (tma ? (const void *)k_sweep<true, true> : (const void *)k_sweep<true, false>)
                     : (tma ? (const void *)k_sweep<false, true> : (const void *)k_sweep<false, false>);
  const size_t sweep_smem =
      tma ? (kBlock / 32) * sizeof(WarpSmem) : (kBlock / 32) * kWarpTileArcs * sizeof(double);
  FJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem));
  if (getenv("FJ_CARVEOUT"))  // shared-memory carveout in percent (diagnostics)
    FJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 atoi(getenv("FJ_CARVEOUT"))));
  const int grid = persistent_grid(fn, g->num_sms, sweep_smem);
  float ms_sweep = 0, ms_cert = 0;
  int rounds = 0;
  stats.colors = L.ncolors;
  // one-phase ASYNC runs barrier-free (k_sweep_async) unless FJ_BARRIER=1
  // the barrier-free kernel is opt-in (FJ_ASYNC_FREE=1): measured slower on
  // C4/C5, where overlapping sweeps lose some Gauss–Seidel ordering
  const bool barrier_free = L.ncolors == 1 && !tma && getenv("FJ_ASYNC_FREE") &&
                            atoi(getenv("FJ_ASYNC_FREE"));
  const void *fa = W ? (const void *)k_sweep_async<true> : (const void *)k_sweep_async<false>;
  const size_t async_smem = (kBlock / 32) * kWarpTileArcs * sizeof(double);
  AsyncCtl *actl = nullptr;
  if (barrier_free) {
    FJ_CUDA(cudaFuncSetAttribute(fa, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)async_smem));
    FJ_CUDA(cudaMallocAsync(&actl, sizeof(AsyncCtl), st));
  }
  const int agrid = barrier_free ? persistent_grid(fa, g->num_sms, async_smem) : 0;
  for (;;) {
    // a3–a5: persistent sweeps with on-device loop control
    FJ_CUDA(cudaMemsetAsync(ctl, 0, sizeof(unsigned) * kCtlWords, st));
    FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(SweepCounters) * 3, st));
    FJ_CUDA(cudaMemsetAsync(outv, 0, sizeof(unsigned long long) * 8, st));
    FJ_CUDA(cudaEventRecord(es0, st));
    if (barrier_free) {
      FJ_CUDA(cudaMemsetAsync(actl, 0, sizeof(AsyncCtl), st));
      void *args[] = {&p, &actl};
      fj::count_launch();
      FJ_CUDA(cudaLaunchKernel(fa, agrid, kBlock, args, async_smem, st));
      fj::count_launch();
      k_async_result<<<1, 1, 0, st>>>(actl, outv, (unsigned long long)p.max_sweeps);
    } else {
      void *args[] = {&p};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, sweep_smem, st));
    }
    FJ_CUDA(cudaEventRecord(es1, st));
    // fp64 compensated certificate over every non-empty row
    if (o->certify) {
      KP q = p;
      q.ctr = ctl + 5;
      FJ_CUDA(cudaEventRecord(ec0, st));
      const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
      void *cargs[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchKernel(cf, persistent_grid(cf, g->num_sms), kBlock, cargs, 0, st));
      FJ_CUDA(cudaEventRecord(ec1, st));
    }
    unsigned long long h[8];
    FJ_CUDA(cudaMemcpyAsync(h, outv, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    float a = 0;
    FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
    ms_sweep += a;
    if (o->certify) {
      FJ_CUDA(cudaEventElapsedTime(&a, ec0, ec1));
      ms_cert += a;
    }
    stats.sweeps += (int64_t)h[0];
    stats.relaxations += (int64_t)h[1];
    stats.edge_updates += (int64_t)h[2];
    stats.reason = (int)h[3];
    stats.cert_ratio = o->certify ? __builtin_bit_cast(double, h[4]) : 0.0;
    if (stats.reason != 0) break;
    if (!o->certify || stats.cert_ratio <= 1.0 || rounds >= o->cert_rounds) break;
    rounds++;  // resume from ẑ (Lemma 3: ẑ fully determines r)
    p.max_sweeps = std::min(o->max_sweeps, 2000);  // a resume starts next to the fixed point
    // the sweep's plain fp64 residual agreed with h where the compensated
    // one did not: resume with a stricter sweep threshold so that every row
    // the certificate rejects is relaxed again
    p.theta *= 0.5;
  }
  if (actl) cudaFreeAsync(actl, st);
  stats.cert_rounds = rounds;
  stats.phases = stats.sweeps * L.ncolors;
  stats.rows_read = stats.sweeps * L.active_rows;
  stats.arcs_read = stats.sweeps * L.m;
  stats.relaxations += L.empty_rows;  // rows solved exactly at init

  // a6: unshift
  fj::count_launch();
  k_finalize<<<gridn(n), kBlock, 0, st>>>(n, L.iperm, z, S, zdev ? z_out : zo,
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
  stats.cert_ms = ms_cert;
  stats.c = hs.c;
  stats.eps_prime = hs.eps_p;

  cudaFreeAsync(s_l, st);
  cudaFreeAsync(z, st);
  cudaFreeAsync(smin, st);
  cudaFreeAsync(S, st);
  cudaFreeAsync(partial, st);
  cudaFreeAsync(arrive, st);
  cudaFreeAsync(ctl, st);
  cudaFreeAsync(cnt, st);
  cudaFreeAsync(outv, st);
  if (zo) cudaFreeAsync(zo, st);
  if (zp) cudaFreeAsync(zp, st);
  if (s.owned) cudaFreeAsync(s.owned, st);
  for (cudaEvent_t e : {e0, e1, es0, es1, ec0, ec1}) cudaEventDestroy(e);
  FJ_CUDA(cudaGetLastError());

  fj_status rc = finish_status(hs, stats, o, omega);
  if (st_out) *st_out = stats;
  return rc;
}

fj_status measures_impl(fj_graph *g, const float *z_in, const float *s_in, fj_measures_t *out) {
  NvtxRange nv("fj_measures");
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  const Layout &L = g->async_layout;
  Staged z{}, s{};
  FJ_TRY(stage_in(z_in, n, st, z));
  if (s_in) FJ_TRY(stage_in(s_in, n, st, s));
  double *zl = nullptr, *sums = nullptr;
  unsigned *ctr = nullptr;
  FJ_CUDA(cudaMallocAsync(&zl, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&sums, sizeof(double) * 5, st));
  FJ_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * 5, st));
  FJ_CUDA(cudaMallocAsync(&ctr, sizeof(unsigned), st));
  FJ_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned), st));
  fj::count_launch();
  k_meas_nodes1<<<gridn(n), kBlock, 0, st>>>(n, L.perm, z.dev, zl, sums);
  fj::count_launch();
  k_meas_nodes2<<<gridn(n), kBlock, 0, st>>>(n, z.dev, s.dev, sums);
  KP p = make_kp(g, L);
  p.z = zl;
  p.ctr = ctr;
  p.dis = sums + 4;
  const bool W = g->weighted != 0;
  const void *fn = W ? (const void *)k_pass<DIS, true> : (const void *)k_pass<DIS, false>;
  void *args[] = {&p};
  fj::count_launch();
  FJ_CUDA(cudaLaunchKernel(fn, persistent_grid(fn, g->num_sms), kBlock, args, 0, st));
  double h[5];
  FJ_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  cudaFreeAsync(zl, st);
  cudaFreeAsync(sums, st);
  cudaFreeAsync(ctr, st);
  if (z.owned) cudaFreeAsync(z.owned, st);
  if (s.owned) cudaFreeAsync(s.owned, st);
  FJ_CUDA(cudaGetLastError());
  out->polarization = h[1];
  // each undirected edge is stored as two arcs (reading R14)
  out->disagreement = g->directed ? h[4] : 0.5 * h[4];
  out->internal_conflict = s_in ? h[2] : 0.0;
  out->controversy = h[3];
  return FJ_OK;
}


// ------------------------------------------------------------- ω selection
// y_i ← ((J x)_i + x_i)/2 with J = (I+D)^{-1} A; Σ y², Σ x·y
__global__ void k_jacobi_scale(int64_t n, const int64_t *__restrict__ rp, const double *__restrict__ d1,
                               const double *__restrict__ x, double *__restrict__ y,
                               double *__restrict__ sums) {
  __shared__ double sm[kBlock / 32];
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double yy = 0.0, xy = 0.0;
  if (i < n) {
    const double dv = d1 ? d1[i] : (double)(rp[i + 1] - rp[i] + 1);
    const double v = 0.5 * (y[i] / dv + x[i]);  // (J + I)/2: Perron root strictly dominant
    y[i] = v;
    yy = v * v;
    xy = x[i] * v;
  }
  yy = block_reduce<double>(yy, sm);
  xy = block_reduce<double>(xy, sm);
  if (threadIdx.x == 0) {
    atomicAdd(sums, yy);
    atomicAdd(sums + 1, xy);
  }
}
__global__ void k_scale_copy(int64_t n, double f, const double *__restrict__ y, double *__restrict__ x) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = y[i] * f;
}
__global__ void k_fill(int64_t n, double v, double *__restrict__ x) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = v;
}

// μ = ρ((I+D)^{-1} A) by power iteration on (J+I)/2 from x = 1 (J ≥ 0, so ρ
// is its Perron root; the shift keeps it strictly dominant even for
// bipartite graphs where −μ is also an eigenvalue), then ω_opt = 1 + (μ/(1+√(1−μ²)))² (Eq. optimal-omega).
fj_status omega_opt_impl(fj_graph *g, int max_iters, double tol, double *mu_out,
                         double *omega_out, int *iters_out) {
  cudaStream_t st = g->stream;
  const Layout &L = g->async_layout;
  const int64_t n = g->n;
  double *x = nullptr, *y = nullptr, *sums = nullptr, *partial = nullptr;
  unsigned *ctr = nullptr;
  FJ_CUDA(cudaMallocAsync(&x, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&y, sizeof(double) * n, st));
  FJ_CUDA(cudaMallocAsync(&sums, sizeof(double) * 2, st));
  FJ_CUDA(cudaMallocAsync(&ctr, sizeof(unsigned), st));
  fj::count_launch();
  k_fill<<<gridn(n), kBlock, 0, st>>>(n, 1.0 / sqrt((double)n), x);
  KP p = make_kp(g, L);
  p.ctr = ctr;
  const bool W = g->weighted != 0;
  const void *fn = W ? (const void *)k_pass<SPMV, true> : (const void *)k_pass<SPMV, false>;
  const int grid = persistent_grid(fn, g->num_sms);
  double mu = 0.0, prev = -1.0;
  int it = 0;
  for (; it < max_iters; it++) {
    FJ_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * n, st));
    FJ_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * 2, st));
    p.z = x;
    p.rout = y;
    void *args[] = {&p};
    fj::count_launch();
    FJ_CUDA(cudaLaunchKernel(fn, grid, kBlock, args, 0, st));
    fj::count_launch();
    k_jacobi_scale<<<gridn(n), kBlock, 0, st>>>(n, L.rp, L.d1, x, y, sums);
    double h[2];
    FJ_CUDA(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    const double ny = sqrt(h[0]);
    mu = 2.0 * ny - 1.0;  // ||(J+I)x/2|| → (μ+1)/2 with ||x|| = 1
    if (ny == 0.0) break;
    fj::count_launch();
    k_scale_copy<<<gridn(n), kBlock, 0, st>>>(n, 1.0 / ny, y, x);
    if (fabs(mu - prev) <= tol * mu) break;
    prev = mu;
  }
  cudaFreeAsync(x, st);
  cudaFreeAsync(y, st);
  cudaFreeAsync(sums, st);
  cudaFreeAsync(ctr, st);
  (void)partial;
  FJ_CUDA(cudaStreamSynchronize(st));
  if (mu > 1.0) mu = 1.0;
  *mu_out = mu;
  const double r = mu / (1.0 + sqrt(fmax(0.0, 1.0 - mu * mu)));
  *omega_out = 1.0 + r * r;
  if (iters_out) *iters_out = it + 1;
  return FJ_OK;
}
}  // namespace fj

extern "C" {

fj_status fj_solve_ex(fj_graph_t g, const float *s, double eps, double omega, const fj_opts *o,
                      float *z_out, fj_stats *st) {
  fj_opts d;
  fj_opts_default(&d);
  if (o) {
    d = *o;
    if (!(d.sigma > 0)) d.sigma = 1e-5;
    if (d.max_sweeps <= 0) d.max_sweeps = 1000000;
    if (d.cert_rounds < 0) d.cert_rounds = 3;
  }
  if (!g || !s || !z_out) {
    fj::set_error("fj_solve: null argument");
    return FJ_ERR_INVALID;
  }
  if (!(eps > 0.0 && eps < 1.0)) {
    fj::set_error("fj_solve: eps must lie in (0, 1), got %g", eps);
    return FJ_ERR_INVALID;
  }
  if (!(omega > 0.0 && omega < 2.0)) {
    fj::set_error("fj_solve: omega must lie in (0, 2), got %g", omega);
    return FJ_ERR_INVALID;
  }
  if (d.method < FJ_METHOD_AUTO || d.method > FJ_METHOD_PUSH) {
    fj::set_error("fj_solve: unknown method %d", d.method);
    return FJ_ERR_INVALID;
  }
  return fj::solve_impl(g, s, eps, omega, &d, z_out, st);
}

fj_status fj_omega_opt(fj_graph_t g, int max_iters, double tol, double *mu, double *omega) {
  if (!g || !mu || !omega || max_iters < 1 || !(tol > 0)) {
    fj::set_error("fj_omega_opt: bad argument");
    return FJ_ERR_INVALID;
  }
  return fj::omega_opt_impl(g, max_iters, tol, mu, omega, nullptr);
}

fj_status fj_omega_sweep(fj_graph_t g, const float *s, double eps, double lo, double hi, double step,
                         int method, double *best_omega, double *table, int *npts) {
  if (!g || !s || !best_omega || !npts || !(step > 0) || !(lo > 0) || !(hi < 2) || hi < lo) {
    fj::set_error("fj_omega_sweep: bad argument");
    return FJ_ERR_INVALID;
  }
  const int cap = *npts;
  int k = 0;
  double best = 1.0;
  int64_t best_cost = -1;
  float *z = nullptr;
  FJ_CUDA(cudaMallocAsync(&z, sizeof(float) * g->n, g->stream));
  fj_opts o;
  fj_opts_default(&o);
  o.method = method;
  // the paper's heuristic: start near 2, lower ω by a fixed step to 1,
  // keep the ω with the fewest updates; diverging ω cost +inf
  for (int i = 0;; i++) {
    const double om = hi - i * step;
    if (om < lo - 1e-12) break;
    fj_stats st;
    fj_status rc = fj_solve_ex(g, s, eps, om, &o, z, &st);
    if (rc != FJ_OK && rc != FJ_ERR_NUMERIC) {
      cudaFreeAsync(z, g->stream);
      return rc;
    }
    if (table && k < cap) {
      table[3 * k] = om;
      table[3 * k + 1] = (double)st.relaxations;
      table[3 * k + 2] = (double)rc;
    }
    k++;
    if (rc == FJ_OK && (best_cost < 0 || st.relaxations <= best_cost)) {
      best_cost = st.relaxations;  // ties go to the smaller ω
      best = om;
    }
  }
  cudaFreeAsync(z, g->stream);
  cudaStreamSynchronize(g->stream);
  *npts = k;
  *best_omega = best;
  if (best_cost < 0) {
    fj::set_error("fj_omega_sweep: no ω in the grid converged");
    return FJ_ERR_NUMERIC;
  }
  return FJ_OK;
}

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
  if (!g || !S || !Z_out || k < 1 || k > 4) {
    fj::set_error("fj_solve_batch: need non-null arguments and 1 <= k <= 4");
    return FJ_ERR_INVALID;
  }
  if (!(eps > 0.0 && eps < 1.0) || !(omega > 0.0 && omega < 2.0)) {
    fj::set_error("fj_solve_batch: eps in (0,1) and omega in (0,2) required");
    return FJ_ERR_INVALID;
  }
  if (d.method != FJ_METHOD_AUTO && d.method != FJ_METHOD_ASYNC) {
    fj::set_error("fj_solve_batch: only the ASYNC schedule is batched");
    return FJ_ERR_INVALID;
  }
  return fj::batch_solve_impl(g, S, k, eps, omega, &d, Z_out, st);
}

fj_status fj_solve(fj_graph_t g, const float *s, double eps, double omega, float *z_out) {
  return fj_solve_ex(g, s, eps, omega, nullptr, z_out, nullptr);
}

fj_status fj_measures_ex(fj_graph_t g, const float *z, const float *s, fj_measures_t *out) {
  if (!g || !z || !out) {
    fj::set_error("fj_measures: null argument");
    return FJ_ERR_INVALID;
  }
  return fj::measures_impl(g, z, s, out);
}

fj_status fj_measures(fj_graph_t g, const float *z, double *polarization, double *disagreement) {
  if (!polarization || !disagreement) {
    fj::set_error("fj_measures: null output");
    return FJ_ERR_INVALID;
  }
  fj_measures_t m;
  fj_status s = fj_measures_ex(g, z, nullptr, &m);
  if (s != FJ_OK) return s;
  *polarization = m.polarization;
  *disagreement = m.disagreement;
  return FJ_OK;
}

}  // extern "C"
