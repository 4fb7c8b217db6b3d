// sweep_common.cuh — device building blocks shared by the sweep, push and
// batch translation units (internal; not part of the ABI).  See solve.cu for
// the method notes (Theorem 3 sweep form of the paper's push).
#pragma once
#include <stdlib.h>

#include <algorithm>
#include <cuda/atomic>
#include <nvtx3/nvToolsExt.h>
#include <type_traits>

#include "fj_internal.cuh"

// -DFJ_BOUNDS: diagnostic build with device-side bounds checks (compute-sanitizer is not
// available on the GPU pool): a failed check traps the kernel and the call returns
// FJ_ERR_CUDA.  Used by tools/bounds_check.sh over the tiny GPU tests.
#ifdef FJ_BOUNDS
#define FJ_CHECK(cond) do { if (!(cond)) { printf("FJ_BOUNDS %s:%d: %s\n", __FILE__, __LINE__, #cond); __trap(); } } while (0)
#else
#define FJ_CHECK(cond) do { } while (0)
#endif

namespace fj {

struct NvtxRange {  // tracing: one NVTX range per library phase (nsys/ncu timelines)
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

enum Mode { RELAX = 0, CERT = 1, DIS = 2, SPMV = 3 };
#ifndef FJ_THIN_DIV
#define FJ_THIN_DIV 256  // default thin-sweep threshold: non-empty rows / 256
#endif
#ifndef FJ_DEPCHUNK
#define FJ_DEPCHUNK 256  // (1024: 2–6 % slower, the scatter of a hub's entry is one long chain)
#endif
constexpr int kDepChunk = FJ_DEPCHUNK;  // frontier phase: dependents of a relaxed row per list entry
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
  // shadow ẑ (k_sweep_sh): fixed point on [0, 2^e), 2^e ≥ max s' (twice that when ω > 1 or
  // warm-started): decode fma(2^52 + u, sh_scale, sh_off) = u·2^(e−32); encode ẑ'·sh_enc
  double sh_scale, sh_off, sh_enc;
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
  // row slices (k_sweep / k_sweep_sh with SL): the layout's slice sweep list and slots
  const Task *__restrict__ stasks;
  const int *sphase_begin;
  const int32_t *__restrict__ scol;
  const float *__restrict__ sw;
#ifdef FJ_BOUNDS
  int64_t nslots;
#endif
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
  int kreal;                // batched solves: right-hand sides that count (the rest is padding)
  int tail_pct;             // k_sweep: percent of each phase's items claimed dynamically at its end
  const double *omegas;     // ω batch (fj_solve_batch_omega): ω per column [K]; else null
  int *colbad;              // ω batch: per-column divergence flags [K]; null otherwise
  unsigned long long *colupd;  // ω batch: per-column relaxations [K]
  int tail_phase;           // merged tail colors (reading R23); −1 if none
  int64_t tail_row0, tail_row1;  // rows of the tail phase (empty range if none)
  const float *tail_beta;   // per tail row: β_i (see color.cu)
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
  const unsigned long long *stop;  // sharded solve: nonzero = the loop has ended (k_sweep)
  int64_t empty0, empty1;  // rows with no arcs (the layout's last group): CERT covers them too
  // shadow sweeps (k_sweep_sh, solve.cu): 32-bit fixed-point copy of ẑ' for the gathers
  unsigned *zs;            // [n] layout order: u = round(ẑ'·S.sh_enc), ẑ' ≈ u·S.sh_scale
  const unsigned long long *prev;  // out[] of the launch before this one (fp64 tail after shadow)
  int skip_if_done;        // k_sweep: return at once if the launch before converged (prev[3] == 0)
  // frontier phase (k_front, solve.cu): thin = a sweep that relaxes fewer rows (but some)
  // ends the sweep loop with reason 3; the residuals, lists and maps of the phase
  unsigned long long thin;
  double *fr_r;            // [n] residuals r = s' − (I+L)ẑ', layout order (k_pass<CERT> writes them)
  int *fr_rows;            // [2][fr_cap] rows to pop this / next round
  int4 *fr_push;           // [fr_pcap] (row, chunk of its dependents, Δẑ bits) to scatter
  unsigned *fr_cnt;        // [0,1] row-list counts, [2,3] scatter entries of an even / odd round
  int fr_cap, fr_pcap;
  const int64_t *in_rp;    // canonical in-CSR, original ids: row u lists the rows that gather u
  const int32_t *in_col;
  const float *in_w;       // their weights a (null: 1)
  const int32_t *perm, *iperm;
  int fr_max_rounds;
};

// CSR streams are read once per sweep: read-only path, no L1 allocation, so
// L1 keeps the gathered ẑ values (hub rows are hit by many arcs).  The asm is
// not volatile (so the compiler may batch these loads) — which also lets it
// speculate them: never guard a call with a condition (`ok ? ld_stream(q) :
// 0`), clamp the address to a valid slot instead.
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
__device__ __forceinline__ unsigned ld_zs(const unsigned *q) { return *q; }

// Shadow ẑ (k_sweep_sh): the gathers read a 32-bit fixed-point copy of ẑ'
// (4 B per gather, the whole copy resident in L2; SURVEY §8(d) "fp32 shadow",
// fixed point because ẑ' is bounded: its error is uniform, ≤ 2^-33·range).
// decode: u·scale, exact, as one FMA on the double 2^52 + u (no I2F).
__device__ __forceinline__ double sh_dec(unsigned u, double scale, double off) {
  return fma(__hiloint2double(0x43300000, (int)u), scale, off);
}

// Hub-row pieces (see do_warp): a piece's partial sum is stored, then its
// arrival is counted with release semantics (MEMBAR.ALL.GPU orders the store
// before the atomic; unlike __threadfence / acquire operations it emits no
// CCTL.IVALL, so L1 keeps its cached ẑ lines).  The last-arriving warp reads
// the partials with gpu-scope strong loads, which are served by L2 — the point
// of coherence the releasing stores have reached — never by a stale L1 line.
__device__ __forceinline__ int arrive_release(int *q) {
#ifdef FJ_OLD_FENCE
  __threadfence();
  const int old = atomicAdd(q, 1);
  __threadfence();
  return old;
#else
  int old;
  asm volatile("atom.add.release.gpu.s32 %0, [%1], 1;" : "=r"(old) : "l"(q) : "memory");
  return old;
#endif
}
__device__ __forceinline__ double2 ld_partial(const double2 *q) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(q)
               : "memory");
  return v;
}

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

// relax one row from its residual; row state loaded by the caller (prefetched)
// 1/x to ≈ 4e-15 relative (single-precision reciprocal + one Newton step): the size of a
// relaxation step need not be exactly rounded (Lemma 3: any amount is a valid state)
__device__ __forceinline__ double rcp_newton(double x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"((float)x));
  const double y = (double)r;
  return y * fma(-x, y, 2.0);
}

template <int SH = 0>
__device__ __forceinline__ void relax_row_pre(const KP &p, const Scalars &S, int row, int len,
                                              dd total, float sv, double zi, double d1, TAcc &t) {
  const double sp = (double)sv + S.c;
  const double h = threshold(S, sp);
  // shadow sweeps: plain fp64 combination (the shadow's rounding is far above its error)
  const double rho = SH == 1 ? fma(-d1, zi, sp + total.hi) : residual_dd(total, sp, d1, zi);
  const double ar = fabs(rho);
  if (ar > p.theta * h) {
    // tail phase (R23): ω_i = min(ω, 1.98/(1+β_i)) keeps |1−ω_i| + ω_i β_i < 1
    double om = p.omega;
    if (p.tail_phase >= 0 && row >= p.tail_row0 && row < p.tail_row1)
      om = fmin(om, 1.98 / (1.0 + (double)p.tail_beta[row - p.tail_row0]));
    // (the fp64 kernel keeps the division: the reciprocal form costs it registers — spills)
    const double dz = SH == 1 ? om * rho * rcp_newton(d1) : om * rho / d1;
    const double zn = zi + dz;
    __stcg(p.z + row, zn);
    if constexpr (SH == 1) {
      // outside the shadow's range [0, 2^e): the shadow loop ends and the fp64 sweeps
      // carry on from ẑ (Lemma 3: any ẑ is a valid state)
      const double ze = zn * S.sh_enc;
      if (!(ze >= 0.0 && ze <= 4294967295.0)) t.bad |= 1;
      // bit 1: this sweep still moved some ẑ' by ≥ 4 shadow quanta.  The shadow's own
      // rounding can move a row by < ω quanta at most (Σ_j a_ij·½ quantum·ω/(1+d_i)), so
      // a sweep without such a move is relaxing rounding noise (at ω ≠ 1 that noise need
      // not die out): the shadow loop ends and the fp64 sweeps take over
      if (fabs(dz) * S.sh_enc >= 4.0) t.bad |= 2;
      const unsigned u = __double2uint_rn(ze);
      __stcg(p.zs + row, u);
    }
    t.upd++;
    t.eu += (unsigned long long)len;
  }
  if (!(ar <= S.sentinel)) t.bad |= 1;
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
      static_assert(MODE != RELAX, "RELAX runs as warp tiles / warp units");
      if constexpr (MODE == CERT) cert_row<W>(p, S, row, len, a, t);
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
// kWarpPiece-arc piece of it in registers — U = 4 independent col/w loads, then
// 4 ẑ gathers per lane per step (U = 4 measured best with the warp tiles in the
// same kernel: C3 −5 %, C5 −7 %, C4 −1 % per sweep against U = 8) — and reduces
// with shuffles (no block barrier).
// Pieces of one row are combined by the last-arriving warp in piece order
// (deterministic).
// SH (RELAX only): 0 = fp64 ẑ gathers; 1 = shadow gathers (sh_dec of p.zs).
// Shadow sums are plain fp64: the shadow's own rounding (2^-33·range per value) is far
// above what double-double would recover; the fp64 tail sweeps and the certificate follow.
template <int MODE, bool W, int SH = 0>
__device__ __forceinline__ void do_warp(const KP &p, const Scalars &S, const Task &tk, TAcc &t) {
  static_assert(SH != 1 || MODE == RELAX, "shadow gathers are a RELAX path");
  // rows above 256 arcs accumulate in double-double for RELAX and CERT
  using A = typename std::conditional<MODE == DIS || MODE == SPMV || SH == 1, double, dd>::type;
#ifndef FJ_WU
#define FJ_WU 4
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
    if constexpr (SH != 1) {
#pragma unroll
      for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
    } else {
      unsigned zu[U];
#pragma unroll
      for (int u = 0; u < U; u++) zu[u] = ld_zs(p.zs + j[u]);
#pragma unroll
      for (int u = 0; u < U; u++) zj[u] = sh_dec(zu[u], S.sh_scale, S.sh_off);
    }
    // stage 3: accumulate
#pragma unroll
    for (int u = 0; u < U; u++) {
      if constexpr (SH == 1) {
        a = fma((double)wv[u], zj[u], a);
      } else if constexpr (MODE == SPMV) {
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
    dd ad;
    if constexpr (SH == 1) ad = dd{a, 0.0};
    else ad = a;
    if (np > 1) {
      __stcg(p.partial + slot + piece, make_double2(ad.hi, ad.lo));
      // cumulative arrival count: the np-th, 2np-th, ... arrival finishes the
      // row (no reset, so overlapping sweeps of the barrier-free kernel can
      // never lose an arrival; mixing partials of two sweeps is still a
      // valid relaxation amount by Lemma 3 and the certificate decides).
      // Release arrival + L2 (gpu-scope) reads of the partials: no
      // __threadfence, whose CCTL.IVALL would wipe this SM's L1 — the home of
      // the hub ẑ gathers — once per hub piece.
      const int old = arrive_release(p.arrive + slot);
      if ((old + 1) % np != 0) return;
      acc_zero(ad);
      for (int q = 0; q < np; q++) {  // fixed order ⇒ deterministic row sum
        const double2 x = ld_partial(p.partial + slot + q);
        acc_merge(ad, dd{x.x, x.y});
      }
    }
    if constexpr (MODE == RELAX) {
      // a non-final piece returned above; a multi-piece row is finished by
      // the last-arriving warp, whose prefetched ẑ_row is still current (only
      // this row's finisher writes it, once per phase)
      relax_row_pre<SH>(p, S, row, len, ad, sv, zi, d1, t);
    } else {
      const int lenc = (int)(__ldg(p.rp + row + 1) - __ldg(p.rp + row));
      cert_row<W>(p, S, row, lenc, ad, t);
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
template <bool W, int SH = 0>
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
  if constexpr (SH != 1) {
#pragma unroll
    for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
  } else {
    unsigned zu[U];
#pragma unroll
    for (int u = 0; u < U; u++) zu[u] = ld_zs(p.zs + j[u]);
#pragma unroll
    for (int u = 0; u < U; u++) zj[u] = sh_dec(zu[u], S.sh_scale, S.sh_off);
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    const int e = u * 32 + lane;
    if (e < na) wprod[e] = (double)wv[u] * zj[u];
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 2; q++) {
    if (SH == 1 && q == 1 && tk.a + ng >= tk.b) break;  // no rows left for the second step (uniform)
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
      relax_row_pre<SH>(p, S, row, len, dd{a, 0.0}, sv[q], zi[q],
                        W ? d1[q] : (double)(len + 1), t);
    }
  }
  __syncwarp();  // the slice is reused by this warp's next task
}

// RELAX on a row slice (sliced ELL, Layout::scol / sw): ≤ 32 short rows, one lane per
// row.  Slot 32 t + lane holds arc t of the lane's row, so every column / weight load of
// the warp is one 128-byte line, each lane sums its own row in a register (no staging, no
// shuffles, no shared memory) and all 32 lanes relax at once.  Rows of a slice have the
// same length but at class boundaries (the layout sorts short rows by length); shorter
// rows are padded with (column n, weight 0): ẑ'[n] = 0 and its shadow sit after the last
// row.  Up to 8 column loads, then 8 gathers, per lane in flight (4 and 2 measured slower).
// (G lanes per row with a shuffle sum — shorter items, more of them — measured slower:
// C4 1.11 vs 0.99 ms per sweep, profiles/r02_slices_ab.txt.)
template <bool W, int SH, int U>
__device__ __forceinline__ void slice_step(const KP &p, const Scalars &S, const int32_t *cp,
                                           const float *wp, double &a) {
  int j[U];
  float wv[U];
#pragma unroll
  for (int u = 0; u < U; u++) {
    FJ_CHECK(cp + 32 * u >= p.scol && cp + 32 * u < p.scol + p.nslots);
    j[u] = ld_stream(cp + 32 * u);
    wv[u] = W ? ld_stream(wp + 32 * u) : 1.0f;
    FJ_CHECK(j[u] >= 0 && j[u] <= p.empty1);  // a row, or the padding column n
  }
  double zj[U];
  if constexpr (SH != 1) {
#pragma unroll
    for (int u = 0; u < U; u++) zj[u] = ld_z(p.z + j[u]);
  } else {
    unsigned zu[U];
#pragma unroll
    for (int u = 0; u < U; u++) zu[u] = ld_zs(p.zs + j[u]);
#pragma unroll
    for (int u = 0; u < U; u++) zj[u] = sh_dec(zu[u], S.sh_scale, S.sh_off);
  }
#pragma unroll
  for (int u = 0; u < U; u++) {
    if (W) a = fma((double)wv[u], zj[u], a);
    else a += zj[u];
  }
}

template <bool W, int SH = 0>
__device__ __forceinline__ void relax_slice(const KP &p, const Scalars &S, const Task &tk, TAcc &t) {
  const int lane = threadIdx.x & 31;
  const int row = tk.a + lane;
  const bool ok = row < tk.b;
  int wd = tk.slot;
  FJ_CHECK(tk.a >= 0 && tk.b <= p.empty0 && tk.b - tk.a <= 32 && tk.a1 - tk.a0 == 32 * (int64_t)wd);
  const int32_t *cp = p.scol + tk.a0 + lane;
  const float *wp = W ? p.sw + tk.a0 + lane : nullptr;
  float sv = 0.f;
  double zi = 0.0, d1 = 1.0;
  int len = 0;
  if (ok) {
    sv = __ldg(p.s + row);
    zi = __ldcg(p.z + row);
    if (W) d1 = __ldg(p.d1 + row);
    len = (int)(__ldg(p.rp + row + 1) - __ldg(p.rp + row));
  }
  double a = 0.0;
  for (; wd >= 8; wd -= 8) {
    slice_step<W, SH, 8>(p, S, cp, wp, a);
    cp += 256;
    if (W) wp += 256;
  }
  if (wd & 4) {
    slice_step<W, SH, 4>(p, S, cp, wp, a);
    cp += 128;
    if (W) wp += 128;
  }
  if (wd & 2) {
    slice_step<W, SH, 2>(p, S, cp, wp, a);
    cp += 64;
    if (W) wp += 64;
  }
  if (wd & 1) slice_step<W, SH, 1>(p, S, cp, wp, a);
  if (ok) relax_row_pre<SH>(p, S, row, len, dd{a, 0.0}, sv, zi, W ? d1 : (double)(len + 1), t);
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

// End of a sweep: every thread's (relaxations, edge updates, sentinel flag)
// go into the ring slot of sweep `sw` by warp-aggregated atomics; one grid
// barrier; then every thread of every block reads the grid totals into dec.
// The slot two sweeps ahead is cleared for reuse (3-slot ring: no second
// barrier needed between reading a slot and clearing it).
__device__ __forceinline__ void sweep_totals(SweepCounters *cnt, unsigned *bar, int sw, TAcc &t,
                                             unsigned long long *s_dec,
                                             unsigned long long (&dec)[3]) {
  unsigned long long u = t.upd, e = t.eu, b = t.bad;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, off);
    e += __shfl_xor_sync(0xffffffffu, e, off);
    b |= __shfl_xor_sync(0xffffffffu, b, off);
  }
  SweepCounters *c = cnt + sw % 3;
  if ((threadIdx.x & 31) == 0 && (u | e | b)) {
    atomicAdd(&c->upd, u);
    atomicAdd(&c->eu, e);
    if (b) atomicOr(&c->bad, b);
  }
  t.upd = t.eu = t.bad = 0;
  grid_sync(bar);
  if (threadIdx.x == 0) {
    s_dec[0] = __ldcg(&c->upd);
    s_dec[1] = __ldcg(&c->eu);
    s_dec[2] = __ldcg(&c->bad);
    if (blockIdx.x == 0) {
      SweepCounters *zc = cnt + (sw + 2) % 3;
      zc->upd = zc->eu = zc->bad = 0;
    }
  }
  __syncthreads();
  dec[0] = s_dec[0];
  dec[1] = s_dec[1];
  dec[2] = s_dec[2];
  __syncthreads();
}

// the loop's outcome for the host: sweeps, relaxations, edge updates, reason
__device__ __forceinline__ void sweep_result(unsigned long long *out, int sweeps,
                                             unsigned long long upd, unsigned long long eu,
                                             int reason) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = (unsigned long long)sweeps;
    out[1] = upd;
    out[2] = eu;
    out[3] = (unsigned long long)reason;
  }
}

#ifndef FJ_MINB
#define FJ_MINB 4
#endif

// ------------------------------------------ one pass over all tasks (CERT/DIS)
template <int MODE, bool W>
__global__ void __launch_bounds__(kBlock, 4) k_pass(KP p) {
  // (frontier phase: the residual pass runs only if the sweeps before ended on a thin sweep)
  if (MODE == CERT && p.prev && __ldcg(p.prev + 3) != 3ull) return;
  Scalars S{};
  if (MODE == CERT) S = *p.sc;
  TAcc t{};
  const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
  for (int wi = warp_id; wi < p.nwtasks_all; wi += gridDim.x * (kBlock / 32))
    do_warp<MODE, W>(p, S, p.wtasks[wi], t);
  for (int ti = blockIdx.x; ti < p.ntasks_all; ti += gridDim.x)
    dispatch_tile<MODE, W>(p, S, p.tasks[ti], t);
  if constexpr (MODE == CERT) {
    // rows without arcs: r = s' − ẑ' (exactly 0 after the pull solvers' init,
    // R20; PUSH relaxes them like any other row, so they are certified too)
    for (int64_t row = p.empty0 + blockIdx.x * (int64_t)kBlock + threadIdx.x; row < p.empty1;
         row += (int64_t)gridDim.x * kBlock)
      cert_row<W>(p, S, (int)row, 0, dd{0.0, 0.0}, t);
  }
  if constexpr (MODE == CERT) {
    // NaN-propagating warp max: a non-finite residual in any lane must fail
    // the certificate (fmax would drop it)
    double m = t.certmax;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, m, off);
      m = (isnan(o) || o > m) ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m != 0.0)
      atomicMax(p.cert_max, (unsigned long long)__double_as_longlong(m));
  } else if constexpr (MODE == DIS) {
    double sdis = t.dis;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sdis += __shfl_xor_sync(0xffffffffu, sdis, off);
    if ((threadIdx.x & 31) == 0 && sdis != 0.0) atomicAdd(p.dis, sdis);
  }
}

// ----------------------------------------------------------- node kernels
static __global__ void k_scalars(const float *__restrict__ smin, const float *__restrict__ smax,
                          double eps, double sigma, double c_override, Scalars *S,
                          int sh_wide = 0) {
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
  {
    int e = 0;
    const double top = (hi + s.c) * (sh_wide ? 2.0 : 1.0);
    if (isfinite(top) && top > 0) frexp(top, &e);  // top < 2^e
    s.sh_scale = ldexp(1.0, e - 32);
    s.sh_enc = ldexp(1.0, 32 - e);
    s.sh_off = -ldexp(1.0, e + 20);
  }
  *S = s;
}

// s into layout order; ẑ' = 0 (Alg. 1 init) except rows with no arcs,
// whose equation is (1 + 0) z_v = s'_v: solved exactly (ẑ'_v = s'_v)
static __global__ void k_init(int64_t n, const int32_t *__restrict__ perm, const int64_t *__restrict__ rp,
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

static __global__ void k_finalize(int64_t n, const int32_t *__restrict__ iperm, const double *__restrict__ z,
                           const Scalars *__restrict__ S, float *__restrict__ zout,
                           double *__restrict__ zprime) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u >= n) return;
  const double zp = z[iperm[u]];
  zout[u] = (float)(zp - S->c);  // ẑ_v − c
  if (zprime) zprime[u] = zp;
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

// host data staged into a workspace buffer; device pointers pass through
static fj_status stage_in(const float *src, int64_t n, Workspace &ws, Staged &out) {
  if (is_device_ptr(src)) {
    out.dev = src;
    return FJ_OK;
  }
  float *d = nullptr;
  FJ_CUDA(ws.alloc(&d, (size_t)n));
  FJ_CUDA(cudaMemcpyAsync(d, src, sizeof(float) * n, cudaMemcpyHostToDevice, ws.st));
  out.dev = d;
  return FJ_OK;
}

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
  p.stasks = L.stasks;
  p.sphase_begin = L.d_sphase_begin;
  p.scol = L.scol;
  p.sw = L.sw;
#ifdef FJ_BOUNDS
  p.nslots = L.nslots;
#endif
  p.phase_begin = L.d_phase_begin;
  p.wphase_begin = L.d_wphase_begin;
  p.ncolors = L.ncolors;
  p.tail_phase = L.tail_phase;
  p.tail_row0 = L.tail_row0;
  p.tail_row1 = L.tail_row1;
  p.tail_beta = L.tail_beta;
  p.ntasks_all = L.ntasks;
  p.nwtasks_all = L.nwtasks;
  p.empty0 = L.n - L.empty_rows;
  p.empty1 = L.n;
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


// implemented in push.cu / batch.cu / solve.cu
const void *sweep_kernel(bool weighted);  // k_sweep<W, false> (solve.cu): the warp-tile list
size_t sweep_kernel_smem();
const void *front_kernel(bool weighted);  // k_front<W> (solve.cu)
fj_status push_solve_impl(fj_graph *g, const float *s_in, double eps, double omega,
                          const fj_opts *o, float *z_out, fj_stats *st_out);
fj_status batch_solve_impl(fj_graph *g, const float *S_in, int k, double eps, double omega,
                           const fj_opts *o, float *Z_out, fj_stats *st_out,
                           const double *omegas, int64_t *relax_out, int *status_out);

}  // namespace fj
