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
// color share no arc, so each phase equals sequential SOR over that color
// (the tiny tail colors of power-law graphs are merged into one asynchronous
// phase with a per-row bound on ω, reading R23, color.cu).
// The loop ends on the first sweep that relaxes nothing: every residual was
// then evaluated on the final ẑ and is ≤ h — the paper's "Q = ∅".
// A separate compensated fp64 pass (certificate) re-checks max |r_v|/h_v.
#include <stdlib.h>

#include <vector>


#include "sweep_common.cuh"

namespace fj {

// ------------------------------------------------------ persistent sweeps
// The sweep list of a phase holds warp units (rows above kWarpTileArcs arcs, or
// kWarpPiece-arc pieces of hub rows; longest first) and warp tiles (short rows
// of one length class).  Warps take the items round-robin, the next item's
// descriptor prefetched; the items are balanced by construction, so no claim
// atomics sit on the hot loop.  One grid barrier ends each color phase.
// SL: the short rows run as row slices (Layout::stasks, one lane per row, no shared
// memory) instead of warp tiles (Layout::rtasks, products staged in shared memory).
template <bool W, int SH, bool SL>
__device__ __forceinline__ void sweep_item(const KP &p, const Scalars &S, const Task &cur, TAcc &t,
                                           double *wprod) {
  if ((cur.kind & 0xff) == kWarp) do_warp<RELAX, W, SH>(p, S, cur, t);
  else if constexpr (SL) relax_slice<W, SH>(p, S, cur, t);
  else relax_warp_tile<W, SH>(p, S, cur, t, wprod);
}

// dynamic part of a phase's list: warps claim chunks of kClaimChunk consecutive items in
// list order (lane 0's atomic; one claim per item costs C5 0.33 ms per sweep — 524 K
// atomics on one address — chunks of 4 or 8 nothing; 16 clump the work again)
#ifndef FJ_CHUNK
#define FJ_CHUNK 4
#endif
constexpr int kClaimChunk = FJ_CHUNK;
__device__ __forceinline__ int claim_chunk(unsigned *claim, int ns) {
  int c = 0;
  if ((threadIdx.x & 31) == 0) c = ns + kClaimChunk * (int)atomicAdd(claim, 1u);
  return __shfl_sync(0xffffffffu, c, 0);
}

template <bool W, bool SL>
__global__ void __launch_bounds__(kBlock, FJ_MINB) k_sweep(KP p) {
  extern __shared__ double s_prod[];  // per warp: the products of its warp tile (!SL)
  __shared__ unsigned long long s_dec[3];
  // sharded solve: sweeps queued after the global stopping sweep do nothing
  if (p.stop && __ldcg(p.stop) != 0ull) return;
  __shared__ Scalars sS;  // shift / thresholds: shared memory, not registers
  if (threadIdx.x == 0) sS = *p.sc;
  __syncthreads();
  const Scalars &S = sS;
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1;
  int phase = 0;
  int max_sweeps = p.max_sweeps;
  int sweeps0 = 0;
  if (p.prev) {
    // fp64 tail of a shadow solve: the totals continue those of the shadow launch
    // (whatever ended it: the tail restarts from ẑ, Lemma 3)
    sweeps0 = (int)__ldcg(p.prev);
    tot_upd = __ldcg(p.prev + 1);
    tot_eu = __ldcg(p.prev + 2);
    max_sweeps = max(1, max_sweeps - sweeps0);
    if (p.skip_if_done && __ldcg(p.prev + 3) == 0ull) {  // the launch before converged
      sweep_result(p.out, sweeps0, tot_upd, tot_eu, 0);
      return;
    }
  }
  for (int sw = 0; sw < max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k, ++phase) {
      const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
      const Task *__restrict__ list = SL ? p.stasks : p.rtasks;
      const int *pb = SL ? p.sphase_begin : p.rphase_begin;
      const int r0 = pb[k], nr = pb[k + 1] - r0;
      const int stride = gridDim.x * (kBlock / 32);
      double *wprod = SL ? nullptr : s_prod + (threadIdx.x >> 5) * kWarpTileArcs;
      // the first items round-robin (the Gauss–Seidel order of the list), the
      // last tail_pct percent claimed in chunks, so no SM idles at the end
      int ns = nr - (int)((long long)nr * p.tail_pct / 100);
      // (slice lists: the warp units, the head of the list, always stay round-robin —
      // a chunk of consecutive hub rows in one warp would serialise them)
      if (SL) ns = max(ns, min(nr, p.wphase_begin[k + 1] - p.wphase_begin[k]));
      unsigned *claim = p.ctr + (phase % 3);
      if (blockIdx.x == 0 && threadIdx.x == 0) p.ctr[(phase + 2) % 3] = 0u;
      int wi = warp_id;
      Task nxt;
      if (wi < ns) nxt = list[r0 + wi];
      while (wi < ns) {
        const Task cur = nxt;
        const int wn = wi + stride;
        if (wn < ns) nxt = list[r0 + wn];
        sweep_item<W, 0, SL>(p, S, cur, t, wprod);
        wi = wn;
      }
      if constexpr (!SL) {
        for (; ns < nr;) {  // warp tiles: one claim per item
          int c = 0;
          if ((threadIdx.x & 31) == 0) c = ns + (int)atomicAdd(claim, 1u);
          c = __shfl_sync(0xffffffffu, c, 0);
          if (c >= nr) break;
          const Task cur = list[r0 + c];
          sweep_item<W, 0, SL>(p, S, cur, t, wprod);
        }
      } else if (ns < nr) {
        // (the next descriptor, and at a chunk's end the next claim, are in flight behind
        // the current item)
        int c = claim_chunk(claim, ns), e = min(c + kClaimChunk, nr);
        if (c < nr) nxt = list[r0 + c];
        while (c < nr) {
          const Task cur = nxt;
          int cn = c + 1;
          if (cn >= e) {
            cn = claim_chunk(claim, ns);
            e = min(cn + kClaimChunk, nr);
          }
          if (cn < nr) nxt = list[r0 + cn];
          sweep_item<W, 0, SL>(p, S, cur, t, wprod);
          c = cn;
        }
      }
      if (k + 1 < p.ncolors) grid_sync(p.bar);
    }
    // grid totals of this sweep (relaxations, edge updates, sentinel)
    unsigned long long dec[3];
    sweep_totals(p.cnt, p.bar, sw, t, s_dec, dec);
    tot_upd += dec[0];
    tot_eu += dec[1];
    sweeps = sw + 1;
    const bool bad = dec[2] != 0, done = dec[0] == 0;
    if (bad) { reason = 2; break; }
    if (done) { reason = 0; break; }
    if (dec[0] < p.thin) { reason = 3; break; }  // thin sweep: the frontier phase takes over
  }
  sweep_result(p.out, sweeps0 + sweeps, tot_upd, tot_eu, reason);
}

// Shadow sweeps (fj_opts.shadow): k_sweep with the ẑ gathers served by the 32-bit
// fixed-point shadow of ẑ' (sweep_common.cuh: sh_dec) — 4 B per gather as SURVEY §8(d)
// counts them, and the whole shadow (n·4 B) stays in L2 where fp64 ẑ' (n·8 B) does not on
// C4.  A relaxed row stores its fp64 ẑ' and its shadow.  The shadow loop ends like
// k_sweep's (a sweep without relaxations, the sentinel, the watchdog), when a value
// leaves the shadow's range, or when a sweep moved no ẑ' by ≥ 4 shadow quanta (it is then
// relaxing the shadow's rounding noise); the fp64 sweeps of k_sweep then run from the
// same ẑ' until nothing relaxes (Lemma 3: ẑ alone determines r), and the
// compensated certificate decides as always.
template <bool W, bool SL>
__global__ void __launch_bounds__(kBlock, FJ_MINB) k_sweep_sh(KP p) {
  extern __shared__ double s_prod[];
  __shared__ unsigned long long s_dec[3];
  __shared__ Scalars sS;
  if (threadIdx.x == 0) sS = *p.sc;
  __syncthreads();
  const Scalars &S = sS;
  TAcc t{};
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps = 0, reason = 1;
  int phase = 0;
  for (int sw = 0; sw < p.max_sweeps; ++sw) {
    for (int k = 0; k < p.ncolors; ++k, ++phase) {
      const int warp_id = blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
      const Task *__restrict__ list = SL ? p.stasks : p.rtasks;
      const int *pb = SL ? p.sphase_begin : p.rphase_begin;
      const int r0 = pb[k], nr = pb[k + 1] - r0;
      const int stride = gridDim.x * (kBlock / 32);
      double *wprod = SL ? nullptr : s_prod + (threadIdx.x >> 5) * kWarpTileArcs;
      int ns = nr - (int)((long long)nr * p.tail_pct / 100);
      // (slice lists: the warp units, the head of the list, always stay round-robin —
      // a chunk of consecutive hub rows in one warp would serialise them)
      if (SL) ns = max(ns, min(nr, p.wphase_begin[k + 1] - p.wphase_begin[k]));
      unsigned *claim = p.ctr + (phase % 3);
      if (blockIdx.x == 0 && threadIdx.x == 0) p.ctr[(phase + 2) % 3] = 0u;
      int wi = warp_id;
      Task nxt;
      if (wi < ns) nxt = list[r0 + wi];
      while (wi < ns) {
        const Task cur = nxt;
        const int wn = wi + stride;
        if (wn < ns) nxt = list[r0 + wn];
        sweep_item<W, 1, SL>(p, S, cur, t, wprod);
        wi = wn;
      }
      if constexpr (!SL) {
        for (; ns < nr;) {  // warp tiles: one claim per item
          int c = 0;
          if ((threadIdx.x & 31) == 0) c = ns + (int)atomicAdd(claim, 1u);
          c = __shfl_sync(0xffffffffu, c, 0);
          if (c >= nr) break;
          const Task cur = list[r0 + c];
          sweep_item<W, 1, SL>(p, S, cur, t, wprod);
        }
      } else if (ns < nr) {
        // (the next descriptor, and at a chunk's end the next claim, are in flight behind
        // the current item)
        int c = claim_chunk(claim, ns), e = min(c + kClaimChunk, nr);
        if (c < nr) nxt = list[r0 + c];
        while (c < nr) {
          const Task cur = nxt;
          int cn = c + 1;
          if (cn >= e) {
            cn = claim_chunk(claim, ns);
            e = min(cn + kClaimChunk, nr);
          }
          if (cn < nr) nxt = list[r0 + cn];
          sweep_item<W, 1, SL>(p, S, cur, t, wprod);
          c = cn;
        }
      }
      if (k + 1 < p.ncolors) grid_sync(p.bar);
    }
    unsigned long long dec[3];
    sweep_totals(p.cnt, p.bar, sw, t, s_dec, dec);
    tot_upd += dec[0];
    tot_eu += dec[1];
    sweeps = sw + 1;
    // dec[2]: bit 0 = sentinel or shadow range, bit 1 = some move of ≥ 4 quanta
    const bool bad = (dec[2] & 1) != 0, done = dec[0] == 0 || (dec[2] & 2) == 0;
    if (bad) { reason = 2; break; }
    if (done) { reason = 4; break; }  // 4: the shadow loop is done, fp64 sweeps must follow
    if (dec[0] < p.thin) { reason = 3; break; }  // thin sweep: the frontier phase takes over
  }
  sweep_result(p.out, sweeps, tot_upd, tot_eu, reason);
}

// Frontier phase: the paper's queue (Alg. 1, Alg. 3) on the thin tail
// of a solve.  Late sweeps relax a few thousand rows each and still read every arc — on C4
// the last 30–60 of ≈ 260 sweeps.  Once a sweep relaxes fewer than KP::thin rows the sweep
// loop ends (reason 3); k_pass<CERT> then writes every row's compensated residual
// r_v = s'_v − ((I+L)ẑ')_v into KP::fr_r, and this kernel runs the push form of the
// method on exactly the rows above threshold, round by round:
//   pop      every listed row v with |r_v| > θ h_v (P:221/453/458; round 0 lists every
//            non-empty row) takes Δ = ω r_v/(1+d_v), ẑ'_v += Δ (equ:sor1), r_v ← (1−ω) r_v
//            (equ:sor2) and leaves one scatter entry per kDepChunk rows that gather it;
//   scatter  a warp per entry adds a_uv Δ to r_u of the rows u that gather v (equ:sor3,
//            P:452; the canonical in-CSR lists them) with fp64 atomics; a row whose |r_u|
//            thereby crosses θ h_u joins the next round's list;
// until a round's list is empty (reason 0: every residual is ≤ θ h — the paper's Q = ∅,
// P:216), a list overflows or the round limit is hit (reason 3: the fp64 sweeps that
// follow carry on from ẑ'; every update made here was a valid relaxation, Lemma 3).
// Pops take r_v by atomic exchange, so a row listed twice is relaxed once.  The residuals
// are exact up to the rounding of their increments (≈ 1e-16 relative); the fp64
// certificate after the solve re-checks every row from ẑ' as always.
// out[4] = rounds, out[5] = scatter entries.
template <bool W>
__global__ void __launch_bounds__(kBlock, 4) k_front(KP p) {
  __shared__ unsigned long long s_dec[3];
  __shared__ Scalars sS;
  unsigned long long tot_upd = 0, tot_eu = 0;
  int sweeps0 = 0;
  if (p.prev) {
    sweeps0 = (int)__ldcg(p.prev);
    tot_upd = __ldcg(p.prev + 1);
    tot_eu = __ldcg(p.prev + 2);
    if (__ldcg(p.prev + 3) != 3ull) {  // the sweeps did not end on a thin sweep: pass through
      sweep_result(p.out, sweeps0, tot_upd, tot_eu, (int)__ldcg(p.prev + 3));
      return;
    }
  }
  if (threadIdx.x == 0) sS = *p.sc;
  __syncthreads();
  const Scalars &S = sS;
  TAcc t{};
  const int lane = threadIdx.x & 31;
  const int64_t gtid = blockIdx.x * (int64_t)kBlock + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * kBlock;
  const int warp_id = (int)(gtid >> 5), nwarps = (int)(nthr >> 5);
  int reason = 3, cur = 0;
  unsigned long long rounds = 0, entries = 0;
  for (int r = 0; r < p.fr_max_rounds; ++r) {
    // ---- pop
    const int64_t cnt = r == 0 ? p.empty0 : (int64_t)__ldcg(p.fr_cnt + cur);
    if (cnt == 0) { reason = 0; break; }
    if (r > 0 && cnt > p.fr_cap) break;  // the list overflowed: the sweeps carry on
    const int *F = p.fr_rows + (size_t)cur * p.fr_cap;
    int *Fn = p.fr_rows + (size_t)(cur ^ 1) * p.fr_cap;
    unsigned *pcnt = p.fr_cnt + 2 + (r & 1);
    for (int64_t e = gtid; e < cnt; e += nthr) {
      const int i = r == 0 ? (int)e : __ldcg(F + e);
      FJ_CHECK(i >= 0 && i < p.empty0);
      const double h = p.theta * threshold(S, (double)p.s[i] + S.c);
      if (!(fabs(__ldcg(p.fr_r + i)) > h)) continue;
      const double rv = __longlong_as_double(
          (long long)atomicExch((unsigned long long *)(p.fr_r + i), 0ull));
      if (!(fabs(rv) <= S.sentinel)) t.bad |= 1;
      if (!(fabs(rv) > h)) {  // another entry of the same row popped it
        if (rv != 0.0) atomicAdd(p.fr_r + i, rv);
        continue;
      }
      const int len = (int)(p.rp[i + 1] - p.rp[i]);
      const double d1 = W ? p.d1[i] : (double)(len + 1);
      // the step ẑ' actually takes (ẑ'_v + Δ rounds; near the fp64 floor of a hub row Δ is a
      // few ulps of ẑ'_v): r_v and the scattered amounts follow the stored value, so the
      // residuals stay those of ẑ' itself — r_v ← r_v − (1+d_v)Δ, (1−ω) r_v in exact terms
      const double zo = __ldcg(p.z + i), zn = zo + p.omega * rv / d1;
      const double dz = zn - zo;
      __stcg(p.z + i, zn);
      const double rem = fma(-d1, dz, rv);
      if (rem != 0.0) {
        atomicAdd(p.fr_r + i, rem);
        if (fabs(rem) > h && dz != 0.0) {  // still above threshold (ω far from 1): stays listed
          // (dz == 0: ẑ'_v cannot move by so little — the row is at fp64's floor and is left
          // to the certificate)
          const unsigned pos = atomicAdd(p.fr_cnt + (cur ^ 1), 1u);
          if (pos < (unsigned)p.fr_cap) Fn[pos] = i;
        }
      }
      if (dz == 0.0) continue;
      t.upd++;
      t.eu += (unsigned long long)len;
      const int u = p.perm[i];
      const unsigned nd = (unsigned)(p.in_rp[u + 1] - p.in_rp[u]);
      const unsigned nc = (nd + kDepChunk - 1) / kDepChunk;
      if (nc) {
        const unsigned pos = atomicAdd(pcnt, nc);
        const long long bits = __double_as_longlong(dz);
        for (unsigned c = 0; c < nc && pos + c < (unsigned)p.fr_pcap; c++)
          p.fr_push[pos + c] = make_int4(i, (int)c, (int)(bits & 0xffffffffll), (int)(bits >> 32));
      }
    }
    grid_sync(p.bar);
    // ---- scatter
    const unsigned np = __ldcg(pcnt);
    if (np > (unsigned)p.fr_pcap) break;  // entries were dropped: ẑ' is valid, r is not
    for (unsigned e = warp_id; e < np; e += nwarps) {
      const int4 q = p.fr_push[e];
      const double dz = __longlong_as_double(((long long)q.w << 32) | (unsigned)q.z);
      FJ_CHECK(q.x >= 0 && q.x < p.empty0 && q.y >= 0);
      const int u = p.perm[q.x];
      const int64_t k0 = p.in_rp[u] + (int64_t)q.y * kDepChunk;
      const int64_t k1 = min(p.in_rp[u + 1], k0 + kDepChunk);
      for (int64_t k = k0 + lane; k < k1; k += 32) {
        const int v = p.iperm[p.in_col[k]];
        FJ_CHECK(k >= p.in_rp[u] && k < p.in_rp[u + 1] && v >= 0 && v < p.empty0);
        const double inc = (W ? (double)p.in_w[k] : 1.0) * dz;
        const double old = atomicAdd(p.fr_r + v, inc);
        const double hv = p.theta * threshold(S, (double)p.s[v] + S.c);
        if (fabs(old) <= hv && fabs(old + inc) > hv) {
          const unsigned pos = atomicAdd(p.fr_cnt + (cur ^ 1), 1u);
          if (pos < (unsigned)p.fr_cap) Fn[pos] = v;
        }
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.fr_cnt[cur] = 0u;                // this round's list is used up
      p.fr_cnt[2 + ((r + 1) & 1)] = 0u;  // the next round's scatter count
    }
    unsigned long long dec[3];
    sweep_totals(p.cnt, p.bar, r, t, s_dec, dec);
    tot_upd += dec[0];
    tot_eu += dec[1];
    rounds = (unsigned long long)(r + 1);
    entries += np;
    cur ^= 1;
    if (dec[2] != 0) { reason = 2; break; }
  }
  sweep_result(p.out, sweeps0, tot_upd, tot_eu, reason);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.out[4] = rounds;
    p.out[5] = entries;
  }
}

// shadow init: zs = encode(ẑ') for every row
__global__ void k_shadow_init(int64_t n, const double *__restrict__ z, const Scalars *__restrict__ S,
                              unsigned *__restrict__ zs) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) zs[i] = __double2uint_rn(z[i] * S->sh_enc);
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

// the one-sweep-per-launch entry of the sharded solve (shard.cu)
const void *sweep_kernel(bool weighted) {
  return weighted ? (const void *)k_sweep<true, false> : (const void *)k_sweep<false, false>;
}
size_t sweep_kernel_smem() { return (kBlock / 32) * kWarpTileArcs * sizeof(double); }
// the frontier phase's kernel, for the batched solve (batch.cu runs it column by column)
const void *front_kernel(bool weighted) {
  return weighted ? (const void *)k_front<true> : (const void *)k_front<false>;
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
  if (method == FJ_METHOD_COLORED) FJ_TRY(build_coloring(g, o));
  if (method == FJ_METHOD_PUSH) {
    if (o->z_init) {
      set_error("fj_solve: z_init (warm start) is supported by ASYNC/COLORED, not PUSH");
      return FJ_ERR_INVALID;
    }
    return push_solve_impl(g, s_in, eps, omega, o, z_out, st_out);
  }
  const Layout &L = (method == FJ_METHOD_COLORED) ? g->color_layout : g->async_layout;
  const bool W = g->weighted != 0;
  // shadow sweeps (fj_opts.shadow; default: on hub-dominated layouts, where the warp units
  // hold over half the arcs — C2 / C4 gain 5–8 % per sweep, the short-row layouts C3 / C5
  // lose as much to the extra shadow store and decode, profiles/r02_shadow_*.txt)
  const bool use_shadow =
      L.m > 0 && (o->shadow > 0 || (o->shadow < 0 && 2 * L.warp_unit_arcs > L.m));

  Workspace ws(st);
  cudaEvent_t e0, e1, es0, es1, ec0, ec1;
  for (cudaEvent_t *e : {&e0, &e1, &es0, &es1, &ec0, &ec1}) FJ_CUDA(ws.event(e));
  FJ_CUDA(cudaEventRecord(e0, st));

  Staged s{};
  FJ_TRY(stage_in(s_in, n, ws, s));
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
  unsigned *zs = nullptr;
  // ẑ' and its shadow carry one more entry, 0: the column of the row slices' padding
  if (use_shadow) {
    FJ_CUDA(ws.alloc(&zs, n + 1));
    FJ_CUDA(cudaMemsetAsync(zs + n, 0, sizeof(unsigned), st));
  }
  FJ_CUDA(ws.alloc(&s_l, n));
  FJ_CUDA(ws.alloc(&z, n + 1));
  FJ_CUDA(cudaMemsetAsync(z + n, 0, sizeof(double), st));
  FJ_CUDA(ws.alloc(&smin, 2));
  smax = smin + 1;
  FJ_CUDA(ws.alloc(&S, 1));
  FJ_CUDA(ws.alloc(&partial, std::max(1, L.npartials)));
  FJ_CUDA(ws.alloc(&arrive, std::max(1, L.npartials)));
  FJ_CUDA(ws.alloc(&ctl, kCtlWords));
  FJ_CUDA(ws.alloc(&cnt, 3));
  FJ_CUDA(ws.alloc(&outv, 48));  // [0..3] sweep result, [4] certificate; stage results of the
                                 // chain at 8 (first sweeps), 16 / 32 (frontier), 24 (fp64)
  certbits = outv + 4;
  if (!zdev) FJ_CUDA(ws.alloc(&zo, n));
  if (o->zprime_out && !zpdev) FJ_CUDA(ws.alloc(&zp, n));

  // a2: shift and init (Alg. 2)
  FJ_TRY(minmax_f32(s.dev, n, smin, ws, g->num_sms));  // smin[0] = min s, smin[1] = smax = max s
  fj::count_launch();
  k_scalars<<<1, 1, 0, st>>>(smin, smax, eps, o->sigma, o->c, S,
                             (omega > 1.0 || o->z_init) ? 1 : 0);
  const double *zinit = nullptr;
  double *zinit_owned = nullptr;
  if (o->z_init) {
    if (is_device_ptr(o->z_init)) {
      zinit = o->z_init;
    } else {
      FJ_CUDA(ws.alloc(&zinit_owned, n));
      FJ_CUDA(cudaMemcpyAsync(zinit_owned, o->z_init, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      zinit = zinit_owned;
    }
  }
  fj::count_launch();
  k_init<<<gridn(n), kBlock, 0, st>>>(n, L.perm, L.rp, s.dev, S, s_l, z, zinit);
  if (use_shadow) {
    fj::count_launch();
    k_shadow_init<<<gridn(n), kBlock, 0, st>>>(n, z, S, zs);
  }

  KP p = make_kp(g, L);
  p.zs = zs;
  p.s = s_l;
  p.z = z;
  p.sc = S;
  p.omega = omega;
  p.theta = 1.0;
  p.partial = partial;
  p.arrive = arrive;
  p.max_sweeps = o->max_sweeps;
  p.ctr = ctl;
  p.bar = ctl + 8;
  p.cnt = cnt;
  p.out = outv;
  p.cert_max = certbits;

  // short rows as row slices (fj_opts.slices; the layout carries them unless it is a
  // shard's) or as warp tiles.  Default: slices, except on colored layouts with rows
  // above 32 arcs — every phase then waits for its deepest slice (a lane walks up to 256
  // arcs): C3 at ω = 1.6, 12 phases, 0.76 vs 0.63 ms per sweep and 130 vs 109 sweeps
  // (profiles/r02_slices_variants_ab.txt)
  const bool SL = L.scol != nullptr &&
                  (o->slices > 0 || (o->slices < 0 && (L.ncolors == 1 || L.max_len <= 32)));
  const void *fn = SL ? (W ? (const void *)k_sweep<true, true> : (const void *)k_sweep<false, true>)
                      : (W ? (const void *)k_sweep<true, false> : (const void *)k_sweep<false, false>);
  const size_t sweep_smem = SL ? 0 : sweep_kernel_smem();
  FJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem));
  // Shared-memory carveout: the tile staging needs ≈ 68 KB per SM, for which
  // the driver's default picks the 132 KB configuration (124 KB of L1).  On
  // hub-dominated layouts (warp units hold over half the arcs: C2, C4) the
  // 100 KB configuration's larger L1 (156 KB) keeps more hub ẑ lines: C4
  // 1.418 → 1.335 ms per sweep, C2 0.1055 → 0.1015; on short-row layouts the
  // staler L1 lines cost more sweeps than the larger L1 saves (C3 +6 % sweeps),
  // so they keep the default (profiles/r02_carveout_ab.txt).
#ifdef FJ_CARVE
  const int carve = FJ_CARVE;  // diagnostic build: forced preference (percent)
#else
  const int carve = SL ? 0 : (2 * L.warp_unit_arcs > L.m ? 31 : -1);
#endif
  // Dynamic share of each phase's work list.  Warp tiles (equal items): the last 15 % on
  // hub-dominated layouts (C4 1.358 → 1.315 ms per sweep, C2 and C3 within ±1 %, C5 +3 %:
  // profiles/r02_tailclaim_ab.txt), else none.  Row slices (items from 32 to 8192 arcs, so
  // round-robin leaves SMs waiting at the sweep's barrier: 12 % of the warp samples): the
  // last 50 % of the items, chunks of 4 — C4 0.99 → 0.94 ms per sweep, C3 −8 %, C2 −6 %,
  // C5 ±0 (profiles/r02_slices_variants_ab.txt) — on one-phase lists of at least 4 items
  // per warp; short lists and color phases stay round-robin (C1 2.6 vs 1.5 ms, C5 at
  // ω = 1.25 12.1 vs 11.1 ms with claims)
#ifdef FJ_TAILPCT
  p.tail_pct = FJ_TAILPCT;
#else
  p.tail_pct = SL ? -1 : (2 * L.warp_unit_arcs > L.m ? 15 : 0);  // −1: set below (needs the grid)
#endif
  // (a per-function setting: set on every solve, −1 = the driver's default)
  FJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                               carve >= 0 ? carve : (int)cudaSharedmemCarveoutDefault));
  const int grid = persistent_grid(fn, g->num_sms, sweep_smem);
  if (p.tail_pct < 0)
    p.tail_pct = (L.ncolors == 1 && L.nstasks >= 4 * grid * (kBlock / 32)) ? 50 : 0;
  // shadow launch: the fp64 kernel's shape (same staging, carveout and grid)
  const void *shfn =
      SL ? (W ? (const void *)k_sweep_sh<true, true> : (const void *)k_sweep_sh<false, true>)
         : (W ? (const void *)k_sweep_sh<true, false> : (const void *)k_sweep_sh<false, false>);
  int sh_grid = 0;
  if (use_shadow) {
    FJ_CUDA(cudaFuncSetAttribute(shfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sweep_smem));
    FJ_CUDA(cudaFuncSetAttribute(shfn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 carve >= 0 ? carve : (int)cudaSharedmemCarveoutDefault));
    sh_grid = persistent_grid(shfn, g->num_sms, sweep_smem);
  }
  cudaEvent_t esh, ef[4];
  FJ_CUDA(ws.event(&esh));
  for (cudaEvent_t &e : ef) FJ_CUDA(ws.event(&e));
  // Frontier phase (fj_opts.frontier): once a sweep relaxes fewer than `thin` rows, k_front
  // runs the push form on the rows above threshold (any layout: it works on rows, not items).
  // (colored layouts: the rounds pop with ω = 1 — Jacobi-ordered rounds carry no SOR
  // guarantee, plain pops converge in any order and Lemma 3 allows any amount)
  const bool use_front = o->frontier != 0 && L.active_rows > 0;
  const void *ffn = W ? (const void *)k_front<true> : (const void *)k_front<false>;
  int fgrid = 0;
  if (use_front) {
    const int64_t act = std::max<int64_t>(1, L.active_rows);
    p.thin = o->frontier > 0 ? (unsigned long long)o->frontier
                             : (unsigned long long)std::max<int64_t>(32, act / FJ_THIN_DIV);
    p.fr_cap = (int)std::min<int64_t>(std::max<int64_t>(4096, act / 4), 1 << 30);
    p.fr_pcap = (int)std::min<int64_t>((int64_t)p.fr_cap + L.m / kDepChunk, 1 << 30);
    FJ_CUDA(ws.alloc(&p.fr_r, (size_t)n));
    FJ_CUDA(ws.alloc(&p.fr_rows, 2 * (size_t)p.fr_cap));
    FJ_CUDA(ws.alloc(&p.fr_push, (size_t)p.fr_pcap));
    FJ_CUDA(ws.alloc(&p.fr_cnt, 4));
    p.in_rp = g->in_rp;
    p.in_col = g->in_col;
    p.in_w = g->in_w;
    p.perm = L.perm;
    p.iperm = L.iperm;
    p.fr_max_rounds = 100000;
    FJ_CUDA(cudaFuncSetAttribute(ffn, cudaFuncAttributePreferredSharedMemoryCarveout, 0));
    fgrid = persistent_grid(ffn, g->num_sms, 0);
  }
  const unsigned long long thin = p.thin;
  float ms_sweep = 0, ms_cert = 0, ms_shadow = 0, ms_front = 0;
  int rounds = 0;
  stats.colors = L.ncolors;
  // counters at rest before every launch of the chain (ring slots, claim words, arrivals)
  auto rest = [&]() -> fj_status {
    FJ_CUDA(cudaMemsetAsync(ctl, 0, sizeof(unsigned) * kCtlWords, st));
    FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(SweepCounters) * 3, st));
    // hub-piece arrival counters start at 0 for every launch (a resumed
    // sweep or the certificate never inherits a half-finished count)
    FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
    return FJ_OK;
  };
  const void *rfn = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
  unsigned long long *scratch_max = nullptr;
  if (use_front) FJ_CUDA(ws.alloc(&scratch_max, 1));
  auto launch_front = [&](unsigned long long *prev, unsigned long long *out, int ev) -> fj_status {
    FJ_TRY(rest());
    FJ_CUDA(cudaMemsetAsync(p.fr_cnt, 0, sizeof(unsigned) * 4, st));
    FJ_CUDA(cudaMemsetAsync(scratch_max, 0, sizeof(unsigned long long), st));
    FJ_CUDA(cudaEventRecord(ef[ev], st));
    {  // residuals of every row from ẑ' (compensated; runs only after a thin exit)
      KP q = p;
      q.prev = prev;
      q.ctr = ctl + 5;
      q.rout = p.fr_r;
      q.cert_max = scratch_max;
      void *args[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchKernel(rfn, persistent_grid(rfn, g->num_sms), kBlock, args, 0, st));
    }
    FJ_TRY(rest());
    KP q = p;
    q.prev = prev;
    q.out = out;
    if (L.ncolors > 1) q.omega = 1.0;
    void *args[] = {&q};
    fj::count_launch();
    FJ_CUDA(cudaLaunchCooperativeKernel(ffn, fgrid, kBlock, args, 0, st));
    FJ_CUDA(cudaEventRecord(ef[ev + 1], st));
    return FJ_OK;
  };
  for (;;) {
    // a3–a5: persistent sweeps with on-device loop control.  The chain of a round:
    //   [shadow sweeps | fp64 sweeps] (thin exit) → frontier → fp64 sweeps (thin exit) →
    //   frontier → fp64 sweeps; every stage continues the totals of the one before and
    //   passes through at once if that one converged (frontier: unless it ended thin)
    FJ_TRY(rest());
    FJ_CUDA(cudaMemsetAsync(outv, 0, sizeof(unsigned long long) * 48, st));
    FJ_CUDA(cudaEventRecord(es0, st));
    const bool sh_round = use_shadow && rounds == 0;  // resumes run in fp64 only
    p.prev = nullptr;
    p.thin = thin;
    p.skip_if_done = 0;
    if (sh_round) {
      KP q = p;
      q.out = outv + 8;
      void *args[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(shfn, sh_grid, kBlock, args, sweep_smem, st));
      FJ_CUDA(cudaEventRecord(esh, st));
      p.prev = outv + 8;
    } else if (use_front) {
      KP q = p;
      q.out = outv + 8;
      void *args[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, sweep_smem, st));
      p.prev = outv + 8;
    }
    if (use_front) {
      FJ_TRY(launch_front(outv + 8, outv + 16, 0));
      FJ_TRY(rest());
      KP q = p;  // fp64 sweeps; they may end thin again (rows the shadow sweeps left)
      q.prev = outv + 16;
      q.out = outv + 24;
      q.skip_if_done = 1;
      void *args[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, sweep_smem, st));
      FJ_TRY(launch_front(outv + 24, outv + 32, 2));
      p.prev = outv + 32;
      p.skip_if_done = 1;
      p.thin = 0;
    }
    if (p.prev) FJ_TRY(rest());
    {
      void *args[] = {&p};
      fj::count_launch();
      FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, sweep_smem, st));
    }
    FJ_CUDA(cudaEventRecord(es1, st));
    // fp64 compensated certificate over every non-empty row
    if (o->certify) {
      KP q = p;
      q.ctr = ctl + 5;
      q.prev = nullptr;  // (with prev set the pass is the frontier phase's conditional one)
      FJ_CUDA(cudaMemsetAsync(arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
      FJ_CUDA(cudaEventRecord(ec0, st));
      const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
      void *cargs[] = {&q};
      fj::count_launch();
      FJ_CUDA(cudaLaunchKernel(cf, persistent_grid(cf, g->num_sms), kBlock, cargs, 0, st));
      FJ_CUDA(cudaEventRecord(ec1, st));
    }
    unsigned long long h[48];
    FJ_CUDA(cudaMemcpyAsync(h, outv, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    float a = 0;
    FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
    ms_sweep += a;
    if (sh_round) {
      FJ_CUDA(cudaEventElapsedTime(&a, es0, esh));
      ms_shadow += a;
      stats.shadow_sweeps += (int64_t)h[8];
    }
    if (use_front) {
      for (int e = 0; e < 4; e += 2) {
        FJ_CUDA(cudaEventElapsedTime(&a, ef[e], ef[e + 1]));
        ms_front += a;
      }
      stats.frontier_rounds += (int64_t)(h[16 + 4] + h[32 + 4]);
      stats.frontier_pushes += (int64_t)(h[16 + 5] + h[32 + 5]);
    }
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
  stats.shadow_ms = ms_shadow;
  stats.frontier_ms = ms_front;
  stats.cert_ms = ms_cert;
  stats.c = hs.c;
  stats.eps_prime = hs.eps_p;

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
  Workspace ws(st);
  Staged z{}, s{};
  FJ_TRY(stage_in(z_in, n, ws, z));
  if (s_in) FJ_TRY(stage_in(s_in, n, ws, s));
  double *zl = nullptr, *sums = nullptr;
  unsigned *ctr = nullptr;
  FJ_CUDA(ws.alloc(&zl, n));
  FJ_CUDA(ws.alloc(&sums, 5));
  FJ_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * 5, st));
  FJ_CUDA(ws.alloc(&ctr, 1));
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
  FJ_CUDA(cudaGetLastError());
  out->polarization = h[1];
  // each undirected edge is stored as two arcs (reading R14)
  out->disagreement = g->directed ? h[4] : 0.5 * h[4];
  out->internal_conflict = s_in ? h[2] : 0.0;
  out->controversy = h[3];
  return FJ_OK;
}


// ------------------------------------------------- practical roofline probe
// Σ_k w_k · x[col_k] over the layout's arc stream, 8 arcs per thread in
// flight, grid-stride; the sum only keeps the loads alive
template <bool W>
__global__ void __launch_bounds__(kBlock) k_gather_probe(int64_t m, const int32_t *__restrict__ col,
                                                         const float *__restrict__ w,
                                                         const double *__restrict__ x,
                                                         double *__restrict__ sink) {
  constexpr int U = 8;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < m; k0 += stride * U) {
    int j[U];
    float wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t k = k0 + u * stride;
      const bool ok = k < m;
      j[u] = ld_stream(col + (ok ? k : 0));
      wv[u] = ok ? (W ? ld_stream(w + (ok ? k : 0)) : 1.0f) : 0.0f;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = ld_z(x + j[u]);
#pragma unroll
    for (int u = 0; u < U; u++) acc = fma((double)wv[u], v[u], acc);
  }
  if (acc == 1.2345e300) *sink = acc;
}

fj_status gather_probe_impl(fj_graph *g, int reps, double *ms_per_pass) {
  cudaStream_t st = g->stream;
  const Layout &L = g->async_layout;
  Workspace ws(st);
  double *x = nullptr;
  FJ_CUDA(ws.alloc(&x, (size_t)g->n + 1));
  FJ_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (g->n + 1), st));
  const void *fn = L.w ? (const void *)k_gather_probe<true> : (const void *)k_gather_probe<false>;
  const int grid = persistent_grid(fn, g->num_sms);
  int64_t m = L.m;
  const int32_t *col = L.col;
  const float *w = L.w;
  double *sink = x + g->n;
  void *args[] = {&m, &col, &w, &x, &sink};
  cudaEvent_t a, b;
  FJ_CUDA(ws.event(&a));
  FJ_CUDA(ws.event(&b));
  fj::count_launch();
  FJ_CUDA(cudaLaunchKernel(fn, grid, kBlock, args, 0, st));  // warm-up
  FJ_CUDA(cudaEventRecord(a, st));
  for (int r = 0; r < reps; r++) {
    fj::count_launch();
    FJ_CUDA(cudaLaunchKernel(fn, grid, kBlock, args, 0, st));
  }
  FJ_CUDA(cudaEventRecord(b, st));
  FJ_CUDA(cudaEventSynchronize(b));
  float ms = 0.f;
  FJ_CUDA(cudaEventElapsedTime(&ms, a, b));
  FJ_CUDA(cudaStreamSynchronize(st));
  *ms_per_pass = ms / reps;
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
  Workspace ws(st);
  FJ_CUDA(ws.alloc(&x, (size_t)n));
  FJ_CUDA(ws.alloc(&y, n));
  FJ_CUDA(ws.alloc(&sums, 2));
  FJ_CUDA(ws.alloc(&ctr, 1));
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

fj_status fj_gather_probe(fj_graph_t g, int reps, double *ms_per_pass) {
  if (!g || reps < 1 || !ms_per_pass) {
    fj::set_error("fj_gather_probe: need g, reps >= 1, ms_per_pass");
    return FJ_ERR_INVALID;
  }
  return fj::gather_probe_impl(g, reps, ms_per_pass);
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
  if (method == FJ_METHOD_PUSH) {
    fj::set_error("fj_omega_sweep: the sweep runs batched (ASYNC / COLORED), not PUSH");
    return FJ_ERR_INVALID;
  }
  const int cap = *npts;
  // the paper's heuristic: start near 2, lower ω by a fixed step to 1,
  // keep the ω with the fewest updates; diverging ω cost +inf.  The
  // grid runs as ω batches of up to 8 columns (fj_solve_batch_omega): one
  // schedule for every ω of the grid, one set of CSR streams per batch.
  std::vector<double> grid;
  for (int i = 0;; i++) {
    const double om = hi - i * step;
    if (om < lo - 1e-12) break;
    grid.push_back(om);
  }
  float *z = nullptr;
  FJ_CUDA(cudaMallocAsync(&z, sizeof(float) * g->n * 8, g->stream));
  fj_opts o;
  fj_opts_default(&o);
  o.method = method;
  double best = 1.0;
  int64_t best_cost = -1;
  int k = 0;
  for (size_t c0 = 0; c0 < grid.size(); c0 += 8) {
    const int kc = (int)std::min<size_t>(8, grid.size() - c0);
    int64_t rel[8];
    int stat[8];
    fj_stats st;
    fj_status rc = fj_solve_batch_omega(g, s, kc, grid.data() + c0, eps, &o, z, &st, rel, stat);
    if (rc != FJ_OK && rc != FJ_ERR_NUMERIC) {
      cudaFreeAsync(z, g->stream);
      return rc;
    }
    for (int r = 0; r < kc; r++, k++) {
      const double om = grid[c0 + r];
      if (table && k < cap) {
        table[3 * k] = om;
        table[3 * k + 1] = (double)rel[r];
        table[3 * k + 2] = (double)stat[r];
      }
      if (stat[r] == FJ_OK && (best_cost < 0 || rel[r] <= best_cost)) {
        best_cost = rel[r];  // ties go to the smaller ω: later in the walk
        best = om;
      }
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

