// color.cu — distance-1 coloring of the symmetrised graph (§8 row a1, K4),
// built lazily for the COLORED (multicolor SOR) schedule.
//
// Rows of one color share no arc in either direction, so relaxing them
// simultaneously equals relaxing them one after another: a colored sweep is a
// sequential SOR sweep in (color, id) order, which is what Theorem 3
// and the SOR derivation assume.
//
// Algorithm: speculative first-fit in largest-first degree buckets.  Vertices
// are bucketed by ⌊log2(symmetrised degree)⌋ and the buckets are colored from
// the largest degrees down, as sequential largest-first greedy would.  Inside
// a bucket every worklist vertex takes, all at once, the smallest color absent
// from its neighbours' FINAL colors (other worklist members are ignored, so the
// result does not depend on timing: deterministic); then every vertex sharing
// its color with a higher-priority worklist neighbour (priority = (degree,
// hash(id))) goes to the next worklist, the others are final.  C3: 99 colors in
// ≈ 30 ms; Jones–Plassmann (FJ_COLORING=jp: a vertex colors only when it is
// the local priority maximum) gave 96 colors but needed 1,318 full passes and
// 3.6 s, since the mutually adjacent hubs color one per round.
#include <stdio.h>
#include <string.h>


#include "fj_internal.cuh"

namespace fj {

__device__ __forceinline__ uint64_t prio(int64_t deg, int32_t v) {
  uint32_t h = (uint32_t)v * 0x9E3779B1u;
  h ^= h >> 15;
  h *= 0x85EBCA77u;
  h ^= h >> 13;
  return ((uint64_t)deg << 32) | h;
}

// warp per vertex
__global__ void k_jp_round(int64_t n, const int64_t *__restrict__ irp, const int32_t *__restrict__ icol,
                           const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                           const int32_t *__restrict__ cold, int32_t *__restrict__ cnew,
                           unsigned long long *__restrict__ remaining, int *__restrict__ maxc) {
  const int lane = threadIdx.x & 31;
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps) {
    if (cold[v] >= 0) continue;
    const int64_t ib = irp[v], ie = irp[v + 1], ob = orp[v], oe = orp[v + 1];
    const uint64_t pv = prio((ie - ib) + (oe - ob), (int32_t)v);
    bool blocked = false;
    for (int64_t k = ib + lane; k < ie && !blocked; k += 32) {
      const int32_t u = icol[k];
      if (cold[u] < 0 && prio((irp[u + 1] - irp[u]) + (orp[u + 1] - orp[u]), u) > pv) blocked = true;
    }
    for (int64_t k = ob + lane; k < oe && !blocked; k += 32) {
      const int32_t u = ocol[k];
      if (cold[u] < 0 && prio((irp[u + 1] - irp[u]) + (orp[u + 1] - orp[u]), u) > pv) blocked = true;
    }
    if (__any_sync(0xffffffffu, blocked)) {
      if (lane == 0) atomicAdd(remaining, 1ull);
      continue;
    }
    int chosen = -1;
    for (int base = 0; chosen < 0; base += 64) {
      uint64_t used = 0;
      for (int64_t k = ib + lane; k < ie; k += 32) {
        const int c = cold[icol[k]] - base;
        if (c >= 0 && c < 64) used |= 1ull << c;
      }
      for (int64_t k = ob + lane; k < oe; k += 32) {
        const int c = cold[ocol[k]] - base;
        if (c >= 0 && c < 64) used |= 1ull << c;
      }
      const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)used);
      const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(used >> 32));
      const uint64_t all = ((uint64_t)hi << 32) | lo;
      if (all != ~0ull) chosen = base + __ffsll((long long)~all) - 1;
    }
    if (lane == 0) {
      cnew[v] = chosen;
      atomicMax(maxc, chosen);
    }
  }
}

// rows per color
__global__ void k_color_hist(int64_t n, const int32_t *__restrict__ c, int nc,
                             unsigned long long *__restrict__ cnt) {
  extern __shared__ unsigned long long h[];
  for (int i = threadIdx.x; i < nc; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(h + c[v], 1ull);
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x)
    if (h[i]) atomicAdd(cnt + i, h[i]);
}

__global__ void k_color_clamp(int64_t n, int32_t *__restrict__ c, int K) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    if (c[v] > K) c[v] = K;
}

// Tail merge (reading R23).  First-fit colorings of power-law graphs have a
// long tail of tiny colors (the dense core: C3 has 96 colors, the last ~85
// holding ~2% of the rows), and every color costs a grid barrier plus a
// phase tail.  Colors K.. are merged into ONE phase whose rows may be
// adjacent and are relaxed asynchronously.  Rows of colors < K keep the exact
// sequential SOR semantics with the caller's ω.  A tail row i relaxes with
// ω_i = min(ω, 1.98/(1+β_i)), β_i = Σ_{j in tail} a_ij/(1+d_i): then every
// row of the tail block's iteration matrix T = I − Ω D⁻¹ A_BB has
// |1−ω_i| + ω_i β_i < 1, i.e. ‖T‖_∞ < 1, the Chazan–Miranker condition under
// which asynchronous relaxation of the block converges whatever the update
// order and staleness.  K = the smallest index whose tail holds at most
// fj_opts.tail_frac (default 1%) of the rows; 0 disables the merge.
static fj_status merge_tail_colors(fj_graph *g, double frac) {
  cudaStream_t st = g->stream;
  const int nc = g->ncolors;
  g->ncolors_raw = nc;
  g->tail_color = -1;
  if (!(frac > 0.0) || nc <= 2 || nc > 6000) return FJ_OK;
  Workspace ws(st);
  unsigned long long *cnt = nullptr;
  FJ_CUDA(ws.alloc(&cnt, (size_t)nc));
  FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * nc, st));
  fj::count_launch();
  k_color_hist<<<std::max(1, std::min(g->num_sms * 4, (int)((g->n + kBlock - 1) / kBlock))), kBlock,
                 sizeof(unsigned long long) * nc, st>>>(g->n, g->colors, nc, cnt);
  std::vector<unsigned long long> h(nc);
  FJ_CUDA(cudaMemcpyAsync(h.data(), cnt, sizeof(unsigned long long) * nc, cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  const double cap = frac * (double)g->n;
  int K = nc;
  double tail = 0.0;
  while (K > 0 && tail + (double)h[K - 1] <= cap) tail += (double)h[--K];
  if (nc - K < 2) return FJ_OK;  // nothing to merge
  fj::count_launch();
  k_color_clamp<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((g->n + kBlock - 1) / kBlock, (int64_t)g->num_sms * 8)), kBlock, 0, st>>>(g->n, g->colors, K);
  g->ncolors = K + 1;
  g->tail_color = K;
  return FJ_OK;
}

// β_i for the rows [r0, r1) of the tail phase (warp per row)
template <bool W>
__global__ void k_tail_beta(int64_t r0, int64_t r1, const int64_t *__restrict__ rp,
                            const int32_t *__restrict__ col, const float *__restrict__ w,
                            const double *__restrict__ d1, float *__restrict__ beta) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = r0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < r1; i += nw) {
    const int64_t b = rp[i], e = rp[i + 1];
    double a = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) {
      const int32_t j = col[k];
      if (j >= r0 && j < r1) a += W ? (double)w[k] : 1.0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) beta[i - r0] = (float)(a / (W ? d1[i] : (double)(e - b + 1)));
  }
}

fj_status tail_bounds(fj_graph *g, Layout *L) {
  L->tail_phase = g->tail_color;
  if (g->tail_color < 0) return FJ_OK;
  cudaStream_t st = g->stream;
  const int64_t r0 = L->crow[g->tail_color], r1 = L->crow[g->tail_color + 1];
  L->tail_row0 = r0;
  L->tail_row1 = r1;
  FJ_CUDA(cudaMallocAsync(&L->tail_beta, sizeof(float) * std::max<int64_t>(1, r1 - r0), st));
  if (r1 > r0) {
    const unsigned blocks =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(((r1 - r0) * 32 + kBlock - 1) / kBlock,
                                                         (int64_t)g->num_sms * 8));
    fj::count_launch();
    if (g->weighted)
      k_tail_beta<true><<<blocks, kBlock, 0, st>>>(r0, r1, L->rp, L->col, L->w, L->d1, L->tail_beta);
    else
      k_tail_beta<false><<<blocks, kBlock, 0, st>>>(r0, r1, L->rp, L->col, L->w, L->d1, L->tail_beta);
  }
  return FJ_OK;
}

// worklist entry i: smallest color absent from the neighbours (in- and
// out-arcs) of v = wl[i], read from the live color array (warp per vertex)
__global__ void k_spec_assign(int64_t nw, const int32_t *__restrict__ wl,
                              const int64_t *__restrict__ irp, const int32_t *__restrict__ icol,
                              const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                              const int32_t *__restrict__ mark, int round, int32_t *color) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < nw; i += nwarps) {
    const int32_t v = wl[i];
    const int64_t ib = irp[v], ie = irp[v + 1], ob = orp ? orp[v] : 0, oe = orp ? orp[v + 1] : 0;
    int chosen = -1;
    for (int base = 0; chosen < 0; base += 64) {
      uint64_t used = 0;
      for (int64_t k = ib + lane; k < ie; k += 32) {
        const int32_t u = icol[k];
        const int c = mark[u] == round ? -1 : color[u] - base;  // only final colors count
        if (c >= 0 && c < 64) used |= 1ull << c;
      }
      for (int64_t k = ob + lane; k < oe; k += 32) {
        const int32_t u = ocol[k];
        const int c = mark[u] == round ? -1 : color[u] - base;
        if (c >= 0 && c < 64) used |= 1ull << c;
      }
      const unsigned lo = __reduce_or_sync(0xffffffffu, (unsigned)used);
      const unsigned hi = __reduce_or_sync(0xffffffffu, (unsigned)(used >> 32));
      const uint64_t all = ((uint64_t)hi << 32) | lo;
      if (all != ~0ull) chosen = base + __ffsll((long long)~all) - 1;
    }
    if (lane == 0) color[v] = chosen;
  }
}

// conflicts: v loses (next worklist) if a neighbour has its color and a higher
// priority; winners are final (their colors feed the color count)
__global__ void k_spec_detect(int64_t nw, const int32_t *__restrict__ wl,
                              const int64_t *__restrict__ irp, const int32_t *__restrict__ icol,
                              const int64_t *__restrict__ orp, const int32_t *__restrict__ ocol,
                              const int32_t *__restrict__ color, int32_t *__restrict__ next,
                              unsigned long long *__restrict__ nnext, int *__restrict__ maxc) {
  // (assign read only final colors, so a tie can only be with another vertex
  // of this worklist: the lower priority of the two recolors next round)
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < nw; i += nwarps) {
    const int32_t v = wl[i];
    const int64_t ib = irp[v], ie = irp[v + 1], ob = orp ? orp[v] : 0, oe = orp ? orp[v + 1] : 0;
    const int64_t dv = (ie - ib) + (oe - ob);
    const uint64_t pv = prio(dv, v);
    const int cv = color[v];
    bool lost = false;
    for (int64_t k = ib + lane; k < ie && !lost; k += 32) {
      const int32_t u = icol[k];
      if (color[u] == cv) {
        const int64_t du = (irp[u + 1] - irp[u]) + (orp ? orp[u + 1] - orp[u] : 0);
        if (prio(du, u) > pv) lost = true;
      }
    }
    for (int64_t k = ob + lane; k < oe && !lost; k += 32) {
      const int32_t u = ocol[k];
      if (color[u] == cv) {
        const int64_t du = (irp[u + 1] - irp[u]) + (orp[u + 1] - orp[u]);
        if (prio(du, u) > pv) lost = true;
      }
    }
    lost = __any_sync(0xffffffffu, lost);
    if (lane == 0) {
      if (lost) next[atomicAdd(nnext, 1ull)] = v;
      else atomicMax(maxc, cv);
    }
  }
}

__global__ void k_mark(int64_t nw, const int32_t *__restrict__ wl, int round,
                       int32_t *__restrict__ mark) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nw) mark[wl[i]] = round;
}

__global__ void k_iota32(int64_t n, int32_t *__restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}

// degree bucket key (largest first): 40 − floor(log2(symmetrised degree + 1))
__global__ void k_deg_bucket(int64_t n, const int64_t *__restrict__ irp,
                             const int64_t *__restrict__ orp, uint32_t *__restrict__ key,
                             int32_t *__restrict__ id) {
  const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int64_t d = (irp[v + 1] - irp[v]) + (orp ? orp[v + 1] - orp[v] : 0);
  key[v] = 40u - (uint32_t)(63 - __clzll((unsigned long long)d + 1ull));
  id[v] = (int32_t)v;
}

// speculative coloring into `color` (−1 initialised); returns the color count
static fj_status spec_coloring(fj_graph *g, Workspace &ws, const int64_t *orp, const int32_t *ocol,
                               int32_t *color, int *ncolors, int *rounds_out) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  int32_t *wa = nullptr, *wb = nullptr;
  unsigned long long *cnt = nullptr;
  int *maxc = nullptr;
  FJ_CUDA(ws.alloc(&wa, (size_t)n));
  FJ_CUDA(ws.alloc(&wb, (size_t)n));
  FJ_CUDA(ws.alloc(&cnt, 1));
  FJ_CUDA(ws.alloc(&maxc, 1));
  FJ_CUDA(cudaMemsetAsync(maxc, 0, sizeof(int), st));
  // largest-first by degree buckets (powers of two): the hubs of a power-law
  // graph take the low colors first, as in sequential largest-first greedy,
  // and every bucket is colored speculatively in a few rounds
  int32_t *mark = nullptr;  // round stamp of the current worklist members
  FJ_CUDA(ws.alloc(&mark, (size_t)n));
  FJ_CUDA(cudaMemsetAsync(mark, 0xff, sizeof(int32_t) * n, st));
  uint32_t *k0 = nullptr, *k1 = nullptr;
  int32_t *ord = nullptr;
  FJ_CUDA(ws.alloc(&k0, (size_t)n));
  FJ_CUDA(ws.alloc(&k1, (size_t)n));
  FJ_CUDA(ws.alloc(&ord, (size_t)n));
  fj::count_launch();
  k_deg_bucket<<<(unsigned)((n + kBlock - 1) / kBlock), kBlock, 0, st>>>(n, g->in_rp, orp, k0, wb);
  // stable sort by bucket (prims.cu); the sorted ids end in `ord`, `wb` is free again
  FJ_TRY((radix_sort_pairs<uint32_t, int32_t>(k0, k1, wb, ord, n, 6, ws)));
  std::swap(ord, wb);
  std::vector<uint32_t> hk((size_t)n);
  FJ_CUDA(cudaMemcpyAsync(hk.data(), k0, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  std::vector<int64_t> seg;  // bucket boundaries in the sorted order
  seg.push_back(0);
  for (int64_t i = 1; i < n; i++)
    if (hk[i] != hk[i - 1]) seg.push_back(i);
  seg.push_back(n);
  int rounds = 0;
  for (size_t bi = 0; bi + 1 < seg.size(); bi++) {
  const int64_t nb0 = seg[bi], nb1 = seg[bi + 1];
  FJ_CUDA(cudaMemcpyAsync(wa, ord + nb0, sizeof(int32_t) * (nb1 - nb0), cudaMemcpyDeviceToDevice,
                          st));
  int64_t nw = nb1 - nb0;
  while (nw > 0) {
    const unsigned blocks = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((nw * 32 + kBlock - 1) / kBlock, (int64_t)g->num_sms * 64));
    FJ_CUDA(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), st));
    fj::count_launch();
    k_mark<<<(unsigned)((nw + kBlock - 1) / kBlock), kBlock, 0, st>>>(nw, wa, rounds, mark);
    fj::count_launch();
    k_spec_assign<<<blocks, kBlock, 0, st>>>(nw, wa, g->in_rp, g->in_col, orp, ocol, mark, rounds,
                                             color);
    fj::count_launch();
    k_spec_detect<<<blocks, kBlock, 0, st>>>(nw, wa, g->in_rp, g->in_col, orp, ocol, color, wb, cnt,
                                             maxc);
    unsigned long long h = 0;
    FJ_CUDA(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    nw = (int64_t)h;
    std::swap(wa, wb);
    if (++rounds > 100000) {
      set_error("coloring did not terminate");
      return FJ_ERR_CUDA;
    }
  }
  }
  int hmax = 0;
  FJ_CUDA(cudaMemcpyAsync(&hmax, maxc, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  *ncolors = hmax + 1;
  *rounds_out = rounds;
  return FJ_OK;
}

fj_status build_coloring(fj_graph *g, const fj_opts *o) {
  const double frac = o->tail_frac < 0 ? 0.01 : o->tail_frac;
  const int algo = o->coloring == 1 ? 1 : 0;
  if (g->colors && g->color_tail_frac == frac && g->color_algo == algo) return FJ_OK;
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  if (g->colors) {  // other options: drop the old coloring and its layouts
    cudaFreeAsync(g->colors, st);
    g->colors = nullptr;
    g->color_layout.release(st);
    g->push_color_layout.release(st);
  }
  g->color_tail_frac = frac;
  g->color_algo = algo;
  Workspace ws(st);  // the pull CSR and the round buffers; the colors go to g
  // the pull CSR: for an undirected graph it IS the canonical in-CSR (graph
  // create checked the symmetry), so only directed graphs transpose again
  const int64_t *ort = g->in_rp;
  const int32_t *ocol = g->in_col;
  const float *ow = g->in_w;
  if (g->directed) {
    int64_t *t_rp = nullptr;
    int32_t *t_col = nullptr;
    float *t_w = nullptr;
    FJ_TRY(transpose_in_csr(g, ws, &t_rp, &t_col, &t_w));
    ort = t_rp;
    ocol = t_col;
    ow = t_w;
  }
  const bool jp = algo == 1;
  if (!jp) {
    int32_t *cs = nullptr;
    FJ_CUDA(ws.alloc(&cs, (size_t)n));
    FJ_CUDA(cudaMemsetAsync(cs, 0xff, sizeof(int32_t) * n, st));
    int nc = 0, rounds = 0;
    // undirected: the in-CSR already holds both directions of every edge
    FJ_TRY(spec_coloring(g, ws, g->directed ? ort : nullptr, g->directed ? ocol : nullptr, cs, &nc,
                         &rounds));
#ifdef FJ_DIAG
    fprintf(stderr, "fj coloring: %d speculative rounds, %d colors\n", rounds, nc);
#endif
    ws.keep(cs);
    g->ncolors = nc;
    g->colors = cs;
    FJ_TRY(merge_tail_colors(g, frac));
    fj_status s = build_layout_from_out(g, ort, ocol, ow, g->colors, g->ncolors, &g->color_layout, false, true);
    if (s == FJ_OK) s = tail_bounds(g, &g->color_layout);
    FJ_CUDA(cudaStreamSynchronize(st));
    return s;
  }
  int32_t *c0 = nullptr, *c1 = nullptr;
  unsigned long long *rem = nullptr;
  int *maxc = nullptr;
  FJ_CUDA(ws.alloc(&c0, (size_t)n));
  FJ_CUDA(ws.alloc(&c1, (size_t)n));
  FJ_CUDA(ws.alloc(&rem, 1));
  FJ_CUDA(ws.alloc(&maxc, 1));
  FJ_CUDA(cudaMemsetAsync(c0, 0xff, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMemsetAsync(c1, 0xff, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMemsetAsync(maxc, 0, sizeof(int), st));
  int64_t blocks = std::min<int64_t>((n * 32 + kBlock - 1) / kBlock, (int64_t)g->num_sms * 64);
  unsigned long long left = 1;
  int rounds = 0;
  while (left > 0) {
    FJ_CUDA(cudaMemsetAsync(rem, 0, sizeof(unsigned long long), st));
    fj::count_launch();
    k_jp_round<<<(unsigned)blocks, kBlock, 0, st>>>(n, g->in_rp, g->in_col, ort, ocol, c0, c1, rem,
                                                    maxc);
    FJ_CUDA(cudaMemcpyAsync(c0, c1, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
    FJ_CUDA(cudaMemcpyAsync(&left, rem, sizeof(left), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
#ifdef FJ_DIAG
    if (rounds < 64 || rounds % 100 == 0) fprintf(stderr, "fj JP round %d: %llu vertices left\n", rounds, left);
#endif
    if (++rounds > 1000000) {
      set_error("coloring did not terminate");
      return FJ_ERR_CUDA;
    }
  }
#ifdef FJ_DIAG
  fprintf(stderr, "fj coloring: %d JP rounds\n", rounds);
#endif
  int hmax = 0;
  FJ_CUDA(cudaMemcpyAsync(&hmax, maxc, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  ws.keep(c0);
  g->ncolors = hmax + 1;
  g->colors = c0;
  FJ_TRY(merge_tail_colors(g, frac));
  fj_status s = build_layout_from_out(g, ort, ocol, ow, g->colors, g->ncolors, &g->color_layout, false, true);
  if (s == FJ_OK) s = tail_bounds(g, &g->color_layout);
  FJ_CUDA(cudaStreamSynchronize(st));
  return s;
}

}  // namespace fj
