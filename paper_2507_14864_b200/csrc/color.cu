// color.cu — distance-1 coloring of the symmetrised graph (§8 row a1, K4),
// built lazily for the COLORED (multicolor SOR) schedule.
//
// Rows of one color share no arc in either direction, so relaxing them
// simultaneously equals relaxing them one after another: a colored sweep is a
// sequential SOR sweep in (color, id) order, which is what Theorem 3
// and the SOR derivation assume.
//
// Algorithm: Jones–Plassmann with first-fit colors.  Priority = (symmetrised
// degree, hash(id)); in each round every uncolored vertex whose priority
// exceeds that of all its uncolored neighbours takes the smallest color
// absent from its colored neighbours.  Two adjacent vertices are never both
// local maxima, so rounds never conflict; colors are read from the previous
// round's array (double buffering).
#include <cub/cub.cuh>

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

fj_status build_coloring(fj_graph *g) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n;
  int64_t *ort = nullptr;
  int32_t *ocol = nullptr;
  float *ow = nullptr;
  FJ_TRY(transpose_in_csr(g, &ort, &ocol, &ow));
  int32_t *c0 = nullptr, *c1 = nullptr;
  unsigned long long *rem = nullptr;
  int *maxc = nullptr;
  FJ_CUDA(cudaMallocAsync(&c0, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&c1, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&rem, sizeof(unsigned long long), st));
  FJ_CUDA(cudaMallocAsync(&maxc, sizeof(int), st));
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
    if (++rounds > 1000000) {
      set_error("coloring did not terminate");
      return FJ_ERR_CUDA;
    }
  }
  int hmax = 0;
  FJ_CUDA(cudaMemcpyAsync(&hmax, maxc, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  g->ncolors = hmax + 1;
  g->colors = c0;
  cudaFreeAsync(c1, st);
  cudaFreeAsync(rem, st);
  cudaFreeAsync(maxc, st);
  fj_status s = build_layout_from_out(g, ort, ocol, ow, g->colors, g->ncolors, &g->color_layout);
  cudaFreeAsync(ort, st);
  cudaFreeAsync(ocol, st);
  if (ow) cudaFreeAsync(ow, st);
  FJ_CUDA(cudaStreamSynchronize(st));
  return s;
}

}  // namespace fj
