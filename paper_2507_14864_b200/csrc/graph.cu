// graph.cu — fj_graph_create / fj_graph_destroy (§8 row a1).
//
// Steps (all on the graph's stream):
//   1. stage the caller's in-CSR into library-owned device memory;
//   2. validate row_ptr (FJ_ERR_INVALID on failure);
//   3. transpose to the pull (out-) CSR with a stable radix sort on u whose
//      payload is the out-CSR entry itself (v, or v | weight bits; arc
//      indices only while host weights are still being copied); the keys
//      pass validates columns (range, self-loops), weights, and notes rows
//      that are not strictly increasing;
//   4. only then, canonicalise the in-CSR (rows sorted by column) with a radix
//      sort of (v, u) keys; adjacent equal keys are duplicate arcs;
//   5. d_u = Σ_v a_uv over the out-rows in fp64, deterministic order (P:78,
//      reading R3);
//   6. undirected input: check the arc set is symmetric with equal weights;
//   7. build the sweep layout (layout.cu).
// Sorting and scans use CUB (toolkit library primitives); every kernel here
// is a one-pass O(m) integer/fp64 kernel.
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include <algorithm>

#include <nvtx3/nvToolsExt.h>

#include "fj_internal.cuh"

namespace fj {

static int bits_for(int64_t n) {
  int b = 1;
  while ((int64_t(1) << b) < n) b++;
  return b;
}

// ---------------------------------------------------------------- kernels
__global__ void k_validate_rowptr(int64_t n, int64_t m, const int64_t *__restrict__ rp,
                                  int *__restrict__ err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  int64_t x = rp[i];
  if (i == 0 && x != 0) atomicOr(err, 1);
  if (i == n && x != m) atomicOr(err, 1);
  if (i < n && rp[i + 1] < x) atomicOr(err, 1);
  if (x < 0 || x > m) atomicOr(err, 1);
}

// (v, u) keys of the in-CSR arcs (only when rows must be sorted)
__global__ void k_in_keys(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                          int nb, uint64_t *__restrict__ keys) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t v = warp; v < n; v += nwarps)
    for (int64_t e = rp[v] + lane; e < rp[v + 1]; e += 32)
      keys[e] = ((uint64_t)v << nb) | (uint64_t)col[e];
}

__global__ void k_iota_u32(int64_t m, uint32_t *__restrict__ x) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) x[i] = (uint32_t)i;
}

// after sorting: duplicates; split keys into (row, col); permute weights
__global__ void k_unpack_sorted(int64_t m, int nb, const uint64_t *__restrict__ keys,
                                const uint32_t *__restrict__ idx, const float *__restrict__ w_src,
                                int32_t *__restrict__ col, float *__restrict__ w_dst,
                                int *__restrict__ err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  uint64_t k = keys[i];
  if (i > 0 && keys[i - 1] == k) atomicOr(err, 16);
  col[i] = (int32_t)(k & ((uint64_t(1) << nb) - 1));
  if (w_dst) w_dst[i] = w_src[idx[i]];
}

// Transpose inputs, one pass over the in-CSR that also validates the
// caller's columns — range (bit 2), self-loop (4), rows not strictly
// increasing (64: not canonical) and, packed with weights, the weight (8).
//   KIdx:  key u, payload arc index e, row v of every arc (host weights still
//          in flight: they are gathered by index after the sort);
//   KV32:  key u, payload v (unweighted: the sorted payload is the out-CSR);
//   KV64:  key u, payload v | bits(w) << 32 (weights on the device).
// Chunked: a warp walks the concatenated arcs of 32 consecutive rows (all
// lanes busy for short rows); chunks above kChunkArcs arcs are cut into
// pieces for k_out_keys_long (hub rows spread over many warps).
enum KeyMode { KIdx = 0, KV32 = 1, KV64 = 2 };
struct KeyOut {
  uint32_t *key, *idx, *row, *v32;
  uint64_t *v64;
};

template <int KM>
__device__ __forceinline__ void keys_walk(int64_t n, int64_t i0, int nr, int64_t my_rp,
                                          int64_t k0, int64_t k1, const int32_t *__restrict__ col,
                                          const float *__restrict__ w, KeyOut o, int *err) {
  const int lane = threadIdx.x & 31;
  int bad = 0;
  for (int64_t k = k0 + lane; k - lane < k1; k += 32) {
    const int r = chunk_row_of(nr, my_rp, k);
    const int64_t rs = __shfl_sync(0xffffffffu, my_rp, r);
    if (k >= k1) continue;
    const int64_t v = i0 + r;
    const int32_t u = col[k];
    if (err) {
      if (u < 0 || u >= n) bad |= 2;
      if (u == v) bad |= 4;
      if (k > rs && col[k - 1] >= u) bad |= 64;
    }
    o.key[k] = (u >= 0 && u < n) ? (uint32_t)u : 0u;
    if constexpr (KM == KIdx) {
      o.idx[k] = (uint32_t)k;
      o.row[k] = (uint32_t)v;
    } else if constexpr (KM == KV32) {
      o.v32[k] = (uint32_t)v;
    } else {
      const float x = w[k];
      if (err && !(x > 0.0f && isfinite(x))) bad |= 8;
      o.v64[k] = (uint64_t)(uint32_t)v | ((uint64_t)__float_as_uint(x) << 32);
    }
  }
  if (err) {
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(err, bad);
  }
}

template <int KM>
__global__ void k_out_keys(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                           const float *__restrict__ w, KeyOut o, int *err, unsigned *long_cnt,
                           int2 *long_list) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i0 = warp * 32; i0 < n; i0 += nwarps * 32) {
    const int nr = (int)(n - i0 < 32 ? n - i0 : 32);
    const int64_t my_rp = lane < nr ? rp[i0 + lane] : 0;
    const int64_t a0 = __shfl_sync(0xffffffffu, my_rp, 0);
    const int64_t a1 = rp[i0 + nr];
    if (a1 - a0 > kChunkArcs) {
      const int np = (int)((a1 - a0 + kChunkArcs - 1) / kChunkArcs);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(long_cnt, (unsigned)np);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int q = lane; q < np; q += 32) long_list[base + q] = make_int2((int)(i0 >> 5), q);
      continue;
    }
    keys_walk<KM>(n, i0, nr, my_rp, a0, a1, col, w, o, err);
  }
}

template <int KM>
__global__ void k_out_keys_long(int64_t n, const int64_t *__restrict__ rp,
                                const int32_t *__restrict__ col, const float *__restrict__ w,
                                KeyOut o, int *err, const unsigned *long_cnt,
                                const int2 *long_list) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int64_t items = (int64_t)*long_cnt;
  for (int64_t it = warp; it < items; it += nwarps) {
    const int2 pc = long_list[it];
    const int64_t i0 = 32 * (int64_t)pc.x;
    const int nr = (int)(n - i0 < 32 ? n - i0 : 32);
    const int64_t my_rp = lane < nr ? rp[i0 + lane] : 0;
    const int64_t a0 = __shfl_sync(0xffffffffu, my_rp, 0);
    const int64_t a1 = rp[i0 + nr];
    const int64_t k0 = a0 + (int64_t)pc.y * kChunkArcs;
    const int64_t k1 = k0 + kChunkArcs < a1 ? k0 + kChunkArcs : a1;
    keys_walk<KM>(n, i0, nr, my_rp, k0, k1, col, w, o, err);
  }
}

__global__ void k_out_unpack(int64_t m, const uint64_t *__restrict__ v64, int32_t *__restrict__ ocol,
                             float *__restrict__ ow) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t x = v64[k];
  ocol[k] = (int32_t)(uint32_t)x;
  ow[k] = __uint_as_float((uint32_t)(x >> 32));
}

// row pointers of the out-CSR from the sorted keys (no atomics): ort[u] is
// the first position whose key is >= u (binary search)
__global__ void k_bounds(int64_t n, int64_t m, const uint32_t *__restrict__ key,
                         int64_t *__restrict__ ort) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (u > n) return;
  int64_t lo = 0, hi = m;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)key[mid] < u) lo = mid + 1;
    else hi = mid;
  }
  ort[u] = lo;
}

// out-CSR entries from the stably sorted arc indices (v ascending within u)
__global__ void k_out_fill(int64_t m, const uint32_t *__restrict__ idx, const uint32_t *__restrict__ row,
                           const float *__restrict__ w, int32_t *__restrict__ ocol,
                           float *__restrict__ ow, int *__restrict__ err) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint32_t e = idx[k];
  ocol[k] = (int32_t)row[e];
  if (ow) {
    const float x = w[e];
    ow[k] = x;
    if (err && !(x > 0.0f && isfinite(x))) atomicOr(err, 8);  // weight validity
  }
}

// d_u = Σ_v a_uv over the out-rows, fp64, deterministic (the order of
// the additions depends only on the graph).  Unweighted: d_u = row length.
// Weighted, chunked like the transpose: a warp walks the arcs of 32
// consecutive rows 32 at a time; a segmented lane scan sums each row's arcs
// of the step and the row's owner lane adds its segment total.  Chunks above
// kChunkArcs arcs go to k_row_sums_long (a warp per row, lane-strided sums
// and a fixed shuffle tree).
__global__ void k_row_sums(int64_t n, const int64_t *__restrict__ rp, const float *__restrict__ w,
                           double *__restrict__ d, unsigned *__restrict__ long_cnt,
                           int32_t *__restrict__ long_list) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i0 = warp * 32; i0 < n; i0 += nwarps * 32) {
    const int nr = (int)(n - i0 < 32 ? n - i0 : 32);
    int64_t my_b = 0, my_e = 0;
    if (lane < nr) {
      my_b = rp[i0 + lane];
      my_e = rp[i0 + lane + 1];
    }
    if (!w) {
      if (lane < nr) d[i0 + lane] = (double)(my_e - my_b);
      continue;
    }
    const int64_t a0 = __shfl_sync(0xffffffffu, my_b, 0);
    const int64_t a1 = __shfl_sync(0xffffffffu, my_e, nr - 1);
    if (a1 - a0 > kChunkArcs) {
      if (lane == 0) long_list[atomicAdd(long_cnt, 1u)] = (int32_t)(i0 >> 5);
      continue;
    }
    double acc = 0.0;
    for (int64_t base = a0; base < a1; base += 32) {
      const int64_t k = base + lane;
      const int r = chunk_row_of(nr, my_b, k);
      double v = k < a1 ? (double)w[k] : 0.0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {  // segmented inclusive scan by row
        const double y = __shfl_up_sync(0xffffffffu, v, off);
        const int ry = __shfl_up_sync(0xffffffffu, r, off);
        if (lane >= off && ry == r) v += y;
      }
      const int64_t hi = my_e < base + 32 ? my_e : base + 32;  // my row ∩ this step
      const int64_t lo = my_b > base ? my_b : base;
      const bool has = lane < nr && hi > lo;
      const double seg = __shfl_sync(0xffffffffu, v, has ? (int)(hi - 1 - base) : 0);
      if (has) acc += seg;
    }
    if (lane < nr) d[i0 + lane] = acc;
  }
}

__global__ void k_row_sums_long(int64_t n, const int64_t *__restrict__ rp,
                                const float *__restrict__ w, double *__restrict__ d,
                                const unsigned *__restrict__ long_cnt,
                                const int32_t *__restrict__ long_list) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int64_t items = 32 * (int64_t)*long_cnt;
  for (int64_t it = warp; it < items; it += nwarps) {
    const int64_t u = 32 * (int64_t)long_list[it >> 5] + (it & 31);
    if (u >= n) continue;
    const int64_t b = rp[u], e = rp[u + 1];
    double s = 0.0;
    for (int64_t k = b + lane; k < e; k += 32) s += (double)w[k];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) d[u] = s;
  }
}

template <class T>
__global__ void k_neq(int64_t m, const T *__restrict__ a, const T *__restrict__ b,
                      int *__restrict__ err, int bit) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m && a[i] != b[i]) atomicOr(err, bit);
}

static unsigned grid_for(int64_t work, int per_block = kBlock) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > (1 << 30)) b = 1 << 30;
  return (unsigned)b;
}

static unsigned grid_warps(int64_t rows) {  // warp-per-row kernels: grid-stride
  int64_t b = (rows * 32 + kBlock - 1) / kBlock;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

template <class K, class V>
static fj_status sort_pairs(K *&keys, K *&keys_alt, V *&val, V *&val_alt, int64_t m, int nbits,
                            Workspace &ws) {
  return radix_sort_pairs<K, V>(keys, keys_alt, val, val_alt, m, nbits, ws);  // prims.cu (stable LSD)
}

template <int KM>
static fj_status launch_out_keys(fj_graph *g, Workspace &tmp, const float *w, KeyOut o, int *err) {
  const int64_t n = g->n, m = g->m;
  cudaStream_t st = g->stream;
  unsigned *long_cnt = nullptr;
  int2 *long_list = nullptr;
  FJ_CUDA(tmp.alloc(&long_cnt, 1));
  FJ_CUDA(tmp.alloc(&long_list, (size_t)(m / kChunkArcs + n / 32 + 2)));
  FJ_CUDA(cudaMemsetAsync(long_cnt, 0, sizeof(unsigned), st));
  fj::count_launch();
  k_out_keys<KM><<<grid_for(n), kBlock, 0, st>>>(n, g->in_rp, g->in_col, w, o, err, long_cnt,
                                                 long_list);
  fj::count_launch();
  k_out_keys_long<KM><<<g->num_sms * 8, kBlock, 0, st>>>(n, g->in_rp, g->in_col, w, o, err,
                                                         long_cnt, long_list);
  return FJ_OK;
}

// Transpose the canonical in-CSR into the pull CSR (row u lists v with a_uv),
// rows sorted: a stable radix sort on u alone keeps the v order of the
// canonical input.  *ort, *ocol, *ow live in the caller's workspace `ws`.
fj_status transpose_in_csr(fj_graph *g, Workspace &ws, int64_t **ort, int32_t **ocol, float **ow,
                           int *err) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n, m = g->m;
  Workspace tmp(st);  // sort keys and payloads
  uint32_t *k0 = nullptr, *k1 = nullptr, *i0 = nullptr, *i1 = nullptr, *row = nullptr;
  FJ_CUDA(tmp.alloc(&k0, (size_t)m + 1));
  FJ_CUDA(tmp.alloc(&k1, (size_t)m + 1));
  FJ_CUDA(ws.alloc(ort, (size_t)n + 1));
  FJ_CUDA(ws.alloc(ocol, (size_t)m + 8));
  *ow = nullptr;
  if (g->in_w) FJ_CUDA(ws.alloc(ow, (size_t)m + 8));
  if (!g->w_ready) {
    // weights (if any) are on the device already: sort the out-CSR payload
    // itself (radix passes move 8 or 12 bytes per arc, every access coalesced)
    if (g->in_w) {
      uint64_t *p0 = nullptr, *p1 = nullptr;
      FJ_CUDA(tmp.alloc(&p0, (size_t)m + 1));
      FJ_CUDA(tmp.alloc(&p1, (size_t)m + 1));
      KeyOut o{k0, nullptr, nullptr, nullptr, p0};
      FJ_TRY(launch_out_keys<KV64>(g, tmp, g->in_w, o, err));
      FJ_TRY(sort_pairs(k0, k1, p0, p1, m, bits_for(n), tmp));
      if (m > 0) {
        fj::count_launch();
        k_out_unpack<<<grid_for(m), kBlock, 0, st>>>(m, p0, *ocol, *ow);
      }
    } else {
      uint32_t *v0 = nullptr, *v1 = reinterpret_cast<uint32_t *>(*ocol);
      FJ_CUDA(tmp.alloc(&v0, (size_t)m + 1));
      KeyOut o{k0, nullptr, nullptr, v0, nullptr};
      FJ_TRY(launch_out_keys<KV32>(g, tmp, nullptr, o, err));
      FJ_TRY(sort_pairs(k0, k1, v0, v1, m, bits_for(n), tmp));
      if (m > 0 && v0 != reinterpret_cast<uint32_t *>(*ocol))
        FJ_CUDA(cudaMemcpyAsync(*ocol, v0, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, st));
    }
    fj::count_launch();
    k_bounds<<<grid_for(n + 1), kBlock, 0, st>>>(n, m, k0, *ort);
    FJ_CUDA(cudaGetLastError());
    return FJ_OK;
  }
  // host weights still in flight on the side stream: sort arc indices now and
  // gather the weights once they have landed
  FJ_CUDA(tmp.alloc(&i0, (size_t)m + 1));
  FJ_CUDA(tmp.alloc(&i1, (size_t)m + 1));
  FJ_CUDA(tmp.alloc(&row, (size_t)m + 1));
  {
    KeyOut o{k0, i0, row, nullptr, nullptr};
    FJ_TRY(launch_out_keys<KIdx>(g, tmp, nullptr, o, err));
  }
  FJ_TRY(sort_pairs(k0, k1, i0, i1, m, bits_for(n), tmp));
  if (m > 0) {
    if (g->w_ready) FJ_CUDA(cudaStreamWaitEvent(st, g->w_ready, 0));  // weights staged
    fj::count_launch();
    k_out_fill<<<grid_for(m), kBlock, 0, st>>>(m, i0, row, g->in_w, *ocol, *ow, err);
  }
  fj::count_launch();
  k_bounds<<<grid_for(n + 1), kBlock, 0, st>>>(n, m, k0, *ort);
  FJ_CUDA(cudaGetLastError());
  return FJ_OK;
}

static double wall() {
  timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec + 1e-9 * t.tv_nsec;
}

static fj_status create_impl(int64_t n, int64_t nnz, const int64_t *rp_in, const int32_t *col_in,
                             const float *w_in, int directed, cudaStream_t st, fj_graph *g) {
#ifdef FJ_DIAG
  const bool dbg = true;   // diagnostic build: phase timings on stderr
#else
  const bool dbg = false;
#endif
  double t0 = wall();
  auto mark = [&](const char *what) {
    if (!dbg) return;
    cudaStreamSynchronize(st);
    double t1 = wall();
    fprintf(stderr, "fj create %-28s %8.2f ms\n", what, 1e3 * (t1 - t0));
    t0 = t1;
  };
  g->n = n;
  g->m = nnz;
  g->directed = directed ? 1 : 0;
  g->weighted = w_in ? 1 : 0;
  g->stream = st;
  int dev = 0;
  FJ_CUDA(cudaGetDevice(&dev));
  FJ_CUDA(cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, dev));
  {
    // keep stream-ordered allocations in the pool between calls (graphs and
    // solve workspaces are re-created per call; re-mapping GBs is slow)
    cudaMemPool_t pool;
    FJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    FJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  const int64_t m = nnz;
  const int nb = bits_for(n);

  // 1. stage into library-owned memory (padded: the sweep reads in 16-byte units)
  mark("setup");
  FJ_CUDA(cudaMallocAsync(&g->in_rp, sizeof(int64_t) * (n + 1), st));
  FJ_CUDA(cudaMallocAsync(&g->in_col, sizeof(int32_t) * (m + 8), st));
  if (w_in) FJ_CUDA(cudaMallocAsync(&g->in_w, sizeof(float) * (m + 8), st));
  mark("alloc");
  FJ_CUDA(cudaMemcpyAsync(g->in_rp, rp_in, sizeof(int64_t) * (n + 1), cudaMemcpyDefault, st));
  // host weights travel on a side stream: the copy engine moves them while the
  // column checks, keys and sort of the transpose run (it waits only before
  // the weights are first read)
  cudaStream_t wst = nullptr;
  struct SideStream {
    cudaStream_t &s;
    cudaEvent_t &e;
    ~SideStream() {  // also on early error returns: the copy must not outlive in_w
      if (s) cudaStreamSynchronize(s);
      if (e) cudaEventDestroy(e);
      if (s) cudaStreamDestroy(s);
      e = nullptr;
    }
  } side{wst, g->w_ready};
  if (m > 0) {
    FJ_CUDA(cudaMemcpyAsync(g->in_col, col_in, sizeof(int32_t) * m, cudaMemcpyDefault, st));
    if (w_in && !is_device_ptr(w_in)) {
      FJ_CUDA(cudaStreamCreateWithFlags(&wst, cudaStreamNonBlocking));
      FJ_CUDA(cudaEventCreateWithFlags(&g->w_ready, cudaEventDisableTiming));
      cudaEvent_t staged;  // the buffer exists on st before the side copy starts
      FJ_CUDA(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
      FJ_CUDA(cudaEventRecord(staged, st));
      FJ_CUDA(cudaStreamWaitEvent(wst, staged, 0));
      cudaEventDestroy(staged);
      FJ_CUDA(cudaMemcpyAsync(g->in_w, w_in, sizeof(float) * m, cudaMemcpyDefault, wst));
      FJ_CUDA(cudaEventRecord(g->w_ready, wst));
    } else if (w_in) {
      FJ_CUDA(cudaMemcpyAsync(g->in_w, w_in, sizeof(float) * m, cudaMemcpyDefault, st));
    }
  }
  mark("stage");

  // 2. validate
  Workspace ws(st);  // temporaries of the build; the graph owns the rest
  int *err = nullptr;
  int herr = 0;
  FJ_CUDA(ws.alloc(&err, 1));
  FJ_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  fj::count_launch();
  k_validate_rowptr<<<grid_for(n + 1), kBlock, 0, st>>>(n, m, g->in_rp, err);
  FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  if (herr) {
    set_error("fj_graph_create: in_row_ptr must start at 0, be non-decreasing and end at nnz");
    return FJ_ERR_INVALID;
  }
  mark("validate row_ptr");

  // 3. pull CSR; the transpose pass also validates columns and weights.  Its
  // result does not depend on the order inside the caller's rows (stable sort
  // on u with the arc index as payload), so unsorted input only needs the
  // in-CSR itself canonicalised below
  int64_t *ort = nullptr;
  int32_t *ocol = nullptr;
  float *ow = nullptr;
  FJ_TRY(transpose_in_csr(g, ws, &ort, &ocol, &ow, err));
  FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  mark("transpose + validate");

  // 4. canonical in-CSR: sort rows only if some row is not strictly increasing
  if ((herr & ~64) == 0 && (herr & 64)) {
    uint64_t *k0 = nullptr, *k1 = nullptr;
    uint32_t *i0 = nullptr, *i1 = nullptr;
    int32_t *col_raw = nullptr;
    float *w_raw = nullptr;
    Workspace sw(st);  // sort temporaries
    FJ_CUDA(sw.alloc(&k0, (size_t)m + 1));
    FJ_CUDA(sw.alloc(&k1, (size_t)m + 1));
    FJ_CUDA(sw.alloc(&i0, (size_t)m + 1));
    FJ_CUDA(sw.alloc(&i1, (size_t)m + 1));
    FJ_CUDA(sw.alloc(&col_raw, (size_t)m + 1));
    FJ_CUDA(cudaMemcpyAsync(col_raw, g->in_col, sizeof(int32_t) * m, cudaMemcpyDeviceToDevice, st));
    if (w_in) {
      FJ_CUDA(sw.alloc(&w_raw, (size_t)m + 1));
      FJ_CUDA(cudaMemcpyAsync(w_raw, g->in_w, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
    }
    fj::count_launch();
    k_in_keys<<<grid_warps(n), kBlock, 0, st>>>(n, g->in_rp, col_raw, nb, k0);
    fj::count_launch();
    k_iota_u32<<<grid_for(m), kBlock, 0, st>>>(m, i0);
    FJ_TRY(sort_pairs(k0, k1, i0, i1, m, 2 * nb, sw));
    FJ_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    fj::count_launch();
    k_unpack_sorted<<<grid_for(m), kBlock, 0, st>>>(m, nb, k0, i0, w_raw, g->in_col, g->in_w, err);
    FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    mark("canonicalise (sort)");
  }
  FJ_CUDA(cudaGetLastError());
  if (herr & ~64) {
    set_error("fj_graph_create: %s%s%s%s",
              herr & 2 ? "column index out of range; " : "", herr & 4 ? "self-loop; " : "",
              herr & 8 ? "weight not positive and finite; " : "",
              herr & 16 ? "duplicate arc; " : "");
    return FJ_ERR_INVALID;
  }

  // 5. degrees
  FJ_CUDA(cudaMallocAsync(&g->deg, sizeof(double) * n, st));
  {
    unsigned *long_cnt = nullptr;
    int32_t *long_list = nullptr;
    FJ_CUDA(ws.alloc(&long_cnt, 1));
    FJ_CUDA(ws.alloc(&long_list, (size_t)(n / 32 + 1)));
    FJ_CUDA(cudaMemsetAsync(long_cnt, 0, sizeof(unsigned), st));
    fj::count_launch();
    k_row_sums<<<grid_for(n), kBlock, 0, st>>>(n, ort, ow, g->deg, long_cnt, long_list);
    if (ow) {
      fj::count_launch();
      k_row_sums_long<<<g->num_sms * 8, kBlock, 0, st>>>(n, ort, ow, g->deg, long_cnt, long_list);
    }
  }
  mark("degrees");

  // 6. symmetry of undirected input
  if (!g->directed && m > 0) {
    fj::count_launch();
    k_neq<int64_t><<<grid_for(n + 1), kBlock, 0, st>>>(n + 1, ort, g->in_rp, err, 32);
    fj::count_launch();
    k_neq<int32_t><<<grid_for(m), kBlock, 0, st>>>(m, ocol, g->in_col, err, 32);
    if (ow) {
      fj::count_launch();
      k_neq<float><<<grid_for(m), kBlock, 0, st>>>(m, ow, g->in_w, err, 32);
    }
    FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    if (herr) {
      set_error("fj_graph_create: directed = 0 but the arc set is not symmetric with equal weights");
      return FJ_ERR_INVALID;
    }
    mark("symmetry check");
  }

  // 7. sweep layout (1 color)
  fj_status s = build_layout_from_out(g, ort, ocol, ow, nullptr, 1, &g->async_layout, false, true);
  if (s != FJ_OK) return s;
  FJ_CUDA(cudaStreamSynchronize(st));
  FJ_CUDA(cudaGetLastError());
  mark("layout");
  return FJ_OK;
}

}  // namespace fj

extern "C" {

fj_status fj_graph_create(int64_t n, int64_t nnz, const int64_t *in_row_ptr, const int32_t *in_col,
                          const float *in_w, int directed, void *cuda_stream, fj_graph_t *out) {
  if (!out) {
    fj::set_error("fj_graph_create: out is NULL");
    return FJ_ERR_INVALID;
  }
  *out = nullptr;
  if (n < 1 || n >= (int64_t(1) << 31) || nnz < 0 || nnz >= (int64_t(1) << 40) || !in_row_ptr ||
      (nnz > 0 && !in_col)) {
    fj::set_error("fj_graph_create: need 1 <= n < 2^31, nnz >= 0, non-null row_ptr/col");
    return FJ_ERR_INVALID;
  }
  fj_graph *g = new fj_graph();
  nvtxRangePushA("fj_graph_create");
  fj_status s = fj::create_impl(n, nnz, in_row_ptr, in_col, in_w, directed,
                                (cudaStream_t)cuda_stream, g);
  nvtxRangePop();
  if (s != FJ_OK) {
    fj_graph_destroy(g);
    return s;
  }
  *out = g;
  return FJ_OK;
}

fj_status fj_graph_destroy(fj_graph_t g) {
  if (!g) return FJ_OK;
  cudaStreamSynchronize(g->stream);
  for (void *q : {(void *)g->in_rp, (void *)g->in_col, (void *)g->in_w, (void *)g->deg,
                  (void *)g->colors})
    if (q) cudaFreeAsync(q, g->stream);
  g->async_layout.release(g->stream);
  g->color_layout.release(g->stream);
  g->push_layout.release(g->stream);
  g->push_color_layout.release(g->stream);
  cudaStreamSynchronize(g->stream);
  delete g;
  return FJ_OK;
}

}  // extern "C"
