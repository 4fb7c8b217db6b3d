// layout.cu — the sweep layout (§8 row a1, K3): rows of the pull CSR
// permuted to (color, length class, id) order so that every task handles rows
// of one color and of similar length, and the work list (tasks) that the
// persistent sweep kernel walks (static round-robin by default).  The row
// copy into layout order is chunked: a warp per 32 consecutive new rows
// (which share a length class), hub chunks cut into 2048-arc pieces.
//
// Permuted ids make the per-row state (s, ẑ, 1+d) streams coalesced; within
// one class the original id order is kept (stable), so R-MAT hubs (low ids)
// and lattice neighbours stay close in memory.
#include <stdio.h>
#include <stdlib.h>
#include <time.h>

#include <algorithm>

#include "fj_internal.cuh"

namespace fj {

static constexpr int kClasses = kNumClasses;  // 0..5 tile (G = 1<<k), 6 warp row, 7 warp pieces

__host__ __device__ static inline int row_class(int64_t L) {
  if (L <= 4) return 0;
  if (L <= 8) return 1;
  if (L <= 16) return 2;
  if (L <= 32) return 3;
  if (L <= 64) return 4;
  if (L <= (kWarpTileArcs > 64 ? kWarpTileArcs : 128)) return 5;
  if (L <= kWarpPiece) return 6;
  return 7;
}

static unsigned gridn(int64_t work) {
  int64_t b = (work + kBlock - 1) / kBlock;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 1 << 30));
}

// group of every row (color, length class descending; empty rows last) and, below it,
// the row's length descending inside a short-row class (so that the 32 rows of a row
// slice have the same length but at ≤ 256 boundaries per group) as the sort key, the row
// id as the payload: a stable sort keeps ids ascending among equal keys
constexpr int kSubBits = 8;
__host__ __device__ static inline int class_lmax(int cls) {
  return cls == 5 ? (kWarpTileArcs > 64 ? kWarpTileArcs : 128) : (4 << cls);
}
__global__ void k_layout_keys(int64_t n, const int64_t *__restrict__ ort,
                              const int32_t *__restrict__ color, int ncolors,
                              uint32_t *__restrict__ keys, uint32_t *__restrict__ ids,
                              unsigned long long *__restrict__ gcount) {
  int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint64_t grp = ~0ull;
  if (u < n) {
    int64_t L = ort[u + 1] - ort[u];
    if (L == 0) {
      grp = (uint64_t)ncolors * kClasses;  // empty rows last, never swept
    } else {
      int c = color ? color[u] : 0;
      grp = (uint64_t)c * kClasses + (uint64_t)(kClasses - 1 - row_class(L));
    }
    uint32_t sub = 0;
    if (L > 0) {
      const int cls = row_class(L);
      if (cls <= 5) sub = (uint32_t)min((int64_t)255, (int64_t)class_lmax(cls) - L);
    }
    keys[u] = ((uint32_t)grp << kSubBits) | sub;
    ids[u] = (uint32_t)u;
  }
  // warp-aggregated histogram: one atomic per distinct group in the warp
  const unsigned act = __ballot_sync(0xffffffffu, u < n);
  if (u < n) {
    const unsigned same = __match_any_sync(act, grp);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&gcount[grp], (unsigned long long)__popc(same));
  }
}

__global__ void k_perm(int64_t n, const uint32_t *__restrict__ ids, const int64_t *__restrict__ ort,
                       int32_t *__restrict__ perm, int32_t *__restrict__ iperm,
                       int64_t *__restrict__ len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t u = (int32_t)ids[i];
  perm[i] = u;
  iperm[u] = (int32_t)i;
  len[i] = ort[u + 1] - ort[u];
}

// warp per 32 consecutive new rows (rows of one length class sit together):
// the warp walks the rows' concatenated arc range 32 arcs at a time, each lane
// finding its arc's row among the 32 row starts by a shuffle binary search
// (all lanes busy even for 1–4-arc rows).  Chunks holding more than
// kLongChunk arcs (hub rows) are cut into kLongChunk-arc pieces listed for
// k_copy_long, a warp per piece, so no warp walks a whole hub row alone.
constexpr int64_t kLongChunk = kChunkArcs;

// the 32-row walk over arcs [k0, k1) of the chunk starting at row i0 (lane l
// holds the chunk's row start my_rp and source start my_src of row i0 + l)
__device__ __forceinline__ void copy_walk(int64_t n, int nr, int64_t my_rp, int64_t my_src,
                                          int64_t k0, int64_t k1, const int32_t *__restrict__ iperm,
                                          const int32_t *__restrict__ ocol,
                                          const float *__restrict__ ow, int32_t *__restrict__ col,
                                          float *__restrict__ w) {
  const int lane = threadIdx.x & 31;
  for (int64_t k = k0 + lane; k - lane < k1; k += 32) {
    const int r = chunk_row_of(nr, my_rp, k);
    const int64_t rs = __shfl_sync(0xffffffffu, my_rp, r);
    const int64_t src = __shfl_sync(0xffffffffu, my_src, r);
    if (k < k1) {
      const int64_t sk = src + (k - rs);
      const int32_t c = ocol[sk];
      col[k] = c < n ? iperm[c] : c;  // c ≥ n: a shard's remote column (shard.cu)
      if (w) w[k] = ow[sk];
    }
  }
}
__global__ void k_copy_rows32(int64_t n, const int32_t *__restrict__ perm,
                              const int32_t *__restrict__ iperm, const int64_t *__restrict__ ort,
                              const int32_t *__restrict__ ocol, const float *__restrict__ ow,
                              const double *__restrict__ deg, const int64_t *__restrict__ rp,
                              int32_t *__restrict__ col, float *__restrict__ w,
                              double *__restrict__ d1, unsigned *__restrict__ long_cnt,
                              int2 *__restrict__ long_list) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i0 = warp * 32; i0 < n; i0 += nwarps * 32) {
    const int64_t i = i0 + lane;
    const int nr = (int)(n - i0 < 32 ? n - i0 : 32);
    int64_t my_rp = 0, my_src = 0;
    if (i < n) {
      const int32_t u = perm[i];
      my_rp = rp[i];
      my_src = ort[u];
      if (d1) d1[i] = 1.0 + deg[u];
    }
    const int64_t a0 = __shfl_sync(0xffffffffu, my_rp, 0);
    const int64_t a1 = rp[i0 + nr];
    if (a1 - a0 > kLongChunk) {
      const int np = (int)((a1 - a0 + kLongChunk - 1) / kLongChunk);
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(long_cnt, (unsigned)np);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (int q = lane; q < np; q += 32) long_list[base + q] = make_int2((int)(i0 >> 5), q);
      continue;
    }
    copy_walk(n, nr, my_rp, my_src, a0, a1, iperm, ocol, ow, col, w);
  }
}

// the listed pieces of long chunks, a warp per piece (grid-stride over the
// device-side piece count)
__global__ void k_copy_long(int64_t n, const unsigned *__restrict__ long_cnt,
                            const int2 *__restrict__ long_list, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ iperm, const int64_t *__restrict__ ort,
                            const int32_t *__restrict__ ocol, const float *__restrict__ ow,
                            const int64_t *__restrict__ rp, int32_t *__restrict__ col,
                            float *__restrict__ w) {
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  const int64_t items = (int64_t)*long_cnt;
  for (int64_t it = warp; it < items; it += nwarps) {
    const int2 pc = long_list[it];
    const int64_t i0 = 32 * (int64_t)pc.x;
    const int nr = (int)(n - i0 < 32 ? n - i0 : 32);
    int64_t my_rp = 0, my_src = 0;
    if (lane < nr) {
      my_rp = rp[i0 + lane];
      my_src = ort[perm[i0 + lane]];
    }
    const int64_t a0 = __shfl_sync(0xffffffffu, my_rp, 0);
    const int64_t a1 = rp[i0 + nr];
    const int64_t k0 = a0 + (int64_t)pc.y * kLongChunk;
    const int64_t k1 = k0 + kLongChunk < a1 ? k0 + kLongChunk : a1;
    copy_walk(n, nr, my_rp, my_src, k0, k1, iperm, ocol, ow, col, w);
  }
}

// pieces per row for warp units: class 6 rows → 1, class 7 rows → ⌈L/2048⌉
__global__ void k_piece_counts(int64_t n, const int64_t *__restrict__ rp, int piece,
                               int64_t *__restrict__ np) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) { np[i] = 0; return; }
  const int64_t L = rp[i + 1] - rp[i];
  np[i] = L > (kWarpTileArcs > 64 ? kWarpTileArcs : 128) ? (L + piece - 1) / piece : 0;
}
// warp units in row order: unit scan[i] + p is piece p of row i
__global__ void k_fill_units(int64_t n, const int64_t *__restrict__ scan, Task *__restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = scan[i], np = scan[i + 1] - b;
  for (int64_t p = 0; p < np; p++)
    out[b + p] = Task{(int32_t)i, (int32_t)p, kWarp | (int32_t)(np << 8), (int32_t)b, 0, 0};
}
// values of a device array at host-given positions
__global__ void k_pick(int cnt, const int64_t *__restrict__ pos, const int64_t *__restrict__ src,
                       int64_t *__restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) out[i] = src[pos[i]];
}
// tile tasks of many row groups: group q covers tasks [out0, out0 + count) of
// rows [r0, r1) in steps of `per` rows, kind = class
struct TileGroup {
  int64_t out0, count;
  int32_t r0, r1, per, kind;
};
__global__ void k_fill_tiles(int ng, const TileGroup *__restrict__ gd, int64_t total,
                             Task *__restrict__ out) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= total) return;
  int lo = 0, hi = ng - 1;  // last group with out0 <= t
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (gd[mid].out0 <= t) lo = mid;
    else hi = mid - 1;
  }
  const TileGroup g = gd[lo];
  const int64_t k = t - g.out0;
  const int32_t a = (int32_t)(g.r0 + k * g.per);
  const int32_t b = (int32_t)min((int64_t)g.r1, (int64_t)a + g.per);
  out[t] = Task{a, b, g.kind, 0, 0, 0};
}

// arc range of every task (needs the device row pointers)
__global__ void k_task_arcs(int ntasks, const int64_t *__restrict__ rp, int piece,
                            Task *__restrict__ tasks) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntasks) return;
  Task t = tasks[i];
  if ((t.kind & 0xff) == kWarp) {
    t.a0 = rp[t.a] + (int64_t)t.b * piece;
    t.a1 = min(rp[t.a + 1], t.a0 + (int64_t)piece);
  } else {
    t.a0 = rp[t.a];
    t.a1 = rp[t.b];
  }
  tasks[i] = t;
}

__global__ void k_gather_tasks(int64_t n, const int32_t *__restrict__ idx, const Task *__restrict__ src,
                               Task *__restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}

// ---- row slices (sliced ELL for the single-RHS sweeps' short rows) ----
// slots of every item of the slice sweep list: 32 · (longest row) for a slice, 0 for a
// unit; a warp per item (slots[ntasks] = 0 closes the scan)
__global__ void k_slice_slots(int ntasks, const Task *__restrict__ tasks,
                              const int64_t *__restrict__ rp, int64_t *__restrict__ slots) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (i > ntasks) return;
  int mx = 0;
  if (i < ntasks) {
    const int4 t = *reinterpret_cast<const int4 *>(tasks + i);  // a, b, kind, slot
    if ((t.z & 0xff) == kSlice && t.x + lane < t.y) mx = (int)(rp[t.x + lane + 1] - rp[t.x + lane]);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) slots[i] = 32 * (int64_t)mx;
}
// a warp per slice: slot 32 t + l = arc t of row a + l, or the padding (column n — the
// zero entry after ẑ' — and weight 0); the task gets its slot range and width
__global__ void k_slice_fill(int ntasks, Task *__restrict__ tasks, const int64_t *__restrict__ off,
                             const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                             const float *__restrict__ w, int32_t npad,
                             int32_t *__restrict__ scol, float *__restrict__ sw) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < ntasks; i += nwarps) {
    Task t = tasks[i];
    if ((t.kind & 0xff) != kSlice) continue;
    const int64_t o0 = off[i], o1 = off[i + 1];
    const int wd = (int)((o1 - o0) >> 5);
    const int row = t.a + lane;
    int64_t rb = 0;
    int len = 0;
    if (row < t.b) {
      rb = rp[row];
      len = (int)(rp[row + 1] - rb);
    }
    for (int q = 0; q < wd; q++) {
      const bool ok = q < len;
      scol[o0 + 32 * q + lane] = ok ? col[rb + q] : npad;
      if (sw) sw[o0 + 32 * q + lane] = ok ? w[rb + q] : 0.0f;
    }
    if (lane == 0) {
      t.a0 = o0;
      t.a1 = o1;
      t.slot = wd;
      tasks[i] = t;
    }
  }
}

fj_status build_layout_from_out(fj_graph *g, const int64_t *ort, const int32_t *ocol,
                                const float *ow, const int32_t *color, int ncolors, Layout *L,
                                bool need_d1, bool slices) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n, m = g->m;
#ifdef FJ_DIAG
  const bool dbg = true;   // diagnostic build: phase timings on stderr
#else
  const bool dbg = false;
#endif
  timespec tt0;
  clock_gettime(CLOCK_MONOTONIC, &tt0);
  auto mark = [&](const char *what) {
    if (!dbg) return;
    cudaStreamSynchronize(st);
    timespec t1;
    clock_gettime(CLOCK_MONOTONIC, &t1);
    fprintf(stderr, "fj layout %-26s %8.2f ms\n", what,
            1e3 * (t1.tv_sec - tt0.tv_sec) + 1e-6 * (t1.tv_nsec - tt0.tv_nsec));
    tt0 = t1;
  };
  L->release(st);
  Workspace ws(st);  // keys, counts, scans; the layout arrays belong to L
  L->warp_unit_arcs = 0;
  L->n = n;
  L->m = m;
  L->ncolors = ncolors;
  const int ngroups = ncolors * kClasses + 1;

  uint32_t *k0 = nullptr, *k1 = nullptr, *id0 = nullptr, *id1 = nullptr;
  unsigned long long *gcount = nullptr;
  int64_t *len = nullptr;
  FJ_CUDA(ws.alloc(&k0, n));
  FJ_CUDA(ws.alloc(&k1, n));
  FJ_CUDA(ws.alloc(&id0, n));
  FJ_CUDA(ws.alloc(&id1, n));
  FJ_CUDA(ws.alloc(&gcount, ngroups));
  FJ_CUDA(cudaMemsetAsync(gcount, 0, sizeof(unsigned long long) * ngroups, st));
  FJ_CUDA(ws.alloc(&len, (n + 1)));
  FJ_CUDA(cudaMemsetAsync(len + n, 0, sizeof(int64_t), st));
  fj::count_launch();
  k_layout_keys<<<gridn(n), kBlock, 0, st>>>(n, ort, color, ncolors, k0, id0, gcount);

  int gbits = 1;
  while ((1 << gbits) <= ngroups) gbits++;
  if (gbits + kSubBits > 32) {
    set_error("layout: %d colors exceed the sort key", ncolors);
    return FJ_ERR_INVALID;
  }
  FJ_TRY((radix_sort_pairs<uint32_t, uint32_t>(k0, k1, id0, id1, n, gbits + kSubBits, ws)));  // prims.cu
  FJ_CUDA(cudaMallocAsync(&L->perm, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&L->iperm, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&L->rp, sizeof(int64_t) * (n + 2), st));
  FJ_CUDA(cudaMallocAsync(&L->col, sizeof(int32_t) * (m + kStreamPad), st));
  FJ_CUDA(cudaMemsetAsync(L->col + m, 0, sizeof(int32_t) * kStreamPad, st));
  if (ow) {
    FJ_CUDA(cudaMallocAsync(&L->w, sizeof(float) * (m + kStreamPad), st));
    FJ_CUDA(cudaMemsetAsync(L->w + m, 0, sizeof(float) * kStreamPad, st));
  }
  if (g->weighted || need_d1) FJ_CUDA(cudaMallocAsync(&L->d1, sizeof(double) * n, st));
  fj::count_launch();
  k_perm<<<gridn(n), kBlock, 0, st>>>(n, id0, ort, L->perm, L->iperm, len);
  FJ_TRY(exclusive_scan_i64(len, L->rp, n + 1, ws));
  fj::count_launch();
  mark("keys+sort+perm+scan");
  {
    unsigned *long_cnt = nullptr;
    int2 *long_list = nullptr;
    FJ_CUDA(ws.alloc(&long_cnt, 1));
    FJ_CUDA(ws.alloc(&long_list, (size_t)(m / kLongChunk + n / 32 + 2)));
    FJ_CUDA(cudaMemsetAsync(long_cnt, 0, sizeof(unsigned), st));
    k_copy_rows32<<<gridn(n), kBlock, 0, st>>>(n, L->perm, L->iperm, ort, ocol, ow, g->deg, L->rp,
                                               L->col, L->w, L->d1, long_cnt, long_list);
    fj::count_launch();
    k_copy_long<<<g->num_sms * 8, kBlock, 0, st>>>(n, long_cnt, long_list, L->perm, L->iperm, ort,
                                                   ocol, ow, L->rp, L->col, L->w);
  }

  int64_t *dmax = nullptr;
  int64_t hmax = 0;
  FJ_CUDA(ws.alloc(&dmax, 1));
  FJ_TRY(max_nonneg_i64(len, n, dmax, ws, g->num_sms));
  FJ_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  std::vector<unsigned long long> hcount(ngroups);
  FJ_CUDA(cudaMemcpyAsync(hcount.data(), gcount, sizeof(unsigned long long) * ngroups,
                          cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));

  mark("copy rows + counts");
  // group g covers new rows [gstart[g], gstart[g] + hcount[g])
  std::vector<int64_t> gstart(ngroups + 1, 0);
  for (int q = 0; q < ngroups; q++) gstart[q + 1] = gstart[q] + (int64_t)hcount[q];
  L->empty_rows = (int64_t)hcount[ngroups - 1];
  L->crow.assign(ncolors + 2, 0);
  for (int c = 0; c <= ncolors; c++) L->crow[c] = gstart[c * kClasses];
  L->crow[ncolors + 1] = n;
  L->active_rows = n - L->empty_rows;

  // work lists: tile tasks (classes 0..5) and warp units (classes 6, 7), each
  // grouped by color; within a color, longest rows first
  // ---- work lists, generated on the device ----
  // (1) row_ptr and warp-unit scan at every group boundary
  static const int kLmax[6] = {4, 8, 16, 32, 64, kWarpTileArcs > 64 ? kWarpTileArcs : 128};
  int64_t *npc = nullptr, *scan = nullptr, *dpos = nullptr, *dval = nullptr;
  FJ_CUDA(ws.alloc(&npc, (n + 1)));
  FJ_CUDA(ws.alloc(&scan, (n + 1)));
  fj::count_launch();
  // hub rows are split in warp pieces: long pieces (fewer partial combines)
  // for one-phase sweeps; short ones for colored sweeps, where every phase
  // waits for its slowest warp (a diagnostic build may force -DFJ_PIECE=…)
#ifdef FJ_PIECE
  int piece = FJ_PIECE;
#else
  int piece = ncolors > 1 ? 256 : kWarpPiece;
#endif
  L->piece = piece;
  k_piece_counts<<<gridn(n + 1), kBlock, 0, st>>>(n, L->rp, piece, npc);
  FJ_TRY(exclusive_scan_i64(npc, scan, n + 1, ws));
  std::vector<int64_t> hpos(ngroups + 1), hrp(ngroups + 1), hscan(ngroups + 1);
  for (int q = 0; q <= ngroups; q++) hpos[q] = gstart[q];
  FJ_CUDA(ws.alloc(&dpos, (ngroups + 1)));
  FJ_CUDA(ws.alloc(&dval, 2 * (ngroups + 1)));
  FJ_CUDA(cudaMemcpyAsync(dpos, hpos.data(), sizeof(int64_t) * (ngroups + 1), cudaMemcpyHostToDevice, st));
  fj::count_launch();
  k_pick<<<gridn(ngroups + 1), kBlock, 0, st>>>(ngroups + 1, dpos, L->rp, dval);
  fj::count_launch();
  k_pick<<<gridn(ngroups + 1), kBlock, 0, st>>>(ngroups + 1, dpos, scan, dval + ngroups + 1);
  FJ_CUDA(cudaMemcpyAsync(hrp.data(), dval, sizeof(int64_t) * (ngroups + 1), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaMemcpyAsync(hscan.data(), dval + ngroups + 1, sizeof(int64_t) * (ngroups + 1),
                          cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  // (2) list sizes and group descriptors on the host (O(colors · classes))
  L->phase_begin.assign(ncolors + 1, 0);
  L->wphase_begin.assign(ncolors + 1, 0);
  L->rphase_begin.assign(ncolors + 1, 0);
  L->sphase_begin.assign(ncolors + 1, 0);
  std::vector<TileGroup> ctag, rtag, stag;  // CTA tiles, warp tiles, row slices
  std::vector<std::pair<int64_t, int64_t>> unit_copy;  // per color: (src wtask begin, count)
  int64_t nt = 0, nrt = 0, nst = 0;
  for (int c = 0; c < ncolors; c++) {
    L->phase_begin[c] = (int)nt;
    L->rphase_begin[c] = (int)nrt;
    L->sphase_begin[c] = (int)nst;
    const int q6 = c * kClasses + 0, q5 = c * kClasses + 2;  // cd 0,1 = classes 7,6
    const int64_t u0 = hscan[q6], u1 = hscan[q5];
    L->wphase_begin[c] = (int)u0;
    unit_copy.push_back({u0, u1 - u0});
    nrt += u1 - u0;
    nst += u1 - u0;
    L->warp_unit_arcs += hrp[q5] - hrp[q6];
    for (int cd = 2; cd < kClasses; cd++) {
      const int q = c * kClasses + cd, cls = kClasses - 1 - cd;
      const int64_t r0 = gstart[q], r1 = gstart[q + 1];
      if (r1 <= r0) continue;
      const int64_t per = kBlock >> cls, wper = kWarpTileArcs / kLmax[cls];
      const int64_t cnt = (r1 - r0 + per - 1) / per, wcnt = (r1 - r0 + wper - 1) / wper;
      ctag.push_back(TileGroup{nt, cnt, (int32_t)r0, (int32_t)r1, (int32_t)per, cls});
      rtag.push_back(TileGroup{nrt, wcnt, (int32_t)r0, (int32_t)r1, (int32_t)wper, cls});
      const int64_t scnt = (r1 - r0 + 31) / 32;
      stag.push_back(TileGroup{nst, scnt, (int32_t)r0, (int32_t)r1, 32, kSlice});
      nt += cnt;
      nrt += wcnt;
      nst += scnt;
    }
  }
  const int64_t nwt = hscan[ngroups - 1];  // all warp units precede the empty rows
  L->phase_begin[ncolors] = (int)nt;
  L->wphase_begin[ncolors] = (int)nwt;
  L->rphase_begin[ncolors] = (int)nrt;
  L->sphase_begin[ncolors] = (int)nst;
  if (!slices) nst = 0;
  L->nstasks = (int)nst;
  L->ntasks = (int)nt;
  L->nwtasks = (int)nwt;
  L->nrtasks = (int)nrt;
  L->npartials = (int)nwt;
  // (3) fill the three lists on the device
  FJ_CUDA(cudaMallocAsync(&L->tasks, sizeof(Task) * std::max<int64_t>(1, nt), st));
  FJ_CUDA(cudaMallocAsync(&L->wtasks, sizeof(Task) * std::max<int64_t>(1, nwt), st));
  FJ_CUDA(cudaMallocAsync(&L->rtasks, sizeof(Task) * std::max<int64_t>(1, nrt), st));
  if (nwt > 0) {
    fj::count_launch();
    k_fill_units<<<gridn(n), kBlock, 0, st>>>(n, scan, L->wtasks);
  }
  TileGroup *dg = nullptr;
  const size_t ngd = ctag.size() + rtag.size() + stag.size();
  FJ_CUDA(ws.alloc(&dg, std::max<size_t>(1, ngd)));
  if (nst > 0) {
    FJ_CUDA(cudaMallocAsync(&L->stasks, sizeof(Task) * nst, st));
    if (!stag.empty()) {
      TileGroup *dsg = dg + ctag.size() + rtag.size();
      FJ_CUDA(cudaMemcpyAsync(dsg, stag.data(), sizeof(TileGroup) * stag.size(), cudaMemcpyHostToDevice, st));
      fj::count_launch();
      k_fill_tiles<<<gridn(nst), kBlock, 0, st>>>((int)stag.size(), dsg, nst, L->stasks);
    }
  }
  if (!ctag.empty())
    FJ_CUDA(cudaMemcpyAsync(dg, ctag.data(), sizeof(TileGroup) * ctag.size(), cudaMemcpyHostToDevice, st));
  if (!rtag.empty())
    FJ_CUDA(cudaMemcpyAsync(dg + ctag.size(), rtag.data(), sizeof(TileGroup) * rtag.size(),
                            cudaMemcpyHostToDevice, st));
  if (nt > 0) {
    fj::count_launch();
    k_fill_tiles<<<gridn(nt), kBlock, 0, st>>>((int)ctag.size(), dg, nt, L->tasks);
  }
  if (!rtag.empty()) {
    fj::count_launch();
    k_fill_tiles<<<gridn(nrt), kBlock, 0, st>>>((int)rtag.size(), dg + ctag.size(), nrt, L->rtasks);
  }
  for (int c = 0; c < ncolors; c++)  // warp units of color c head its sweep list
    if (unit_copy[c].second > 0) {
      FJ_CUDA(cudaMemcpyAsync(L->rtasks + L->rphase_begin[c], L->wtasks + unit_copy[c].first,
                              sizeof(Task) * unit_copy[c].second, cudaMemcpyDeviceToDevice, st));
      if (nst > 0)
        FJ_CUDA(cudaMemcpyAsync(L->stasks + L->sphase_begin[c], L->wtasks + unit_copy[c].first,
                                sizeof(Task) * unit_copy[c].second, cudaMemcpyDeviceToDevice, st));
    }
  for (Task *lst : {L->tasks, L->wtasks, L->rtasks, L->stasks}) {
    const int64_t cnt = lst == L->tasks ? nt : lst == L->wtasks ? nwt : lst == L->rtasks ? nrt : nst;
    if (lst && cnt > 0) {
      fj::count_launch();
      k_task_arcs<<<gridn(cnt), kBlock, 0, st>>>((int)cnt, L->rp, piece, lst);
    }
  }
  // Interleave warp units and short-row items in the one-phase sweep lists (Bresenham
  // on the counts) so every SM works on a mix of both at any time.  Measured:
  // C3 (Chung–Lu, few hub rows) 0.477 → 0.450 ms per sweep; C4 (R-MAT-24, 65 %
  // of the arcs in hub rows) 1.386 → 1.40, so only graphs whose warp units hold
  // under half the arcs get it.
  const bool mix = 2 * L->warp_unit_arcs < m;
  auto interleave = [&](Task *list, int64_t N) -> fj_status {
    const int64_t U = L->wphase_begin[1] - L->wphase_begin[0], T = N - U;
    std::vector<int32_t> hp(N);
    int64_t iu = 0, itl = 0;
    for (int64_t i = 0; i < N; i++) {
      const bool take_unit = iu < U && (itl >= T || (iu + 1) * T <= (itl + 1) * U);
      hp[i] = (int32_t)(take_unit ? iu++ : U + itl++);
    }
    int32_t *dp = nullptr;
    Task *tmpt = nullptr;
    FJ_CUDA(ws.alloc(&dp, (size_t)N));
    FJ_CUDA(ws.alloc(&tmpt, (size_t)N));
    FJ_CUDA(cudaMemcpyAsync(dp, hp.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice, st));
    fj::count_launch();
    k_gather_tasks<<<gridn(N), kBlock, 0, st>>>(N, dp, list, tmpt);
    FJ_CUDA(cudaMemcpyAsync(list, tmpt, sizeof(Task) * N, cudaMemcpyDeviceToDevice, st));
    FJ_CUDA(cudaStreamSynchronize(st));  // hp is stack-owned
    return FJ_OK;
  };
  if (ncolors == 1 && mix && nrt > 0) FJ_TRY(interleave(L->rtasks, nrt));
  // (the slice list stays units-first: interleaved it is 18–22 % slower per sweep on
  // C2 / C3, profiles/r02_slices_variants_ab.txt)
  mark("task lists (pre-slices)");
  // row slices: slots per item, scan, fill (the list order is final by now)
  if (nst > 0) {
    int64_t *slots = nullptr, *soff = nullptr;
    FJ_CUDA(ws.alloc(&slots, (size_t)nst + 1));
    FJ_CUDA(ws.alloc(&soff, (size_t)nst + 1));
    fj::count_launch();
    k_slice_slots<<<gridn(32 * (nst + 1)), kBlock, 0, st>>>((int)nst, L->stasks, L->rp, slots);
    FJ_TRY(exclusive_scan_i64(slots, soff, nst + 1, ws));
    int64_t total = 0;
    FJ_CUDA(cudaMemcpyAsync(&total, soff + nst, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    L->nslots = total;
    FJ_CUDA(cudaMallocAsync(&L->scol, sizeof(int32_t) * std::max<int64_t>(1, total), st));
    if (ow) FJ_CUDA(cudaMallocAsync(&L->sw, sizeof(float) * std::max<int64_t>(1, total), st));
    fj::count_launch();
    k_slice_fill<<<g->num_sms * 8, kBlock, 0, st>>>((int)nst, L->stasks, soff, L->rp, L->col, L->w,
                                                    (int32_t)n, L->scol, L->sw);
    mark("slices: slots+scan+fill");
    FJ_CUDA(cudaMallocAsync(&L->d_sphase_begin, sizeof(int) * (ncolors + 1), st));
    FJ_CUDA(cudaMemcpyAsync(L->d_sphase_begin, L->sphase_begin.data(), sizeof(int) * (ncolors + 1),
                            cudaMemcpyHostToDevice, st));
  }
  FJ_CUDA(cudaStreamSynchronize(st));  // host vectors above are stack-owned
  mark("task lists");
  if (dbg) {  // per-color layout summary (diagnostic build)
    std::vector<int64_t> cut(ncolors + 1);
    for (int c = 0; c <= ncolors; c++) cut[c] = gstart[c * kClasses];
    std::vector<int64_t> arc(ncolors + 1);
    for (int c = 0; c <= ncolors; c++)
      FJ_CUDA(cudaMemcpyAsync(&arc[c], L->rp + cut[c], sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    for (int c = 0; c < ncolors; c++)
      fprintf(stderr, "fj layout color %d rows %lld arcs %lld tiles %d warp_units %d\n", c,
              (long long)(cut[c + 1] - cut[c]), (long long)(arc[c + 1] - arc[c]),
              L->phase_begin[c + 1] - L->phase_begin[c], L->wphase_begin[c + 1] - L->wphase_begin[c]);
  }
  L->max_len = hmax;
  FJ_CUDA(cudaMallocAsync(&L->d_phase_begin, sizeof(int) * (ncolors + 1), st));
  FJ_CUDA(cudaMemcpyAsync(L->d_phase_begin, L->phase_begin.data(), sizeof(int) * (ncolors + 1),
                          cudaMemcpyHostToDevice, st));
  FJ_CUDA(cudaMallocAsync(&L->d_wphase_begin, sizeof(int) * (ncolors + 1), st));
  FJ_CUDA(cudaMemcpyAsync(L->d_wphase_begin, L->wphase_begin.data(), sizeof(int) * (ncolors + 1),
                          cudaMemcpyHostToDevice, st));
  FJ_CUDA(cudaMallocAsync(&L->d_rphase_begin, sizeof(int) * (ncolors + 1), st));
  FJ_CUDA(cudaMemcpyAsync(L->d_rphase_begin, L->rphase_begin.data(), sizeof(int) * (ncolors + 1),
                          cudaMemcpyHostToDevice, st));
  FJ_CUDA(cudaMallocAsync(&L->d_crow, sizeof(int64_t) * (ncolors + 2), st));
  FJ_CUDA(cudaMemcpyAsync(L->d_crow, L->crow.data(), sizeof(int64_t) * (ncolors + 2),
                          cudaMemcpyHostToDevice, st));
  FJ_CUDA(cudaStreamSynchronize(st));  // host vectors above are stack-owned
  FJ_CUDA(cudaGetLastError());
  return FJ_OK;
}

}  // namespace fj
