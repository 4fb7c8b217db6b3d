// fj_internal.cuh — internal types of libfj (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/fj.h"

namespace fj {

void set_error(const char *fmt, ...);

#define FJ_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      fj::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));   \
      return FJ_ERR_CUDA;                                                                 \
    }                                                                                     \
  } while (0)

#define FJ_TRY(call)                  \
  do {                                \
    fj_status s_ = (call);            \
    if (s_ != FJ_OK) return s_;       \
  } while (0)

constexpr int kBlock = 256;           // threads per CTA of every task kernel
constexpr int kWarpPiece = 2048;      // arcs of one warp unit (whole row or piece)
constexpr int kTileArcs = 2048;       // max arcs of one CTA tile task (smem products)
#ifndef FJ_WT_ARCS
#define FJ_WT_ARCS 256
#endif
constexpr int kWarpTileArcs = FJ_WT_ARCS;  // max arcs of one warp tile (8 per lane)
constexpr int kNumClasses = 8;        // row-length classes of the layout
constexpr int64_t kStreamPad = 264;   // zero-filled col/w slots after the last arc (16-byte
                                      // sweep loads may run up to 259 slots past a tile start)
constexpr int64_t kChunkArcs = 2048;  // chunked row walks: pieces of long 32-row chunks

// Chunked row walks (graph build, layout copy): a warp owns 32 consecutive
// rows, lane l holding the start my_rp of row i0 + l (nr ≤ 32 rows).  For an
// arc position k in the chunk, the row is the largest r < nr with
// rp[i0 + r] ≤ k (empty rows share a start: the last of them is the owner).
// Five shuffles; every lane of the warp must call it.
__device__ __forceinline__ int chunk_row_of(int nr, int64_t my_rp, int64_t k) {
  int r = 0;
#pragma unroll
  for (int step = 16; step > 0; step >>= 1) {
    const int q = r + step;
    const int64_t v = __shfl_sync(0xffffffffu, my_rp, q < nr ? q : 0);
    if (q < nr && v <= k) r = q;
  }
  return r;
}

// Row-length classes (out-degree L of the pull CSR).  Rows with L == 0 are
// solved exactly at init (z_v = s_v, Eq. (1) with d_v = 0) and never enter a
// sweep.  Classes 0..5 are CTA "tile" tasks with G = 1 << k lanes per row:
//   class 0: L in [1,4]   G = 1        class 3: L in (16,32]   G = 8
//   class 1: L in (4,8]   G = 2        class 4: L in (32,64]   G = 16
//   class 2: L in (8,16]  G = 4        class 5: L in (64,256]  G = 32
// Classes 6 and 7 are warp units (one warp, no block barrier):
//   class 6: L in (256, kWarpPiece]  one warp per row
//   class 7: L > kWarpPiece          pieces of kWarpPiece arcs, one warp each,
//                                    combined by the last-arriving warp
enum TaskKind : int32_t {
  kG1 = 0, kG2 = 1, kG4 = 2, kG8 = 3, kG16 = 4, kG32 = 5,  // CTA tile, G = 1 << kind
  kWarp = 6,                                                  // warp unit
  kSlice = 7                                                  // row slice (sweep list only)
};

// One unit of sweep work.  Tile (kind 0..5): rows [a, b) with
// G = 1 << kind lanes per row, one group per row (b - a <= kBlock / G).
// Warp unit (kind & 0xff == kWarp): row a, piece b of npieces = kind >> 8;
// slot = first partial slot of the row (also its arrival counter index).
// [a0, a1) is the unit's arc range in the layout CSR.
// Row slice (kind kSlice, Layout::stasks only): rows [a, b), b − a ≤ 32, one lane per row;
// slot = the slice's width Wd (its longest row); [a0, a1) = its 32·Wd slots in
// Layout::scol / sw, arc t of row a + l at a0 + 32 t + l (padding: column n, weight 0).
struct alignas(16) Task {
  int32_t a, b, kind, slot;
  int64_t a0, a1;
};

// Sweep layout: the pull CSR (row u lists v with a_uv) with rows permuted to
// (color, class, id) order; ids in `col` are permuted ids.
struct Layout {
  int ncolors = 0;
  int tail_phase = -1;  // merged tail colors (reading R23); −1 if none
  int64_t tail_row0 = 0, tail_row1 = 0;  // (permuted) rows of the tail phase
  float *tail_beta = nullptr;     // β_i = Σ_{j in tail} a_ij / (1 + d_i) per tail row
  int64_t n = 0, m = 0;
  int32_t *perm = nullptr;   // new -> old
  int32_t *iperm = nullptr;  // old -> new
  int64_t *rp = nullptr;     // [n+1]
  int32_t *col = nullptr;    // [m]
  float *w = nullptr;        // [m] or null
  double *d1 = nullptr;      // 1 + d_u (weighted graphs only) [n]
  Task *tasks = nullptr;          // CTA tile tasks, grouped by phase (color)
  int ntasks = 0;
  Task *wtasks = nullptr;         // warp units, grouped by phase
  int nwtasks = 0;
  Task *rtasks = nullptr;         // sweep list: warp units, then warp tiles (short rows)
  int nrtasks = 0;
  std::vector<int> rphase_begin;
  int *d_rphase_begin = nullptr;
  // Row slices (the single-RHS sweeps' short rows): the arcs of rows ≤ kWarpTileArcs in
  // slice order (sliced ELL: 32 rows per slice, one lane per row, coalesced column-major
  // slots), and the sweep list that walks them: warp units, then slices
  int32_t *scol = nullptr;        // [nslots]
  float *sw = nullptr;            // [nslots] or null
  int64_t nslots = 0;
  Task *stasks = nullptr;
  int nstasks = 0;
  std::vector<int> sphase_begin;
  int *d_sphase_begin = nullptr;
  std::vector<int> phase_begin;   // host, ncolors + 1 entries (tile tasks)
  std::vector<int> wphase_begin;  // host, ncolors + 1 entries (warp units)
  int *d_phase_begin = nullptr;   // device copies
  int *d_wphase_begin = nullptr;
  std::vector<int64_t> crow;      // host: first row of each color; [ncolors] = first
                                  // empty row; [ncolors + 1] = n
  int64_t *d_crow = nullptr;      // device copy
  int npartials = 0;              // partial slots for long rows
  int64_t empty_rows = 0;
  int64_t active_rows = 0;        // rows with L > 0
  int64_t max_len = 0;
  int64_t warp_unit_arcs = 0;     // arcs in rows handled by warp units (> kWarpTileArcs)
  int piece = kWarpPiece;         // arcs per warp piece of a hub row
  void release(cudaStream_t st);
};

}  // namespace fj

struct fj_graph {
  int64_t n = 0, m = 0;
  int directed = 0, weighted = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
  // canonical in-CSR (rows sorted), original ids: measures and push method
  int64_t *in_rp = nullptr;
  int32_t *in_col = nullptr;
  float *in_w = nullptr;
  // out-degree in original order, fp64 (d_u = Σ_v a_uv)
  double *deg = nullptr;
  fj::Layout async_layout;   // 1 color, rows grouped by class
  fj::Layout color_layout;   // lazily built for COLORED solves
  fj::Layout push_layout;    // lazily built for PUSH (in-rows: scatter lists)
  fj::Layout push_color_layout;
  int32_t *colors = nullptr; // color per original node (lazy); tail colors merged
  int ncolors = 0;           // phases of a colored sweep (tail merged)
  int ncolors_raw = 0;       // colors of the distance-1 coloring before the merge
  int tail_color = -1;       // merged tail phase (−1: none)
  double color_tail_frac = -2.0;  // fj_opts.tail_frac / .coloring the coloring was built with
  int color_algo = -1;
  cudaEvent_t w_ready = nullptr;  // during create only: host weights staged on a side stream
};

namespace fj {
// Stream-ordered workspace of one call: every buffer and event it hands out is
// released when it goes out of scope, on the normal path and on every early
// error return (an allocation failure half-way through a solve leaks nothing).
struct Workspace {
  cudaStream_t st;
  std::vector<void *> bufs;
  std::vector<cudaEvent_t> evs;
  explicit Workspace(cudaStream_t s) : st(s) {}
  Workspace(const Workspace &) = delete;
  Workspace &operator=(const Workspace &) = delete;
  ~Workspace() {
    for (void *q : bufs)
      if (q) cudaFreeAsync(q, st);
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
  }
  template <class T>
  cudaError_t alloc(T **q, size_t count) {
    *q = nullptr;
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(q),
                                          sizeof(T) * std::max<size_t>(count, 1), st);
    if (e == cudaSuccess) bufs.push_back(*q);
    return e;
  }
  // hand a buffer over to a longer-lived owner (it is no longer freed here)
  void keep(const void *q) {
    for (auto &b : bufs)
      if (b == q) b = nullptr;
  }
  cudaError_t event(cudaEvent_t *e) {
    const cudaError_t r = cudaEventCreate(e);
    if (r == cudaSuccess) evs.push_back(*e);
    return r;
  }
};

// graph.cu
fj_status transpose_in_csr(fj_graph *g, Workspace &ws, int64_t **ort, int32_t **ocol, float **ow,
                           int *err = nullptr);
// layout.cu: sweep layout from the pull CSR (original ids)
fj_status build_layout_from_out(fj_graph *g, const int64_t *ort, const int32_t *ocol,
                                const float *ow, const int32_t *color /* nullable */,
                                int ncolors, Layout *L, bool need_d1 = false,
                                bool slices = false);
// color.cu
fj_status build_coloring(fj_graph *g, const fj_opts *o);  // (re)builds if o asks for other options
// prims.cu: hand-written primitives of the graph build and the shift
fj_status minmax_f32(const float *x, int64_t n, float *out2 /* device [min, max] */, Workspace &ws,
                     int num_sms);
fj_status max_nonneg_i64(const int64_t *x, int64_t n, int64_t *out /* device */, Workspace &ws,
                         int num_sms);
fj_status exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, Workspace &ws);
// stable LSD radix sort on the low nbits of the keys; on return keys/vals point
// at the sorted data (the buffers may have been swapped with the *_alt ones)
template <class K, class V>
fj_status radix_sort_pairs(K *&keys, K *&keys_alt, V *&vals, V *&vals_alt, int64_t m, int nbits,
                           Workspace &ws);
// memory helpers (api.cu)
bool is_device_ptr(const void *p);
// every kernel launch issued by this library is counted (fj_kernel_launches)
void count_launch();
}  // namespace fj
