// fj_internal.cuh — internal types of libfj (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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
constexpr int kPiece = 2048;          // arcs per piece of a long row (8 per thread)
constexpr int kNumClasses = 8;        // row-length classes of the layout

// Row-length classes (out-degree L of the pull CSR).  Rows with L == 0 are
// solved exactly at init (z_v = s_v, Eq. (1) with d_v = 0) and never enter a
// sweep.  class k < 6 uses G = 1 << k lanes per row:
//   class 0: L in [1,4]   G = 1        class 3: L in (16,32]   G = 8
//   class 1: L in (4,8]   G = 2        class 4: L in (32,64]   G = 16
//   class 2: L in (8,16]  G = 4        class 5: L in (64,256]  G = 32
//   class 6: L > 256      long row, split in pieces of kPiece arcs
enum TaskKind : int32_t {
  kG1 = 0, kG2 = 1, kG4 = 2, kG8 = 3, kG16 = 4, kG32 = 5,  // GROUP, G = 1 << kind
  kLong = 7                                                   // one piece of a long row
};

// One unit of sweep work.  GROUP: rows [a, b) with G = 1 << (kind & 0xff).
// LONG: row a, piece b of npieces = kind >> 8; slot = first partial slot of
// the row (also its arrival counter index).
struct Task {
  int32_t a, b, kind, slot;
};

// Sweep layout: the pull CSR (row u lists v with a_uv) with rows permuted to
// (color, class, id) order; ids in `col` are permuted ids.
struct Layout {
  int ncolors = 0;
  int64_t n = 0, m = 0;
  int32_t *perm = nullptr;   // new -> old
  int32_t *iperm = nullptr;  // old -> new
  int64_t *rp = nullptr;     // [n+1]
  int32_t *col = nullptr;    // [m]
  float *w = nullptr;        // [m] or null
  double *d1 = nullptr;      // 1 + d_u (weighted graphs only) [n]
  Task *tasks = nullptr;
  int ntasks = 0;
  std::vector<int> phase_begin;   // host, ncolors + 1 entries
  int *d_phase_begin = nullptr;   // device copy
  int npartials = 0;              // partial slots for long rows
  int64_t empty_rows = 0;
  int64_t active_rows = 0;        // rows with L > 0
  int64_t max_len = 0;
  void release();
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
  int32_t *colors = nullptr; // color per original node (lazy)
  int ncolors = 0;
};

namespace fj {
// graph.cu
fj_status transpose_in_csr(fj_graph *g, int64_t **ort, int32_t **ocol, float **ow);
// layout.cu: sweep layout from the pull CSR (original ids)
fj_status build_layout_from_out(fj_graph *g, const int64_t *ort, const int32_t *ocol,
                                const float *ow, const int32_t *color /* nullable */,
                                int ncolors, Layout *L);
// color.cu
fj_status build_coloring(fj_graph *g);
// memory helpers (api.cu)
bool is_device_ptr(const void *p);
}  // namespace fj
