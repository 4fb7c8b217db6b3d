// layout.cu — the sweep layout (§8 row a1, K3): rows of the pull CSR
// permuted to (color, length class, id) order so that every task handles rows
// of one color and of similar length, and the work list (tasks) that the
// persistent sweep kernel claims dynamically.
//
// Permuted ids make the per-row state (s, ẑ, 1+d) streams coalesced; within
// one class the original id order is kept (stable), so R-MAT hubs (low ids)
// and lattice neighbours stay close in memory.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <cub/cub.cuh>

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

__global__ void k_layout_keys(int64_t n, const int64_t *__restrict__ ort,
                              const int32_t *__restrict__ color, int ncolors,
                              uint64_t *__restrict__ keys, unsigned long long *__restrict__ gcount) {
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
    keys[u] = (grp << 31) | (uint64_t)u;
  }
  // warp-aggregated histogram: one atomic per distinct group in the warp
  const unsigned act = __ballot_sync(0xffffffffu, u < n);
  if (u < n) {
    const unsigned same = __match_any_sync(act, grp);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&gcount[grp], (unsigned long long)__popc(same));
  }
}

__global__ void k_perm(int64_t n, const uint64_t *__restrict__ keys, const int64_t *__restrict__ ort,
                       int32_t *__restrict__ perm, int32_t *__restrict__ iperm,
                       int64_t *__restrict__ len) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t u = (int32_t)(keys[i] & 0x7fffffffull);
  perm[i] = u;
  iperm[u] = (int32_t)i;
  len[i] = ort[u + 1] - ort[u];
}

// warp per new row: copy the out-row of perm[i] with relabelled columns
__global__ void k_copy_rows(int64_t n, const int32_t *__restrict__ perm,
                            const int32_t *__restrict__ iperm, const int64_t *__restrict__ ort,
                            const int32_t *__restrict__ ocol, const float *__restrict__ ow,
                            const double *__restrict__ deg, const int64_t *__restrict__ rp,
                            int32_t *__restrict__ col, float *__restrict__ w,
                            double *__restrict__ d1) {
  int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int64_t nwarps = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t i = warp; i < n; i += nwarps) {
    int32_t u = perm[i];
    int64_t b = ort[u], e = ort[u + 1], o = rp[i];
    for (int64_t k = lane; k < e - b; k += 32) {
      col[o + k] = iperm[ocol[b + k]];
      if (w) w[o + k] = ow[b + k];
    }
    if (lane == 0 && d1) d1[i] = 1.0 + deg[u];
  }
}

// arc range of every task (needs the device row pointers)
__global__ void k_task_arcs(int ntasks, const int64_t *__restrict__ rp, Task *__restrict__ tasks) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntasks) return;
  Task t = tasks[i];
  if ((t.kind & 0xff) == kWarp) {
    t.a0 = rp[t.a] + (int64_t)t.b * kWarpPiece;
    t.a1 = min(rp[t.a + 1], t.a0 + (int64_t)kWarpPiece);
  } else {
    t.a0 = rp[t.a];
    t.a1 = rp[t.b];
  }
  tasks[i] = t;
}

fj_status build_layout_from_out(fj_graph *g, const int64_t *ort, const int32_t *ocol,
                                const float *ow, const int32_t *color, int ncolors, Layout *L,
                                bool need_d1) {
  cudaStream_t st = g->stream;
  const int64_t n = g->n, m = g->m;
  L->release(st);
  L->warp_unit_arcs = 0;
  L->n = n;
  L->m = m;
  L->ncolors = ncolors;
  const int ngroups = ncolors * kClasses + 1;

  uint64_t *k0 = nullptr, *k1 = nullptr;
  unsigned long long *gcount = nullptr;
  int64_t *len = nullptr;
  FJ_CUDA(cudaMallocAsync(&k0, sizeof(uint64_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&k1, sizeof(uint64_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&gcount, sizeof(unsigned long long) * ngroups, st));
  FJ_CUDA(cudaMemsetAsync(gcount, 0, sizeof(unsigned long long) * ngroups, st));
  FJ_CUDA(cudaMallocAsync(&len, sizeof(int64_t) * (n + 1), st));
  FJ_CUDA(cudaMemsetAsync(len + n, 0, sizeof(int64_t), st));
  fj::count_launch();
  k_layout_keys<<<gridn(n), kBlock, 0, st>>>(n, ort, color, ncolors, k0, gcount);

  int gbits = 1;
  while ((1 << gbits) <= ngroups) gbits++;
  {
    cub::DoubleBuffer<uint64_t> dk(k0, k1);
    size_t tmp = 0;
    FJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dk, n, 0, 31 + gbits, st));
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, tmp, st));
    FJ_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, dk, n, 0, 31 + gbits, st));
    FJ_CUDA(cudaFreeAsync(t, st));
    if (dk.Current() != k0) std::swap(k0, k1);
  }
  FJ_CUDA(cudaMallocAsync(&L->perm, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&L->iperm, sizeof(int32_t) * n, st));
  FJ_CUDA(cudaMallocAsync(&L->rp, sizeof(int64_t) * (n + 2), st));
  FJ_CUDA(cudaMallocAsync(&L->col, sizeof(int32_t) * (m + 8), st));
  if (ow) FJ_CUDA(cudaMallocAsync(&L->w, sizeof(float) * (m + 8), st));
  if (g->weighted || need_d1) FJ_CUDA(cudaMallocAsync(&L->d1, sizeof(double) * n, st));
  fj::count_launch();
  k_perm<<<gridn(n), kBlock, 0, st>>>(n, k0, ort, L->perm, L->iperm, len);
  {
    size_t tmp = 0;
    FJ_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, len, L->rp, n + 1, st));
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, tmp, st));
    FJ_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, len, L->rp, n + 1, st));
    FJ_CUDA(cudaFreeAsync(t, st));
  }
  fj::count_launch();
  k_copy_rows<<<gridn(n * 32), kBlock, 0, st>>>(n, L->perm, L->iperm, ort, ocol, ow, g->deg, L->rp,
                                                L->col, L->w, L->d1);

  int64_t *dmax = nullptr;
  int64_t hmax = 0;
  FJ_CUDA(cudaMallocAsync(&dmax, sizeof(int64_t), st));
  {
    size_t tmp = 0;
    FJ_CUDA(cub::DeviceReduce::Max(nullptr, tmp, len, dmax, n, st));
    void *t = nullptr;
    FJ_CUDA(cudaMallocAsync(&t, tmp, st));
    FJ_CUDA(cub::DeviceReduce::Max(t, tmp, len, dmax, n, st));
    FJ_CUDA(cudaFreeAsync(t, st));
  }
  FJ_CUDA(cudaMemcpyAsync(&hmax, dmax, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaFreeAsync(dmax, st));
  std::vector<unsigned long long> hcount(ngroups);
  FJ_CUDA(cudaMemcpyAsync(hcount.data(), gcount, sizeof(unsigned long long) * ngroups,
                          cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));

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
  std::vector<Task> tasks, wtasks, rtasks;
  L->phase_begin.assign(ncolors + 1, 0);
  L->wphase_begin.assign(ncolors + 1, 0);
  L->rphase_begin.assign(ncolors + 1, 0);
  static const int kLmax[6] = {4, 8, 16, 32, 64, kWarpTileArcs > 64 ? kWarpTileArcs : 128};
  int slot = 0;
  for (int c = 0; c < ncolors; c++) {
    L->phase_begin[c] = (int)tasks.size();
    L->wphase_begin[c] = (int)wtasks.size();
    L->rphase_begin[c] = (int)rtasks.size();
    for (int cd = 0; cd < kClasses; cd++) {  // cd = 7 - class
      int q = c * kClasses + cd;
      int cls = kClasses - 1 - cd;
      int64_t r0 = gstart[q], r1 = gstart[q + 1];
      if (r1 <= r0) continue;
      if (cls >= 6) {
        int64_t ra = 0, rz = 0;
        FJ_CUDA(cudaMemcpyAsync(&ra, L->rp + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        FJ_CUDA(cudaMemcpyAsync(&rz, L->rp + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        FJ_CUDA(cudaStreamSynchronize(st));
        L->warp_unit_arcs += rz - ra;
      }
      if (cls == 7) {
        std::vector<int64_t> rph(r1 - r0 + 1);
        FJ_CUDA(cudaMemcpyAsync(rph.data(), L->rp + r0, sizeof(int64_t) * (r1 - r0 + 1),
                                cudaMemcpyDeviceToHost, st));
        FJ_CUDA(cudaStreamSynchronize(st));
        for (int64_t i = r0; i < r1; i++) {
          int64_t len_i = rph[i - r0 + 1] - rph[i - r0];
          int np = (int)((len_i + kWarpPiece - 1) / kWarpPiece);
          for (int p = 0; p < np; p++) {
            wtasks.push_back(Task{(int32_t)i, p, kWarp | (np << 8), slot, 0, 0});
            rtasks.push_back(wtasks.back());
          }
          slot += np;
        }
      } else if (cls == 6) {
        for (int64_t i = r0; i < r1; i++) {
          wtasks.push_back(Task{(int32_t)i, 0, kWarp | (1 << 8), 0, 0, 0});
          rtasks.push_back(wtasks.back());
        }
      } else {
        int G = 1 << cls;
        int64_t per = kBlock / G;  // one G-lane group per row
        for (int64_t a = r0; a < r1; a += per)
          tasks.push_back(Task{(int32_t)a, (int32_t)std::min(r1, a + per), cls, 0, 0, 0});
        // warp tiles for the sweep: <= kWarpTileArcs arcs, 32/G rows per step
        const int64_t wper = kWarpTileArcs / kLmax[cls];
        for (int64_t a = r0; a < r1; a += wper)
          rtasks.push_back(Task{(int32_t)a, (int32_t)std::min(r1, a + wper), cls, 0, 0, 0});
      }
    }
  }
  L->phase_begin[ncolors] = (int)tasks.size();
  L->wphase_begin[ncolors] = (int)wtasks.size();
  L->rphase_begin[ncolors] = (int)rtasks.size();
  L->nrtasks = (int)rtasks.size();
  // measured on all five configs: direct loads beat the TMA-staged stream
  // once short rows run as warp tiles (the stage buffers take L1 away from
  // the ẑ gathers); the TMA path stays selectable with FJ_TMA=1
  L->stream_tma = false;
  if (getenv("FJ_DEBUG")) {  // per-color layout summary (diagnostics)
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
  L->ntasks = (int)tasks.size();
  L->nwtasks = (int)wtasks.size();
  L->npartials = slot;
  L->max_len = hmax;
  for (int which = 0; which < 3; which++) {
    std::vector<Task> &v = which == 0 ? tasks : which == 1 ? wtasks : rtasks;
    Task **dst = which == 0 ? &L->tasks : which == 1 ? &L->wtasks : &L->rtasks;
    FJ_CUDA(cudaMallocAsync(dst, sizeof(Task) * std::max<size_t>(1, v.size()), st));
    if (!v.empty()) {
      FJ_CUDA(cudaMemcpyAsync(*dst, v.data(), sizeof(Task) * v.size(), cudaMemcpyHostToDevice, st));
      fj::count_launch();
      k_task_arcs<<<gridn((int64_t)v.size()), kBlock, 0, st>>>((int)v.size(), L->rp, *dst);
    }
  }
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
  FJ_CUDA(cudaFreeAsync(k0, st));
  FJ_CUDA(cudaFreeAsync(k1, st));
  FJ_CUDA(cudaFreeAsync(gcount, st));
  FJ_CUDA(cudaFreeAsync(len, st));
  FJ_CUDA(cudaGetLastError());
  return FJ_OK;
}

}  // namespace fj
