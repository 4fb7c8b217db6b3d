// api.cu — error state, pointer classification, small C-ABI entry points.
#include <stdarg.h>

#include <atomic>
#include <stdio.h>

#include "fj_internal.cuh"

namespace fj {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: unregistered host memory on old runtimes
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void Layout::release(cudaStream_t st) {
  for (void *q : {(void *)perm, (void *)iperm, (void *)rp, (void *)col, (void *)w, (void *)d1,
                  (void *)tasks, (void *)wtasks, (void *)d_phase_begin, (void *)d_wphase_begin,
                  (void *)d_crow, (void *)rtasks, (void *)d_rphase_begin, (void *)tail_beta,
                  (void *)scol, (void *)sw, (void *)stasks, (void *)d_sphase_begin})
    if (q) cudaFreeAsync(q, st);
  perm = iperm = nullptr;
  rp = nullptr;
  col = nullptr;
  w = nullptr;
  d1 = nullptr;
  tasks = wtasks = nullptr;
  d_phase_begin = d_wphase_begin = nullptr;
  d_crow = nullptr;
  crow.clear();
  tail_beta = nullptr;
  tail_phase = -1;
  tail_row0 = tail_row1 = 0;
  rtasks = nullptr;
  d_rphase_begin = nullptr;
  nrtasks = 0;
  rphase_begin.clear();
  scol = nullptr;
  sw = nullptr;
  stasks = nullptr;
  d_sphase_begin = nullptr;
  nslots = 0;
  nstasks = 0;
  sphase_begin.clear();
  ntasks = nwtasks = 0;
  ncolors = 0;
  phase_begin.clear();
  wphase_begin.clear();
}

}  // namespace fj

extern "C" {

const char *fj_last_error(void) { return fj::g_err; }

int fj_abi_version(void) { return FJ_ABI_VERSION; }

int64_t fj_kernel_launches(void) { return (int64_t)fj::g_launches.load(); }

void fj_opts_default(fj_opts *o) {
  if (!o) return;
  o->sigma = 1e-5;
  o->c = 0.0;
  o->method = FJ_METHOD_AUTO;
  o->max_sweeps = 1000000;
  o->cert_rounds = 3;
  o->certify = 1;
  o->zprime_out = nullptr;
  o->z_init = nullptr;
  o->tail_frac = -1.0;
  o->coloring = 0;
  o->push_compact = 0;
  o->push_sparse_div = 8;
  o->shadow = -1;
  o->slices = -1;
  o->frontier = -1;
}

fj_status fj_graph_get_info(fj_graph_t g, fj_graph_info *info) {
  if (!g || !info) {
    fj::set_error("fj_graph_get_info: null argument");
    return FJ_ERR_INVALID;
  }
  info->n = g->n;
  info->m = g->m;
  info->directed = g->directed;
  info->weighted = g->weighted;
  info->max_out_degree = g->async_layout.max_len;
  info->empty_rows = g->async_layout.empty_rows;
  info->tasks = g->async_layout.ntasks + g->async_layout.nwtasks;
  info->colors = g->ncolors;
  info->num_sms = g->num_sms;
  return FJ_OK;
}

}  // extern "C"
