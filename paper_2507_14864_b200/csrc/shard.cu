// shard.cu — sharded solve over ranks.
//
// A 1-D node partition: rank r owns the equations (rows of I + L, Lemma 1,
// P:87) and the estimates ẑ_u of the nodes u ∈ [begin[r], begin[r+1]).  Its
// sweep layout is fj_solve's (layout.cu) built over the owned OUT-rows only;
// columns are relabelled into the rank's ẑ buffer
//
//     [ own n_local rows (layout order) | halo from slot 0 | … | halo from slot W−2 ]
//
// where slot j is rank (r + 1 + j) mod W and its halo holds exactly the nodes
// of that rank that r's rows read (sorted by their owner's layout position):
// 0.18·n per rank on R-MAT-24 and 0.003·n on the lattice at W = 8, against
// 0.875·n for whole segments.  The sweep kernel is fj_solve's k_sweep, one
// sweep per launch, unchanged: own and halo columns are plain indices into the
// buffer.  After every sweep the ranks exchange halos (each rank packs the
// values its peers need and sends them with grouped ncclSend/ncclRecv over
// NVLink; the in-process transport gathers them directly) and all-reduce
// (relaxations, edge updates, sentinel flag, bad-input flag).  A sweep with
// zero relaxations on every rank read only final values (the last exchange
// delivered every halo as it still is), which is the paper's stopping rule
// Q = ∅; then the fp64 certificate (Lemma 3) runs on every
// rank and the maximum decides, with the resume rule of reading R21.
//
// Schedule across ranks: block-Jacobi with in-place Gauss–Seidel inside each
// block — an asynchronous relaxation with bounded staleness, convergent at
// ω = 1 because I + L is an M-matrix.
#include <dlfcn.h>
#include <nccl.h>
#include <cub/cub.cuh>
#include <string.h>

#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "sweep_common.cuh"

// node kernels of solve.cu
namespace fj {
__global__ void k_meas_nodes1(int64_t n, const int32_t *__restrict__ perm,
                              const float *__restrict__ z, double *__restrict__ zl,
                              double *__restrict__ sums);
}

struct fj_comm {
  int world = 1, rank = 0;
  bool local = true;
  // in-process transport that runs the NCCL path's bookkeeping (send lists,
  // pack kernel, per-peer segments) with device copies in place of
  // ncclSend/ncclRecv: fj_comm_create_loopback (tests)
  bool loopback = false;
  ncclComm_t nc = nullptr;
  cudaStream_t stream = nullptr;
  int num_sms = 0;
};

struct fj_shard {
  fj_comm *comm = nullptr;
  int rank = 0;
  int64_t n = 0;                 // global nodes
  std::vector<int64_t> begin;    // [world + 1]
  int64_t n_local = 0, seg_max = 0, nz = 0;  // nz = n_local + halo entries (after connect)
  fj_graph *g = nullptr;         // owned rows: n = n_local, async layout
  bool connected = false;
  // halo (after connect): entries [hoff[j], hoff[j+1]) come from slot j; need[i]
  // is the position of entry i in its owner's layout order
  std::vector<int64_t> hoff;     // [world] (slot offsets into the halo; hoff[W−1] = total)
  int32_t *need = nullptr;       // [halo]
  // NCCL: the positions of this rank's nodes that each peer reads, by peer rank
  std::vector<int64_t> soff;     // [world + 1] offsets into sendidx / sendbuf
  int32_t *sendidx = nullptr;
  double *sendbuf = nullptr;
};

namespace fj {

constexpr int kMaxLocal = 64;    // shards of one in-process comm
constexpr int kSweepBatch = 16;  // sweeps queued per host check (sharded loop)

// ------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char *(*GetErrorString)(ncclResult_t);
};

static const NcclApi *nccl() {
  static std::once_flag once;
  static NcclApi api{};
  static bool ok = false;
  std::call_once(once, [] {
    // in a PyTorch process this resolves to the libnccl.so.2 torch loaded
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define FJ_SYM(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
    FJ_SYM(GetUniqueId, "ncclGetUniqueId");
    FJ_SYM(CommInitRank, "ncclCommInitRank");
    FJ_SYM(CommDestroy, "ncclCommDestroy");
    FJ_SYM(AllReduce, "ncclAllReduce");
    FJ_SYM(AllGather, "ncclAllGather");
    FJ_SYM(Send, "ncclSend");
    FJ_SYM(Recv, "ncclRecv");
    FJ_SYM(GroupStart, "ncclGroupStart");
    FJ_SYM(GroupEnd, "ncclGroupEnd");
    FJ_SYM(GetErrorString, "ncclGetErrorString");
#undef FJ_SYM
    ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
         api.AllGather && api.Send && api.Recv && api.GroupStart && api.GroupEnd &&
         api.GetErrorString;
  });
  return ok ? &api : nullptr;
}

#define FJ_NCCL(call)                                                               \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) {                                                        \
      fj::set_error("NCCL %s: %s", #call, fj::nccl()->GetErrorString(r_));          \
      return FJ_ERR_CUDA;                                                           \
    }                                                                               \
  } while (0)

// ------------------------------------------------------------------ kernels
// warp per owned row: ids in range, no self-loop, strictly increasing, valid
// weights; then the column code: own node → local id, remote → n_local + v
__global__ void k_shard_rows(int64_t n_local, int64_t b0, int64_t n, const int64_t *__restrict__ rp,
                             const int32_t *__restrict__ col, const float *__restrict__ w,
                             int32_t *__restrict__ enc, int *__restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n_local; u += nw) {
    int bad = 0;
    for (int64_t e = rp[u] + lane; e < rp[u + 1]; e += 32) {
      const int32_t v = col[e];
      if (v < 0 || v >= n) {
        bad |= 2;
        continue;
      }
      if ((int64_t)v == b0 + u) bad |= 4;
      if (w && !(w[e] > 0.0f && isfinite(w[e]))) bad |= 8;
      if (e > rp[u] && col[e - 1] >= v) bad |= 16;
      enc[e] = (v >= b0 && v < b0 + n_local) ? (int32_t)(v - b0) : (int32_t)(n_local + v);
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicOr(err, bad);
  }
}

__global__ void k_shard_rowptr(int64_t n, int64_t m, const int64_t *__restrict__ rp,
                               int *__restrict__ err) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t x = rp[i];
  if ((i == 0 && x != 0) || (i == n && x != m) || (i < n && rp[i + 1] < x) || x < 0 || x > m)
    atomicOr(err, 1);
}

__global__ void k_shard_rowsum(int64_t n, const int64_t *__restrict__ rp, const float *__restrict__ w,
                               double *__restrict__ d) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (gridDim.x * (int64_t)blockDim.x) >> 5;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n; u += nw) {
    double s = 0.0;
    if (w) {
      for (int64_t k = rp[u] + lane; k < rp[u + 1]; k += 32) s += (double)w[k];
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    } else {
      s = (double)(rp[u + 1] - rp[u]);
    }
    if (lane == 0) d[u] = s;  // d_u = Σ_v a_uv
  }
}

// remote column code n_local + v → halo key (slot of v's owner, v's position
// in its owner's layout); own columns → ~0 (sorts last)
__global__ void k_halo_keys(int64_t m, const int32_t *__restrict__ col, int64_t n_local, int rank,
                            int world, int64_t seg_max, const int64_t *__restrict__ begin,
                            const int32_t *__restrict__ iperm_all, uint64_t *__restrict__ keys,
                            int *__restrict__ err) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int32_t c = col[k];
  if (c < n_local) {
    keys[k] = ~0ull;
    return;
  }
  const int64_t v = (int64_t)c - n_local;
  int lo = 0, hi = world - 1;  // owner: last r with begin[r] <= v
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (begin[mid] <= v) lo = mid;
    else hi = mid - 1;
  }
  const int32_t pos = iperm_all[(int64_t)lo * seg_max + (v - begin[lo])];
  if (lo == rank || pos < 0) {
    atomicOr(err, 1);
    keys[k] = ~0ull;
    return;
  }
  const uint64_t slot = (uint64_t)((lo - rank - 1 + world) % world);
  keys[k] = (slot << 32) | (uint64_t)(uint32_t)pos;
}

// remote column → n_local + its index among the sorted unique halo keys
__global__ void k_halo_relabel(int64_t m, int32_t *__restrict__ col, int64_t n_local,
                               const uint64_t *__restrict__ keys, const uint64_t *__restrict__ uniq,
                               int64_t nh) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  const uint64_t key = keys[k];
  if (key == ~0ull) return;
  int64_t lo = 0, hi = nh - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (uniq[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  col[k] = (int32_t)(n_local + lo);
}

// need[i] = position part of halo key i; hoff[j] = first halo entry of slot j
__global__ void k_halo_need(int64_t nh, const uint64_t *__restrict__ uniq, int32_t *__restrict__ need) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nh) need[i] = (int32_t)(uniq[i] & 0xffffffffull);
}
__global__ void k_halo_slots(int64_t nh, const uint64_t *__restrict__ uniq, int nslots,
                             int64_t *__restrict__ hoff) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j > nslots) return;
  const uint64_t key = (uint64_t)j << 32;
  int64_t lo = 0, hi = nh;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (uniq[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  hoff[j] = lo;
}

// halo exchange: dst[i] = src[idx[i]]
__global__ void k_halo_gather(int64_t cnt, const int32_t *__restrict__ idx,
                              const double *__restrict__ src, double *__restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = __ldcg(src + idx[i]);
}

// per-sweep reduction words: relaxations, edge updates, sentinel, bad input
__global__ void k_shard_counts(const unsigned long long *__restrict__ out, const Scalars *__restrict__ S,
                               unsigned long long *__restrict__ agg) {
  agg[0] = out[1];
  agg[1] = out[2];
  agg[2] = out[3] == 2 ? 1ull : 0ull;
  agg[3] = S->bad_input ? 1ull : 0ull;
}

// the loop ends after a sweep with no relaxation on any rank (Q = ∅),
// a sentinel hit or bad input: later queued sweeps see the flag and return
__global__ void k_shard_stop(const unsigned long long *__restrict__ agg,
                             unsigned long long *__restrict__ stop) {
  if (agg[0] == 0ull || agg[2] || agg[3]) *stop = 1ull;
}

// in-process all-reduce (sum) of `len` u64 words over shards on one device
struct PtrSet {
  unsigned long long *p[kMaxLocal];
};
__global__ void k_local_sum(PtrSet ps, int count, int len) {
  const int k = threadIdx.x;
  if (k >= len) return;
  unsigned long long a = 0ull;
  for (int i = 0; i < count; i++) a += ps.p[i][k];
  for (int i = 0; i < count; i++) ps.p[i][k] = a;
}

// Σ (z − mean)², Σ (z − s)², Σ z² with the GLOBAL mean (reading R15)
__global__ void k_shard_meas2(int64_t n_local, double n_global, const float *__restrict__ z,
                              const float *__restrict__ s, double *__restrict__ sums) {
  __shared__ double sm[kBlock / 32];
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double mean = sums[0] / n_global;
  double P = 0, I = 0, C = 0;
  if (i < n_local) {
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

// ------------------------------------------------------------ collectives
// over the shards this process owns: 1 (NCCL) or all `world` (local)
enum RedOp { kSum, kMin, kMax };
enum RedType { kU64, kF32, kF64 };

template <class T>
static T combine(T a, T b, RedOp op) {
  return op == kSum ? a + b : op == kMin ? std::min(a, b) : std::max(a, b);
}

// in-place all-reduce of `len` words of type t
static fj_status allreduce(fj_shard **sh, int count, void **buf, size_t len, RedType t, RedOp op) {
  fj_comm *cm = sh[0]->comm;
  cudaStream_t st = cm->stream;
  if (!cm->local) {
    const ncclRedOp_t o = op == kSum ? ncclSum : op == kMin ? ncclMin : ncclMax;
    const ncclDataType_t dt = t == kU64 ? ncclUint64 : t == kF32 ? ncclFloat32 : ncclFloat64;
    FJ_NCCL(nccl()->AllReduce(buf[0], buf[0], len, dt, o, cm->nc, st));
    return FJ_OK;
  }
  if (count == 1) return FJ_OK;
  if (t == kU64 && op == kSum && len <= 32) {  // per-sweep counters: stay on the device
    PtrSet ps{};
    for (int i = 0; i < count; i++) ps.p[i] = static_cast<unsigned long long *>(buf[i]);
    count_launch();
    k_local_sum<<<1, 32, 0, st>>>(ps, count, (int)len);
    return FJ_OK;
  }
  const size_t word = t == kF32 ? 4 : 8, bytes = len * word;
  std::vector<unsigned char> h(bytes * count);
  for (int i = 0; i < count; i++)
    FJ_CUDA(cudaMemcpyAsync(h.data() + bytes * i, buf[i], bytes, cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  for (size_t k = 0; k < len; k++) {
    for (int i = 1; i < count; i++) {  // rank order, as a reduction tree would not be: fixed
      if (t == kU64) {
        auto *x = reinterpret_cast<unsigned long long *>(h.data());
        x[k] = combine(x[k], x[len * i + k], op);
      } else if (t == kF32) {
        auto *x = reinterpret_cast<float *>(h.data());
        x[k] = combine(x[k], x[len * i + k], op);
      } else {
        auto *x = reinterpret_cast<double *>(h.data());
        x[k] = combine(x[k], x[len * i + k], op);
      }
    }
  }
  for (int i = 0; i < count; i++)
    FJ_CUDA(cudaMemcpyAsync(buf[i], h.data(), bytes, cudaMemcpyHostToDevice, st));
  FJ_CUDA(cudaStreamSynchronize(st));  // h is stack-owned
  return FJ_OK;
}

// every rank's halo refreshed from its owners' current values
static fj_status exchange(fj_shard **sh, int count, double **buf) {
  fj_comm *cm = sh[0]->comm;
  cudaStream_t st = cm->stream;
  const int W = cm->world;
  if (W == 1) return FJ_OK;
  if (!cm->local) {
    const fj_shard *me = sh[0];
    const int64_t ns = me->soff[W];
    if (ns > 0) {
      count_launch();
      k_halo_gather<<<gridn(ns), kBlock, 0, st>>>(ns, me->sendidx, buf[0], me->sendbuf);
    }
    FJ_NCCL(nccl()->GroupStart());
    for (int q = 0; q < W; q++) {
      if (q == me->rank) continue;
      const int j = (q - me->rank - 1 + W) % W;
      const int64_t sc = me->soff[q + 1] - me->soff[q], rc = me->hoff[j + 1] - me->hoff[j];
      if (sc > 0)
        FJ_NCCL(nccl()->Send(me->sendbuf + me->soff[q], (size_t)sc, ncclFloat64, q, cm->nc, st));
      if (rc > 0)
        FJ_NCCL(nccl()->Recv(buf[0] + me->n_local + me->hoff[j], (size_t)rc, ncclFloat64, q,
                             cm->nc, st));
    }
    FJ_NCCL(nccl()->GroupEnd());
    return FJ_OK;
  }
  if (cm->loopback) {  // the NCCL path with copies: pack on every rank, then move
    for (int q = 0; q < count; q++) {
      const int64_t ns = sh[q]->soff[W];
      if (ns > 0) {
        count_launch();
        k_halo_gather<<<gridn(ns), kBlock, 0, st>>>(ns, sh[q]->sendidx, buf[q], sh[q]->sendbuf);
      }
    }
    for (int r = 0; r < count; r++)
      for (int j = 0; j + 1 < W; j++) {
        const int q = (r + 1 + j) % W;
        const int64_t c = sh[r]->hoff[j + 1] - sh[r]->hoff[j];
        if (c == 0) continue;
        if (sh[q]->soff[r + 1] - sh[q]->soff[r] != c) {
          set_error("fj_shard: loopback send/receive counts disagree (%d -> %d)", q, r);
          return FJ_ERR_CUDA;
        }
        FJ_CUDA(cudaMemcpyAsync(buf[r] + sh[r]->n_local + sh[r]->hoff[j],
                                sh[q]->sendbuf + sh[q]->soff[r], sizeof(double) * c,
                                cudaMemcpyDeviceToDevice, st));
      }
    return FJ_OK;
  }
  for (int r = 0; r < count; r++)
    for (int j = 0; j + 1 < W; j++) {
      const int q = (r + 1 + j) % W;
      const int64_t c = sh[r]->hoff[j + 1] - sh[r]->hoff[j];
      if (c == 0) continue;
      count_launch();
      k_halo_gather<<<gridn(c), kBlock, 0, st>>>(c, sh[r]->need + sh[r]->hoff[j], buf[q],
                                                 buf[r] + sh[r]->n_local + sh[r]->hoff[j]);
    }
  return FJ_OK;
}

static fj_status check_set(fj_shard **sh, int count, const char *who) {
  if (!sh || count < 1 || !sh[0] || !sh[0]->comm) {
    set_error("%s: need count >= 1 non-null shards", who);
    return FJ_ERR_INVALID;
  }
  fj_comm *cm = sh[0]->comm;
  if (cm->local ? count != cm->world : count != 1) {
    set_error("%s: pass %s", who, cm->local ? "all world shards of a local comm" : "exactly one shard");
    return FJ_ERR_INVALID;
  }
  for (int i = 0; i < count; i++) {
    if (!sh[i] || sh[i]->comm != cm || sh[i]->rank != (cm->local ? i : cm->rank)) {
      set_error("%s: shards must share one comm and come in rank order", who);
      return FJ_ERR_INVALID;
    }
  }
  return FJ_OK;
}

// ------------------------------------------------------------------ create
static fj_status shard_create_impl(fj_comm *cm, int rank, int64_t n, const int64_t *begin,
                                   const int64_t *rp_in, const int32_t *col_in, const float *w_in,
                                   int directed, fj_shard *s) {
  cudaStream_t st = cm->stream;
  const int W = cm->world;
  s->comm = cm;
  s->rank = rank;
  s->n = n;
  s->begin.assign(begin, begin + W + 1);
  s->n_local = begin[rank + 1] - begin[rank];
  for (int r = 0; r < W; r++) s->seg_max = std::max(s->seg_max, begin[r + 1] - begin[r]);
  s->nz = s->n_local;  // + halo, set by fj_shard_connect
  int64_t m = 0;
  FJ_CUDA(cudaMemcpy(&m, rp_in + s->n_local, sizeof(int64_t), cudaMemcpyDefault));
  if (m < 0 || m >= (int64_t(1) << 40) || (m > 0 && !col_in)) {
    set_error("fj_shard_create: out_row_ptr[n_local] = %lld out of range or out_col NULL",
              (long long)m);
    return FJ_ERR_INVALID;
  }
  fj_graph *g = new fj_graph();
  s->g = g;
  g->n = s->n_local;
  g->m = m;
  g->directed = directed ? 1 : 0;
  g->weighted = w_in ? 1 : 0;
  g->stream = st;
  g->num_sms = cm->num_sms;
  Workspace ws(st);  // staged input and temporaries
  int64_t *rp = nullptr;
  int32_t *col = nullptr, *enc = nullptr;
  float *w = nullptr;
  int *err = nullptr;
  const int64_t nl = s->n_local;
  FJ_CUDA(ws.alloc(&rp, (nl + 1)));
  FJ_CUDA(ws.alloc(&col, (m + 8)));
  FJ_CUDA(ws.alloc(&enc, (m + 8)));
  if (w_in) FJ_CUDA(ws.alloc(&w, (m + 8)));
  FJ_CUDA(ws.alloc(&err, 1));
  FJ_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  FJ_CUDA(cudaMemcpyAsync(rp, rp_in, sizeof(int64_t) * (nl + 1), cudaMemcpyDefault, st));
  if (m > 0) {
    FJ_CUDA(cudaMemcpyAsync(col, col_in, sizeof(int32_t) * m, cudaMemcpyDefault, st));
    if (w_in) FJ_CUDA(cudaMemcpyAsync(w, w_in, sizeof(float) * m, cudaMemcpyDefault, st));
  }
  int herr = 0;
  count_launch();
  k_shard_rowptr<<<gridn(nl + 1), kBlock, 0, st>>>(nl, m, rp, err);
  FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  if (herr) {
    set_error("fj_shard_create: out_row_ptr must start at 0, be non-decreasing and end at nnz");
    return FJ_ERR_INVALID;
  }
  const unsigned wgrid = (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((nl * 32 + kBlock - 1) / kBlock, (int64_t)cm->num_sms * 64));
  count_launch();
  k_shard_rows<<<wgrid, kBlock, 0, st>>>(nl, begin[rank], n, rp, col, w, enc, err);
  FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  if (herr) {
    set_error("fj_shard_create: %s%s%s%s", herr & 2 ? "column id out of range; " : "",
              herr & 4 ? "self-loop; " : "", herr & 8 ? "weight not positive and finite; " : "",
              herr & 16 ? "row not strictly increasing (unsorted or duplicate arc); " : "");
    return FJ_ERR_INVALID;
  }
  FJ_CUDA(cudaMallocAsync(&g->deg, sizeof(double) * nl, st));
  count_launch();
  k_shard_rowsum<<<wgrid, kBlock, 0, st>>>(nl, rp, w, g->deg);
  fj_status rc = build_layout_from_out(g, rp, enc, w, nullptr, 1, &g->async_layout);
  FJ_CUDA(cudaStreamSynchronize(st));
  return rc;
}

static fj_status connect_impl(fj_shard **sh, int count) {
  fj_comm *cm = sh[0]->comm;
  cudaStream_t st = cm->stream;
  const int W = cm->world;
  const int64_t seg = sh[0]->seg_max;
  Workspace ws(st);  // temporaries; the halo lists belong to the shards
  std::vector<int32_t *> pad(count), all(count);
  for (int i = 0; i < count; i++) {
    FJ_CUDA(ws.alloc(&pad[i], seg));
    FJ_CUDA(ws.alloc(&all[i], seg * W));
    FJ_CUDA(cudaMemsetAsync(pad[i], 0xff, sizeof(int32_t) * seg, st));
    FJ_CUDA(cudaMemcpyAsync(pad[i], sh[i]->g->async_layout.iperm, sizeof(int32_t) * sh[i]->n_local,
                            cudaMemcpyDeviceToDevice, st));
  }
  if (!cm->local) {
    FJ_NCCL(nccl()->AllGather(pad[0], all[0], (size_t)seg, ncclInt32, cm->nc, st));
  } else {
    for (int i = 0; i < count; i++)
      for (int r = 0; r < count; r++)
        FJ_CUDA(cudaMemcpyAsync(all[i] + (int64_t)r * seg, pad[r], sizeof(int32_t) * seg,
                                cudaMemcpyDeviceToDevice, st));
  }
  int *err = nullptr;
  int64_t *dbeg = nullptr;
  FJ_CUDA(ws.alloc(&err, 1));
  FJ_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  FJ_CUDA(ws.alloc(&dbeg, (W + 1)));
  FJ_CUDA(cudaMemcpyAsync(dbeg, sh[0]->begin.data(), sizeof(int64_t) * (W + 1),
                          cudaMemcpyHostToDevice, st));
  // per shard: halo keys of the remote columns, sorted and made unique → the
  // halo order; remote columns relabelled to their halo entry
  int herr = 0;
  std::vector<std::vector<int64_t>> need_from(count, std::vector<int64_t>(W, 0));
  for (int i = 0; i < count; i++) {
    fj_shard *S = sh[i];
    Layout &L = S->g->async_layout;
    const int64_t m = L.m;
    uint64_t *keys = nullptr, *k1 = nullptr, *uq = nullptr;
    int64_t *nsel = nullptr, *dhoff = nullptr;
    FJ_CUDA(ws.alloc(&keys, std::max<int64_t>(1, m)));
    FJ_CUDA(ws.alloc(&k1, std::max<int64_t>(1, m)));
    FJ_CUDA(ws.alloc(&uq, std::max<int64_t>(1, m)));
    FJ_CUDA(ws.alloc(&nsel, 1));
    FJ_CUDA(ws.alloc(&dhoff, W));
    FJ_CUDA(cudaMemsetAsync(nsel, 0, sizeof(int64_t), st));
    int64_t nu = 0;
    if (m > 0) {
      count_launch();
      k_halo_keys<<<gridn(m), kBlock, 0, st>>>(m, L.col, S->n_local, S->rank, W, seg, dbeg, all[i],
                                               keys, err);
      size_t t1 = 0, t2 = 0;
      FJ_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, keys, k1, m, 0, 64, st));
      FJ_CUDA(cub::DeviceSelect::Unique(nullptr, t2, k1, uq, nsel, m, st));
      unsigned char *t = nullptr;
      FJ_CUDA(ws.alloc(&t, std::max(t1, t2)));
      FJ_CUDA(cub::DeviceRadixSort::SortKeys(t, t1, keys, k1, m, 0, 64, st));
      FJ_CUDA(cub::DeviceSelect::Unique(t, t2, k1, uq, nsel, m, st));
      FJ_CUDA(cudaMemcpyAsync(&nu, nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      FJ_CUDA(cudaStreamSynchronize(st));
      if (nu > 0) {  // the own-column sentinel sorts last
        uint64_t last = 0;
        FJ_CUDA(cudaMemcpyAsync(&last, uq + nu - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        FJ_CUDA(cudaStreamSynchronize(st));
        if (last == ~0ull) nu--;
      }
    }
    S->hoff.assign(W, 0);
    if (nu > 0) {
      count_launch();
      k_halo_relabel<<<gridn(m), kBlock, 0, st>>>(m, L.col, S->n_local, keys, uq, nu);
      FJ_CUDA(cudaMallocAsync(&S->need, sizeof(int32_t) * nu, st));
      count_launch();
      k_halo_need<<<gridn(nu), kBlock, 0, st>>>(nu, uq, S->need);
      count_launch();
      k_halo_slots<<<1, 128, 0, st>>>(nu, uq, W - 1, dhoff);
      FJ_CUDA(cudaMemcpyAsync(S->hoff.data(), dhoff, sizeof(int64_t) * W, cudaMemcpyDeviceToHost, st));
    }
    FJ_CUDA(cudaStreamSynchronize(st));
    S->hoff[W - 1] = nu;
    S->nz = S->n_local + nu;
    for (int j = 0; j + 1 < W; j++) need_from[i][(S->rank + 1 + j) % W] = S->hoff[j + 1] - S->hoff[j];
  }
  // NCCL (and loopback): every rank learns what each peer reads from it — its
  // send lists; hc[q·W + r] = how many values rank q reads from rank r
  if ((!cm->local || cm->loopback) && W > 1) {
    std::vector<int64_t> hc((size_t)W * W, 0);
    if (!cm->local) {
      int64_t *cnt = nullptr;
      FJ_CUDA(ws.alloc(&cnt, W * (W + 1)));
      FJ_CUDA(cudaMemcpyAsync(cnt + (int64_t)W * W, need_from[0].data(), sizeof(int64_t) * W,
                              cudaMemcpyHostToDevice, st));
      FJ_NCCL(nccl()->AllGather(cnt + (int64_t)W * W, cnt, (size_t)W, ncclInt64, cm->nc, st));
      FJ_CUDA(cudaMemcpyAsync(hc.data(), cnt, sizeof(int64_t) * W * W, cudaMemcpyDeviceToHost, st));
      FJ_CUDA(cudaStreamSynchronize(st));
    } else {
      for (int i = 0; i < count; i++)
        for (int q = 0; q < W; q++) hc[(size_t)i * W + q] = need_from[i][q];
    }
    for (int i = 0; i < count; i++) {
      fj_shard *me = sh[i];
      me->soff.assign(W + 1, 0);
      for (int q = 0; q < W; q++)
        me->soff[q + 1] = me->soff[q] + (q == me->rank ? 0 : hc[(size_t)q * W + me->rank]);
      const int64_t ns = me->soff[W];
      FJ_CUDA(cudaMallocAsync(&me->sendidx, sizeof(int32_t) * std::max<int64_t>(1, ns), st));
      FJ_CUDA(cudaMallocAsync(&me->sendbuf, sizeof(double) * std::max<int64_t>(1, ns), st));
    }
    if (!cm->local) {
      fj_shard *me = sh[0];
      FJ_NCCL(nccl()->GroupStart());
      for (int q = 0; q < W; q++) {
        if (q == me->rank) continue;
        const int j = (q - me->rank - 1 + W) % W;
        const int64_t rc = me->hoff[j + 1] - me->hoff[j], sc = me->soff[q + 1] - me->soff[q];
        if (rc > 0)
          FJ_NCCL(nccl()->Send(me->need + me->hoff[j], (size_t)rc, ncclInt32, q, cm->nc, st));
        if (sc > 0)
          FJ_NCCL(nccl()->Recv(me->sendidx + me->soff[q], (size_t)sc, ncclInt32, q, cm->nc, st));
      }
      FJ_NCCL(nccl()->GroupEnd());
    } else {  // loopback: reader r's need list for q becomes q's send list for r
      for (int r = 0; r < count; r++)
        for (int j = 0; j + 1 < W; j++) {
          const int q = (r + 1 + j) % W;
          const int64_t rc = sh[r]->hoff[j + 1] - sh[r]->hoff[j];
          if (rc > 0)
            FJ_CUDA(cudaMemcpyAsync(sh[q]->sendidx + sh[q]->soff[r], sh[r]->need + sh[r]->hoff[j],
                                    sizeof(int32_t) * rc, cudaMemcpyDeviceToDevice, st));
        }
    }
  }
  FJ_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  FJ_CUDA(cudaStreamSynchronize(st));
  if (herr) {
    set_error("fj_shard_connect: inconsistent partitions across ranks");
    return FJ_ERR_INVALID;
  }
  for (int i = 0; i < count; i++) sh[i]->connected = true;
  return FJ_OK;
}

// ------------------------------------------------------------------- solve
struct ShardWork {
  Staged s{};
  float *s_l = nullptr, *smm = nullptr, *zo = nullptr;
  double *z = nullptr, *zp = nullptr;
  double2 *partial = nullptr;
  int *arrive = nullptr;
  Scalars *S = nullptr;
  unsigned *ctl = nullptr;
  SweepCounters *cnt = nullptr;
  unsigned long long *outv = nullptr, *stop = nullptr, *agg = nullptr;  // agg: [batch][4]
  KP p{};
};

static fj_status shard_solve_impl(fj_shard **sh, int count, const float *const *s_in, double eps,
                                  double omega, const fj_opts *o, float *const *z_out,
                                  double *const *zp_out, fj_stats *st_out) {
  NvtxRange nv("fj_shard_solve");
  fj_comm *cm = sh[0]->comm;
  cudaStream_t st = cm->stream;
  fj_stats stats{};
  stats.colors = 1;
  std::vector<ShardWork> wk(count);
  std::vector<void *> red(count);
  std::vector<double *> zb(count);
  Workspace ws(st);
  cudaEvent_t e0, e1, es0, es1;
  for (cudaEvent_t *e : {&e0, &e1, &es0, &es1}) FJ_CUDA(ws.event(e));
  FJ_CUDA(cudaEventRecord(e0, st));
  for (int i = 0; i < count; i++) {
    ShardWork &w = wk[i];
    const Layout &L = sh[i]->g->async_layout;
    const int64_t nl = sh[i]->n_local;
    FJ_TRY(stage_in(s_in[i], nl, ws, w.s));
    FJ_CUDA(ws.alloc(&w.s_l, nl));
    FJ_CUDA(ws.alloc(&w.smm, 2));
    FJ_CUDA(ws.alloc(&w.z, sh[i]->nz));
    FJ_CUDA(cudaMemsetAsync(w.z, 0, sizeof(double) * sh[i]->nz, st));
    FJ_CUDA(ws.alloc(&w.S, 1));
    FJ_CUDA(ws.alloc(&w.partial, std::max(1, L.npartials)));
    FJ_CUDA(ws.alloc(&w.arrive, std::max(1, L.npartials)));
    FJ_CUDA(cudaMemsetAsync(w.arrive, 0, sizeof(int) * std::max(1, L.npartials), st));
    FJ_CUDA(ws.alloc(&w.ctl, kCtlWords));
    FJ_CUDA(ws.alloc(&w.cnt, 3));
    FJ_CUDA(ws.alloc(&w.outv, (9 + 4 * kSweepBatch)));
    w.stop = w.outv + 8;
    w.agg = w.outv + 9;
    if (!is_device_ptr(z_out[i])) FJ_CUDA(ws.alloc(&w.zo, nl));
    if (zp_out && zp_out[i] && !is_device_ptr(zp_out[i]))
      FJ_CUDA(ws.alloc(&w.zp, nl));
    FJ_TRY(minmax_f32(w.s.dev, nl, w.smm, ws, cm->num_sms));
  }
  // a2: global shift from the global min / max of s (Alg. 2)
  {
    std::vector<void *> lo(count), hi(count);
    for (int i = 0; i < count; i++) {
      lo[i] = wk[i].smm;
      hi[i] = wk[i].smm + 1;
    }
    FJ_TRY(allreduce(sh, count, lo.data(), 1, kF32, kMin));
    FJ_TRY(allreduce(sh, count, hi.data(), 1, kF32, kMax));
  }
  for (int i = 0; i < count; i++) {
    ShardWork &w = wk[i];
    const Layout &L = sh[i]->g->async_layout;
    count_launch();
    k_scalars<<<1, 1, 0, st>>>(w.smm, w.smm + 1, eps, o->sigma, o->c, w.S);
    count_launch();
    k_init<<<gridn(sh[i]->n_local), kBlock, 0, st>>>(sh[i]->n_local, L.perm, L.rp, w.s.dev, w.S,
                                                     w.s_l, w.z, nullptr);
    KP &p = w.p;
    p = make_kp(sh[i]->g, L);
    p.s = w.s_l;
    p.z = w.z;
    p.sc = w.S;
    p.omega = omega;
    p.theta = 1.0;
    p.partial = w.partial;
    p.arrive = w.arrive;
    p.max_sweeps = 1;  // one sweep per launch: the exchange follows every sweep
    p.ctr = w.ctl;
    p.bar = w.ctl + 8;
    p.cnt = w.cnt;
    p.out = w.outv;
    p.cert_max = w.outv + 4;
    p.stop = w.stop;
    zb[i] = w.z;
  }
  FJ_TRY(exchange(sh, count, zb.data()));

  const bool W = sh[0]->g->weighted != 0;
  const void *fn = sweep_kernel(W);
  const size_t smem = sweep_kernel_smem();
  FJ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = persistent_grid(fn, cm->num_sms, smem);
  const void *cf = W ? (const void *)k_pass<CERT, true> : (const void *)k_pass<CERT, false>;
  const int cgrid = persistent_grid(cf, cm->num_sms);
  float ms_sweep = 0.f;
  int rounds = 0, max_sweeps = o->max_sweeps;
  unsigned long long bad_input = 0;
  double theta = 1.0;
  for (;;) {
    int sw = 0;
    stats.reason = 1;
    for (int i = 0; i < count; i++) {
      wk[i].p.theta = theta;
      FJ_CUDA(cudaMemsetAsync(wk[i].stop, 0, sizeof(unsigned long long), st));
    }
    // queue a batch of sweeps (sweep → counters → all-reduce → stop flag →
    // exchange); the host reads the batch's counters once.  Sweeps queued
    // after the stopping one return at once (k_sweep reads the flag).
    while (sw < max_sweeps && stats.reason == 1) {
      const int nb = std::min(kSweepBatch, max_sweeps - sw);
      FJ_CUDA(cudaEventRecord(es0, st));
      for (int j = 0; j < nb; j++) {
        for (int i = 0; i < count; i++) {
          ShardWork &w = wk[i];
          FJ_CUDA(cudaMemsetAsync(w.ctl, 0, sizeof(unsigned) * kCtlWords, st));
          FJ_CUDA(cudaMemsetAsync(w.cnt, 0, sizeof(SweepCounters) * 3, st));
          FJ_CUDA(cudaMemsetAsync(w.outv, 0, sizeof(unsigned long long) * 4, st));
          void *args[] = {&w.p};
          count_launch();
          FJ_CUDA(cudaLaunchCooperativeKernel(fn, grid, kBlock, args, smem, st));
          count_launch();
          k_shard_counts<<<1, 1, 0, st>>>(w.outv, w.S, w.agg + 4 * j);
          red[i] = w.agg + 4 * j;
        }
        FJ_TRY(allreduce(sh, count, red.data(), 4, kU64, kSum));
        for (int i = 0; i < count; i++) {
          count_launch();
          k_shard_stop<<<1, 1, 0, st>>>(wk[i].agg + 4 * j, wk[i].stop);
        }
        FJ_TRY(exchange(sh, count, zb.data()));
      }
      FJ_CUDA(cudaEventRecord(es1, st));
      std::vector<unsigned long long> h(4 * nb);
      FJ_CUDA(cudaMemcpyAsync(h.data(), wk[0].agg, sizeof(unsigned long long) * 4 * nb,
                              cudaMemcpyDeviceToHost, st));
      FJ_CUDA(cudaStreamSynchronize(st));
      float a = 0.f;
      FJ_CUDA(cudaEventElapsedTime(&a, es0, es1));
      ms_sweep += a;
      for (int j = 0; j < nb; j++) {
        const unsigned long long *q = h.data() + 4 * j;
        sw++;
        stats.sweeps++;
        stats.relaxations += (int64_t)q[0];
        stats.edge_updates += (int64_t)q[1];
        bad_input |= q[3];
        if (q[2] || q[3]) {
          stats.reason = 2;
          break;
        }
        if (q[0] == 0) {  // no rank relaxed: Q = ∅
          stats.reason = 0;
          break;
        }
      }
    }
    if (stats.reason != 0 || !o->certify) break;
    // fp64 compensated certificate on every rank; the maximum decides
    std::vector<void *> cb(count);
    for (int i = 0; i < count; i++) {
      ShardWork &w = wk[i];
      FJ_CUDA(cudaMemsetAsync(w.outv + 4, 0, sizeof(unsigned long long), st));
      KP q = w.p;
      q.ctr = w.ctl + 5;
      void *cargs[] = {&q};
      count_launch();
      FJ_CUDA(cudaLaunchKernel(cf, cgrid, kBlock, cargs, 0, st));
      cb[i] = w.outv + 4;
    }
    FJ_TRY(allreduce(sh, count, cb.data(), 1, kU64, kMax));  // non-negative doubles order as bits
    unsigned long long hb = 0;
    FJ_CUDA(cudaMemcpyAsync(&hb, wk[0].outv + 4, sizeof(hb), cudaMemcpyDeviceToHost, st));
    FJ_CUDA(cudaStreamSynchronize(st));
    stats.cert_ratio = __builtin_bit_cast(double, hb);
    if (stats.cert_ratio <= 1.0 || rounds >= o->cert_rounds) break;
    rounds++;  // resume from ẑ with a stricter sweep threshold (reading R21)
    theta *= 0.5;
    max_sweeps = std::min(o->max_sweeps, 2000);
  }
  stats.cert_rounds = rounds;
  stats.phases = stats.sweeps;
  int64_t active = 0, arcs = 0, empty = 0;
  for (int i = 0; i < count; i++) {
    active += sh[i]->g->async_layout.active_rows;
    arcs += sh[i]->g->async_layout.m;
    empty += sh[i]->g->async_layout.empty_rows;
  }
  stats.rows_read = stats.sweeps * active;  // this process's shards
  stats.arcs_read = stats.sweeps * arcs;
  stats.relaxations += empty;

  // a6: unshift into each shard's slice
  Scalars hs{};
  for (int i = 0; i < count; i++) {
    ShardWork &w = wk[i];
    const int64_t nl = sh[i]->n_local;
    float *zo = w.zo ? w.zo : z_out[i];
    double *zp = (zp_out && zp_out[i]) ? (w.zp ? w.zp : zp_out[i]) : nullptr;
    count_launch();
    k_finalize<<<gridn(nl), kBlock, 0, st>>>(nl, sh[i]->g->async_layout.iperm, w.z, w.S, zo, zp);
    if (w.zo) FJ_CUDA(cudaMemcpyAsync(z_out[i], w.zo, sizeof(float) * nl, cudaMemcpyDeviceToHost, st));
    if (w.zp) FJ_CUDA(cudaMemcpyAsync(zp_out[i], w.zp, sizeof(double) * nl, cudaMemcpyDeviceToHost, st));
  }
  FJ_CUDA(cudaMemcpyAsync(&hs, wk[0].S, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaEventRecord(e1, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  float ms = 0.f;
  FJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  stats.solve_ms = ms;
  stats.sweep_ms = ms_sweep;
  stats.c = hs.c;
  stats.eps_prime = hs.eps_p;
  hs.bad_input = bad_input ? 1 : 0;
  FJ_CUDA(cudaStreamSynchronize(st));
  FJ_CUDA(cudaGetLastError());
  fj_status rc = finish_status(hs, stats, o, omega);
  if (st_out) *st_out = stats;
  return rc;
}

static fj_status shard_measures_impl(fj_shard **sh, int count, const float *const *z_in,
                                     const float *const *s_in, fj_measures_t *out) {
  NvtxRange nv("fj_shard_measures");
  fj_comm *cm = sh[0]->comm;
  cudaStream_t st = cm->stream;
  Workspace ws(st);
  std::vector<Staged> z(count), s(count);
  std::vector<double *> zl(count), sums(count);
  std::vector<void *> red(count);
  std::vector<unsigned *> ctr(count);
  for (int i = 0; i < count; i++) {
    const int64_t nl = sh[i]->n_local;
    FJ_TRY(stage_in(z_in[i], nl, ws, z[i]));
    if (s_in && s_in[i]) FJ_TRY(stage_in(s_in[i], nl, ws, s[i]));
    FJ_CUDA(ws.alloc(&zl[i], sh[i]->nz));
    FJ_CUDA(cudaMemsetAsync(zl[i], 0, sizeof(double) * sh[i]->nz, st));
    FJ_CUDA(ws.alloc(&sums[i], 5));
    FJ_CUDA(cudaMemsetAsync(sums[i], 0, sizeof(double) * 5, st));
    FJ_CUDA(ws.alloc(&ctr[i], 1));
    FJ_CUDA(cudaMemsetAsync(ctr[i], 0, sizeof(unsigned), st));
    count_launch();
    k_meas_nodes1<<<gridn(nl), kBlock, 0, st>>>(nl, sh[i]->g->async_layout.perm, z[i].dev, zl[i],
                                                 sums[i]);
    red[i] = sums[i];
  }
  // remote z for the arc pass, then D along the owned out-rows
  FJ_TRY(exchange(sh, count, zl.data()));
  const bool W = sh[0]->g->weighted != 0;
  const void *fn = W ? (const void *)k_pass<DIS, true> : (const void *)k_pass<DIS, false>;
  for (int i = 0; i < count; i++) {
    KP p = make_kp(sh[i]->g, sh[i]->g->async_layout);
    p.z = zl[i];
    p.ctr = ctr[i];
    p.dis = sums[i] + 4;
    void *args[] = {&p};
    count_launch();
    FJ_CUDA(cudaLaunchKernel(fn, persistent_grid(fn, cm->num_sms), kBlock, args, 0, st));
  }
  // global Σ z → mean on every rank, then the node sums with that mean
  FJ_TRY(allreduce(sh, count, red.data(), 1, kF64, kSum));
  for (int i = 0; i < count; i++) {
    count_launch();
    k_shard_meas2<<<gridn(sh[i]->n_local), kBlock, 0, st>>>(
        sh[i]->n_local, (double)sh[i]->n, z[i].dev, (s_in && s_in[i]) ? s[i].dev : nullptr, sums[i]);
  }
  std::vector<void *> tail(count);
  for (int i = 0; i < count; i++) tail[i] = sums[i] + 1;
  FJ_TRY(allreduce(sh, count, tail.data(), 4, kF64, kSum));
  double h[5];
  FJ_CUDA(cudaMemcpyAsync(h, sums[0], sizeof(h), cudaMemcpyDeviceToHost, st));
  FJ_CUDA(cudaStreamSynchronize(st));
  FJ_CUDA(cudaStreamSynchronize(st));
  FJ_CUDA(cudaGetLastError());
  out->polarization = h[1];
  out->disagreement = sh[0]->g->directed ? h[4] : 0.5 * h[4];  // reading R14
  out->internal_conflict = (s_in && s_in[0]) ? h[2] : 0.0;
  out->controversy = h[3];
  return FJ_OK;
}

}  // namespace fj

// ------------------------------------------------------------------- C-ABI
extern "C" {

fj_status fj_shard_plan(int64_t n, const int64_t *row_ptr, int world, int64_t *begin) {
  if (n < 1 || world < 1 || world > n || !row_ptr || !begin) {
    fj::set_error("fj_shard_plan: need 1 <= world <= n and non-null row_ptr, begin");
    return FJ_ERR_INVALID;
  }
  const int64_t m = row_ptr[n];
  if (row_ptr[0] != 0 || m < 0) {
    fj::set_error("fj_shard_plan: row_ptr must start at 0 and end at nnz >= 0");
    return FJ_ERR_INVALID;
  }
  for (int64_t u = 0; u < n; u++)
    if (row_ptr[u + 1] < row_ptr[u]) {
      fj::set_error("fj_shard_plan: row_ptr must be non-decreasing");
      return FJ_ERR_INVALID;
    }
  // work of rows [0, u) = row_ptr[u] + u (arcs plus one per row)
  const double total = (double)m + (double)n;
  begin[0] = 0;
  int64_t u = 0;
  for (int r = 1; r < world; r++) {
    const double target = total * r / world;
    while (u < n && (double)(row_ptr[u] + u) < target) u++;
    begin[r] = std::min(std::max(u, begin[r - 1] + 1), n - (world - r));
    u = begin[r];
  }
  begin[world] = n;
  return FJ_OK;
}

fj_status fj_comm_unique_id(void *id128) {
  if (!id128) {
    fj::set_error("fj_comm_unique_id: null id");
    return FJ_ERR_INVALID;
  }
  if (!fj::nccl()) {
    fj::set_error("fj_comm_unique_id: libnccl.so.2 could not be loaded");
    return FJ_ERR_CUDA;
  }
  ncclUniqueId id;
  FJ_NCCL(fj::nccl()->GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "NCCL unique id size");
  memcpy(id128, &id, sizeof(id));
  return FJ_OK;
}

static fj_status comm_base(fj_comm *c) {
  int dev = 0;
  FJ_CUDA(cudaGetDevice(&dev));
  FJ_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev));
  FJ_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;  // keep stream-ordered allocations pooled (as graph.cu)
  FJ_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = ~0ull;
  FJ_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  return FJ_OK;
}

fj_status fj_comm_create(const void *id128, int rank, int world, fj_comm_t *out) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world) {
    fj::set_error("fj_comm_create: need id, 0 <= rank < world, out");
    return FJ_ERR_INVALID;
  }
  *out = nullptr;
  if (!fj::nccl()) {
    fj::set_error("fj_comm_create: libnccl.so.2 could not be loaded");
    return FJ_ERR_CUDA;
  }
  fj_comm *c = new fj_comm();
  c->world = world;
  c->rank = rank;
  c->local = false;
  fj_status s = comm_base(c);
  if (s == FJ_OK) {
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclResult_t r = fj::nccl()->CommInitRank(&c->nc, world, id, rank);
    if (r != ncclSuccess) {
      fj::set_error("NCCL ncclCommInitRank: %s", fj::nccl()->GetErrorString(r));
      s = FJ_ERR_CUDA;
    }
  }
  if (s != FJ_OK) {
    fj_comm_destroy(c);
    return s;
  }
  *out = c;
  return FJ_OK;
}

static fj_status comm_create_local(int world, bool loopback, fj_comm_t *out) {
  if (!out || world < 1 || world > fj::kMaxLocal) {
    fj::set_error("fj_comm_create_local: need 1 <= world <= %d and out", fj::kMaxLocal);
    return FJ_ERR_INVALID;
  }
  *out = nullptr;
  fj_comm *c = new fj_comm();
  c->world = world;
  c->local = true;
  c->loopback = loopback;
  fj_status s = comm_base(c);
  if (s != FJ_OK) {
    fj_comm_destroy(c);
    return s;
  }
  *out = c;
  return FJ_OK;
}

fj_status fj_comm_create_local(int world, fj_comm_t *out) { return comm_create_local(world, false, out); }

fj_status fj_comm_create_loopback(int world, fj_comm_t *out) { return comm_create_local(world, true, out); }

fj_status fj_comm_destroy(fj_comm_t c) {
  if (!c) return FJ_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->nc && fj::nccl()) fj::nccl()->CommDestroy(c->nc);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return FJ_OK;
}

fj_status fj_shard_create(fj_comm_t comm, int rank, int64_t n, const int64_t *begin,
                          const int64_t *out_row_ptr, const int32_t *out_col, const float *out_w,
                          int directed, fj_shard_t *out) {
  if (!out) {
    fj::set_error("fj_shard_create: out is NULL");
    return FJ_ERR_INVALID;
  }
  *out = nullptr;
  if (!comm || !begin || !out_row_ptr || rank < 0 || rank >= comm->world || n < 1 ||
      n >= (int64_t(1) << 30)) {
    fj::set_error("fj_shard_create: need comm, begin, row_ptr, 0 <= rank < world, 1 <= n < 2^30");
    return FJ_ERR_INVALID;
  }
  if (!comm->local && rank != comm->rank) {
    fj::set_error("fj_shard_create: rank %d on the NCCL comm of rank %d", rank, comm->rank);
    return FJ_ERR_INVALID;
  }
  if (begin[0] != 0 || begin[comm->world] != n) {
    fj::set_error("fj_shard_create: begin[0] must be 0 and begin[world] = n");
    return FJ_ERR_INVALID;
  }
  for (int r = 0; r < comm->world; r++)
    if (begin[r + 1] <= begin[r]) {
      fj::set_error("fj_shard_create: every part must be non-empty (begin strictly increasing)");
      return FJ_ERR_INVALID;
    }
  fj_shard *s = new fj_shard();
  nvtxRangePushA("fj_shard_create");
  fj_status rc = fj::shard_create_impl(comm, rank, n, begin, out_row_ptr, out_col, out_w, directed, s);
  nvtxRangePop();
  if (rc != FJ_OK) {
    fj_shard_destroy(s);
    return rc;
  }
  *out = s;
  return FJ_OK;
}

fj_status fj_shard_connect(fj_shard_t *shards, int count) {
  FJ_TRY(fj::check_set(shards, count, "fj_shard_connect"));
  return fj::connect_impl(shards, count);
}

fj_status fj_shard_solve(fj_shard_t *shards, int count, const float *const *s, double eps,
                         double omega, const fj_opts *o, float *const *z_out,
                         double *const *zprime_out, fj_stats *st) {
  FJ_TRY(fj::check_set(shards, count, "fj_shard_solve"));
  for (int i = 0; i < count; i++)
    if (!shards[i]->connected) {
      fj::set_error("fj_shard_solve: call fj_shard_connect first");
      return FJ_ERR_INVALID;
    }
  fj_opts d;
  fj_opts_default(&d);
  if (o) d = *o;
  if (d.sigma <= 0) d.sigma = 1e-5;
  if (d.max_sweeps <= 0) d.max_sweeps = 1000000;
  if (d.cert_rounds < 0) d.cert_rounds = 3;
  if (!s || !z_out || !(eps > 0 && eps < 1) || !(omega > 0 && omega < 2) ||
      (d.method != FJ_METHOD_AUTO && d.method != FJ_METHOD_ASYNC) || d.z_init || d.zprime_out) {
    fj::set_error("fj_shard_solve: need s, z_out, 0 < eps < 1, 0 < omega < 2, method AUTO/ASYNC, "
                  "no z_init / zprime_out in opts");
    return FJ_ERR_INVALID;
  }
  for (int i = 0; i < count; i++)
    if (!s[i] || !z_out[i]) {
      fj::set_error("fj_shard_solve: null s[%d] or z_out[%d]", i, i);
      return FJ_ERR_INVALID;
    }
  return fj::shard_solve_impl(shards, count, s, eps, omega, &d, z_out, zprime_out, st);
}

fj_status fj_shard_measures(fj_shard_t *shards, int count, const float *const *z,
                            const float *const *s, fj_measures_t *out) {
  FJ_TRY(fj::check_set(shards, count, "fj_shard_measures"));
  if (!z || !out) {
    fj::set_error("fj_shard_measures: need z and out");
    return FJ_ERR_INVALID;
  }
  for (int i = 0; i < count; i++)
    if (!shards[i]->connected || !z[i]) {
      fj::set_error("fj_shard_measures: shard %d not connected or z[%d] null", i, i);
      return FJ_ERR_INVALID;
    }
  return fj::shard_measures_impl(shards, count, z, s, out);
}

fj_status fj_shard_info(fj_shard_t s, int64_t *n_local, int64_t *halo) {
  if (!s || !n_local || !halo) {
    fj::set_error("fj_shard_info: null argument");
    return FJ_ERR_INVALID;
  }
  *n_local = s->n_local;
  *halo = s->connected ? s->nz - s->n_local : 0;
  return FJ_OK;
}

fj_status fj_shard_destroy(fj_shard_t s) {
  if (!s) return FJ_OK;
  for (void *q : {(void *)s->need, (void *)s->sendidx, (void *)s->sendbuf})
    if (q) cudaFree(q);
  if (s->g) fj_graph_destroy(s->g);
  delete s;
  return FJ_OK;
}

}  // extern "C"
