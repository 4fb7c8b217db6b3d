// prims.cu — device primitives of the graph build (§8 row a1) and the shift
// (row a2), hand-written: min/max of the opinions, max of row lengths, an
// exclusive scan, and a stable LSD radix sort of (key, payload) pairs.
//
// Radix sort: 8-bit digits, one pass per digit, each pass a blocked stable
// counting sort — (1) every CTA counts the digits of its tile of kTile keys,
// (2) an exclusive scan over the digit-major count table gives every (digit,
// tile) its output offset, (3) every CTA ranks its keys stably (tile order =
// input order: rounds of kBlock keys, warp match for the rank inside a warp,
// shared-memory counts for the warps and rounds before) and scatters keys and
// payloads.  Stability makes the passes compose into a sort by the whole key
// that keeps the input order of equal keys (the transpose relies on it: the
// out-row of u lists its v ascending because the in-CSR is visited by v).
#include <stdint.h>

#include "fj_internal.cuh"

namespace fj {

constexpr int kRadix = 256;                 // 8-bit digits
constexpr int kTileItems = 16;              // keys per thread per tile
constexpr int kTile = kBlock * kTileItems;  // keys per tile (one CTA)

static unsigned nblocks_for(int64_t work, int64_t per) {
  const int64_t b = (work + per - 1) / per;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 1 << 30));
}

// ---------------------------------------------------------------- min / max
// float order-preserving map to signed ints (for atomicMin / atomicMax)
__device__ __forceinline__ int f2ord(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float ord2f(int i) { return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff); }

__global__ void k_minmax_init(int *mm) {
  mm[0] = 0x7fffffff;  // > every ordered float
  mm[1] = (int)0x80000000;
}
// NaN entries are skipped (fminf / fmaxf), as the sweep's init flags them
__global__ void k_minmax(int64_t n, const float *__restrict__ x, int *__restrict__ mm) {
  float lo = INFINITY, hi = -INFINITY;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, f2ord(lo));
    atomicMax(mm + 1, f2ord(hi));
  }
}
__global__ void k_minmax_out(const int *__restrict__ mm, float *__restrict__ out) {
  out[0] = ord2f(mm[0]);
  out[1] = ord2f(mm[1]);
}

fj_status minmax_f32(const float *x, int64_t n, float *out2, Workspace &ws, int num_sms) {
  int *mm = nullptr;
  FJ_CUDA(ws.alloc(&mm, 2));
  count_launch();
  k_minmax_init<<<1, 1, 0, ws.st>>>(mm);
  count_launch();
  k_minmax<<<std::min<unsigned>(nblocks_for(n, kBlock), (unsigned)num_sms * 8), kBlock, 0, ws.st>>>(
      n, x, mm);
  count_launch();
  k_minmax_out<<<1, 1, 0, ws.st>>>(mm, out2);
  return FJ_OK;
}

// ------------------------------------------------------------------ max i64
__global__ void k_max_i64(int64_t n, const int64_t *__restrict__ x, unsigned long long *out) {
  int64_t m = 0;  // inputs are row lengths (≥ 0)
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, x[i]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)m);
}

fj_status max_nonneg_i64(const int64_t *x, int64_t n, int64_t *out, Workspace &ws, int num_sms) {
  FJ_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), ws.st));
  count_launch();
  k_max_i64<<<std::min<unsigned>(nblocks_for(n, kBlock), (unsigned)num_sms * 8), kBlock, 0, ws.st>>>(
      n, x, reinterpret_cast<unsigned long long *>(out));
  return FJ_OK;
}

// ---------------------------------------------------------- exclusive scan
// Three phases: each CTA scans a tile of kTile values (block sums out), the
// block sums are scanned (recursively), and the tile offsets are added.
template <class T>
__device__ __forceinline__ T block_excl_scan(T v, T *warp_sums, T &total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    T s = lane < kBlock / 32 ? warp_sums[lane] : T(0);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, s, off);
      if (lane >= off) s += y;
    }
    if (lane < kBlock / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  const T warp_base = wid > 0 ? warp_sums[wid - 1] : T(0);
  total = warp_sums[kBlock / 32 - 1];
  __syncthreads();
  return warp_base + x - v;
}

// tile scan: thread t holds kTileItems consecutive values
template <class T>
__global__ void k_scan_tiles(int64_t n, const T *__restrict__ in, T *__restrict__ out,
                             T *__restrict__ block_sums) {
  __shared__ T warp_sums[kBlock / 32];
  const int64_t base = blockIdx.x * (int64_t)kTile + (int64_t)threadIdx.x * kTileItems;
  T v[kTileItems];
  T sum = 0;
#pragma unroll
  for (int i = 0; i < kTileItems; i++) {
    v[i] = base + i < n ? in[base + i] : T(0);
    sum += v[i];
  }
  T total;
  T run = block_excl_scan<T>(sum, warp_sums, total);
#pragma unroll
  for (int i = 0; i < kTileItems; i++) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 0 && block_sums) block_sums[blockIdx.x] = total;
}
template <class T>
__global__ void k_scan_add(int64_t n, T *__restrict__ out, const T *__restrict__ offs) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] += offs[i / kTile];
}

template <class T>
static fj_status exclusive_scan_t(const T *in, T *out, int64_t n, Workspace &ws) {
  if (n <= 0) return FJ_OK;
  const int64_t nt = (n + kTile - 1) / kTile;
  T *sums = nullptr;
  if (nt > 1) FJ_CUDA(ws.alloc(&sums, (size_t)nt));
  count_launch();
  k_scan_tiles<T><<<(unsigned)nt, kBlock, 0, ws.st>>>(n, in, out, sums);
  if (nt > 1) {
    T *offs = nullptr;
    FJ_CUDA(ws.alloc(&offs, (size_t)nt));
    FJ_TRY(exclusive_scan_t<T>(sums, offs, nt, ws));
    count_launch();
    k_scan_add<T><<<nblocks_for(n, kBlock), kBlock, 0, ws.st>>>(n, out, offs);
  }
  return FJ_OK;
}

fj_status exclusive_scan_i64(const int64_t *in, int64_t *out, int64_t n, Workspace &ws) {
  return exclusive_scan_t<int64_t>(in, out, n, ws);
}

// --------------------------------------------------------------- radix sort
// (1) digit counts of every tile, digit-major: counts[d · ntiles + tile]
template <class K>
__global__ void k_radix_count(int64_t m, const K *__restrict__ keys, int shift,
                              unsigned *__restrict__ counts, int64_t ntiles) {
  __shared__ unsigned h[kRadix];
  h[threadIdx.x] = 0;  // kBlock == kRadix
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)kTile;
#pragma unroll 4
  for (int i = 0; i < kTileItems; i++) {
    const int64_t k = base + (int64_t)i * kBlock + threadIdx.x;
    if (k < m) atomicAdd(&h[(keys[k] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  counts[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// (3) stable scatter through shared memory: the tile's keys are first ranked
// and placed in tile-local digit order in shared memory (rounds of kBlock keys
// in input order; a key's local slot = its digit's start in the tile + keys of
// that digit in earlier rounds (run) + in earlier warps of the round (wcnt) +
// in earlier lanes of its warp (match)), then written out in that order, so
// every digit's run of the tile lands contiguously (coalesced) at its offset
template <class K, class V>
__global__ void __launch_bounds__(kBlock) k_radix_scatter(int64_t m, const K *__restrict__ keys,
                                                          const V *__restrict__ vals, int shift,
                                                          const unsigned *__restrict__ counts,
                                                          const unsigned *__restrict__ offs,
                                                          int64_t ntiles, K *__restrict__ keys_out,
                                                          V *__restrict__ vals_out) {
  constexpr int NW = kBlock / 32;
  extern __shared__ unsigned char smem_raw[];
  K *skey = reinterpret_cast<K *>(smem_raw);
  V *sval = reinterpret_cast<V *>(smem_raw + sizeof(K) * kTile);
  __shared__ unsigned lstart[kRadix], run[kRadix], gbase[kRadix], warp_tot[NW];
  __shared__ unsigned wcnt[NW][kRadix];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int dd = threadIdx.x;  // kBlock == kRadix: one thread per digit
  // tile-local digit starts: exclusive scan of this tile's digit counts
  {
    const unsigned c = counts[(int64_t)dd * ntiles + blockIdx.x];
    unsigned x = c;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, x, off);
      if (lane >= off) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    unsigned wb = 0;
    for (int w = 0; w < wid; w++) wb += warp_tot[w];
    lstart[dd] = wb + x - c;
    run[dd] = wb + x - c;
    gbase[dd] = offs[(int64_t)dd * ntiles + blockIdx.x];
  }
#pragma unroll
  for (int w = 0; w < NW; w++) wcnt[w][dd] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)kTile;
  const int nt = (int)min((int64_t)kTile, m - base);
  for (int i = 0; i < kTileItems; i++) {
    const int64_t k = base + (int64_t)i * kBlock + threadIdx.x;
    const bool ok = k < m;
    K key = 0;
    V val{};
    if (ok) {
      key = keys[k];
      val = vals[k];
    }
    const unsigned d = ok ? (unsigned)((key >> shift) & (kRadix - 1)) : (unsigned)kRadix;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned rank = __popc(peers & ((1u << lane) - 1u));
    if (ok && rank == 0) wcnt[wid][d] = __popc(peers);
    __syncthreads();
    {  // per digit: exclusive prefix over the warps, then advance the run
      unsigned s = run[dd];
#pragma unroll
      for (int w = 0; w < NW; w++) {
        const unsigned c = wcnt[w][dd];
        wcnt[w][dd] = s;
        s += c;
      }
      run[dd] = s;
    }
    __syncthreads();
    if (ok) {
      const unsigned lp = wcnt[wid][d] + rank;
      skey[lp] = key;
      sval[lp] = val;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NW; w++) wcnt[w][dd] = 0;
    __syncthreads();  // zeroed before the next round's warp counts land
  }
  // write out in tile-local digit order: runs of one digit are contiguous
  for (int i = threadIdx.x; i < nt; i += kBlock) {
    const K key = skey[i];
    const unsigned d = (unsigned)((key >> shift) & (kRadix - 1));
    const unsigned dst = gbase[d] + (unsigned)i - lstart[d];
    keys_out[dst] = key;
    vals_out[dst] = sval[i];
  }
}

template <class K, class V>
fj_status radix_sort_pairs(K *&keys, K *&keys_alt, V *&vals, V *&vals_alt, int64_t m, int nbits,
                           Workspace &ws) {
  static_assert(kBlock == kRadix, "one thread per digit");
  if (m <= 0) return FJ_OK;
  if (m > (int64_t)0xffffffffLL) {
    set_error("radix sort: more than 2^32 items");
    return FJ_ERR_INVALID;
  }
  const int64_t nt = (m + kTile - 1) / kTile;
  unsigned *counts = nullptr, *offs = nullptr;
  FJ_CUDA(ws.alloc(&counts, (size_t)(kRadix * nt)));
  FJ_CUDA(ws.alloc(&offs, (size_t)(kRadix * nt)));
  const size_t smem = (sizeof(K) + sizeof(V)) * kTile;  // the tile in local digit order
  FJ_CUDA(cudaFuncSetAttribute(k_radix_scatter<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  for (int shift = 0; shift < nbits; shift += 8) {
    count_launch();
    k_radix_count<K><<<(unsigned)nt, kBlock, 0, ws.st>>>(m, keys, shift, counts, nt);
    FJ_TRY(exclusive_scan_t<unsigned>(counts, offs, kRadix * nt, ws));
    count_launch();
    k_radix_scatter<K, V><<<(unsigned)nt, kBlock, smem, ws.st>>>(m, keys, vals, shift, counts, offs,
                                                                 nt, keys_alt, vals_alt);
    std::swap(keys, keys_alt);
    std::swap(vals, vals_alt);
  }
  return FJ_OK;
}

template fj_status radix_sort_pairs<uint32_t, uint32_t>(uint32_t *&, uint32_t *&, uint32_t *&,
                                                        uint32_t *&, int64_t, int, Workspace &);
template fj_status radix_sort_pairs<uint32_t, uint64_t>(uint32_t *&, uint32_t *&, uint64_t *&,
                                                        uint64_t *&, int64_t, int, Workspace &);
template fj_status radix_sort_pairs<uint32_t, int32_t>(uint32_t *&, uint32_t *&, int32_t *&,
                                                       int32_t *&, int64_t, int, Workspace &);
template fj_status radix_sort_pairs<uint64_t, uint32_t>(uint64_t *&, uint64_t *&, uint32_t *&,
                                                        uint32_t *&, int64_t, int, Workspace &);

}  // namespace fj
