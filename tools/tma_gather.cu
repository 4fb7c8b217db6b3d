// tma_gather.cu — diagnostics, not part of libfj: can TMA tile::gather4 move
// random fp64 gathers off the L1TEX LSU path?  The pull sweep is bound by L1TEX
// wavefronts (one per 128-byte line a warp-wide gather touches, ≈ 1 per SM
// clock).  A gather4 fetches four 32-byte rows of a 2-D tensor map
// straight from L2 into shared memory (async proxy, no LSU wavefronts, no L1
// line allocated per miss).  This probe streams col and sums x[col] over m arcs
//   mode 0: LDG gathers (the sweep's path), 4 arcs per lane per step, 2 steps in flight
//   mode 1: gather4 into per-warp shared stages (S stages of 128 arcs), mbarrier completion
//   mode 2: both at once: the first `tma_warps` warps of each CTA run mode 1 on
//           the first `tma_frac` of the arcs, the others mode 0 on the rest
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace {

constexpr int kS = 4;       // TMA stages per warp
constexpr int kChunk = 128;  // arcs per warp stage (4 per lane)

__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void g4(void *dst, const CUtensorMap *tm, int4 r, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(tm), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ int4 ld_col4(const int *p) {
  int4 v;
  asm("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}

// LDG path over chunks [c0, c1) of 128 arcs, warp wi of nwarps
__device__ double ldg_part(const int *col, const double *x, int64_t c0, int64_t c1, int64_t wi,
                           int64_t nwarps) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int64_t c = c0 + wi; c < c1; c += 2 * nwarps) {
    const int64_t c2 = c + nwarps < c1 ? c + nwarps : c;
    const int4 a = ld_col4(col + c * kChunk + 4 * lane);
    const int4 b = ld_col4(col + c2 * kChunk + 4 * lane);
    const double v0 = x[a.x], v1 = x[a.y], v2 = x[a.z], v3 = x[a.w];
    const double v4 = x[b.x], v5 = x[b.y], v6 = x[b.z], v7 = x[b.w];
    acc += v0 + v1 + v2 + v3;
    if (c2 != c) acc += v4 + v5 + v6 + v7;
  }
  return acc;
}

// TMA path over chunks [c0, c1), kS chunks in flight per warp
__device__ double tma_part(const int *col, const CUtensorMap *tm, int64_t c0, int64_t c1,
                           int64_t wi, int64_t nwarps, double *buf, uint64_t *bars) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  int4 hold[kS];
  auto issue = [&](int s, int64_t c) {
    const int4 cc = ld_col4(col + c * kChunk + 4 * lane);
    hold[s] = cc;
    if (lane == 0) mbar_expect(bars + s, kChunk * 32);
    __syncwarp();
    // 128-byte aligned destination: four 32-byte rows (one L2 sector each)
    g4(buf + (s * kChunk + 4 * lane) * 4, tm, make_int4(cc.x >> 2, cc.y >> 2, cc.z >> 2, cc.w >> 2),
       bars + s);
  };
  int64_t it = 0;
#pragma unroll
  for (int s = 0; s < kS; s++) {
    const int64_t c = c0 + wi + s * nwarps;
    if (c < c1) issue(s, c);
  }
  for (int64_t cb = c0 + wi; cb < c1; cb += (int64_t)kS * nwarps, it++) {
#pragma unroll
    for (int s = 0; s < kS; s++) {
      const int64_t c = cb + s * nwarps;
      if (c >= c1) break;
      mbar_wait(bars + s, (uint32_t)(it & 1));
      // read back with few bank conflicts: in read step u lane l takes row
      // i = l % 4 of issuer lane 8u + l / 4 (its column offset comes by shuffle)
      const int4 cc = hold[s];
      const double *q = buf + (size_t)s * kChunk * 4;
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int src = 8 * u + (lane >> 2), i = lane & 3;
        const int cx = __shfl_sync(0xffffffffu, cc.x, src), cy = __shfl_sync(0xffffffffu, cc.y, src);
        const int cz = __shfl_sync(0xffffffffu, cc.z, src), cw = __shfl_sync(0xffffffffu, cc.w, src);
        const int cj = i == 0 ? cx : (i == 1 ? cy : (i == 2 ? cz : cw));
        acc += q[src * 16 + i * 4 + (cj & 3)];
      }
      __syncwarp();
      const int64_t cn = c + (int64_t)kS * nwarps;
      if (cn < c1) issue(s, cn);
    }
  }
  return acc;
}

__global__ void __launch_bounds__(256, 4) k_probe(int mode, int64_t nchunks, const int *col,
                                               const double *x,
                                               const __grid_constant__ CUtensorMap tm,
                                               int tma_warps, int64_t tma_chunks, double *sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int nw = blockDim.x >> 5, wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  if (mode == 0) {
    acc = ldg_part(col, x, 0, nchunks, blockIdx.x * (int64_t)nw + wib, (int64_t)gridDim.x * nw);
  } else {
    const int tw = mode == 1 ? nw : tma_warps;
    const int64_t tc = mode == 1 ? nchunks : tma_chunks;
    if (wib < tw) {
      double *buf = reinterpret_cast<double *>(sm) + (size_t)wib * kS * kChunk * 4;
      uint64_t *bars = reinterpret_cast<uint64_t *>(sm + (size_t)tw * kS * kChunk * 32) + wib * kS;
      if (lane == 0)
        for (int s = 0; s < kS; s++) mbar_init(bars + s);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      __syncwarp();
      acc = tma_part(col, &tm, 0, tc, blockIdx.x * (int64_t)tw + wib, (int64_t)gridDim.x * tw, buf,
                     bars);
    } else {
      const int lw = nw - tw;
      acc = ldg_part(col, x, tc, nchunks, blockIdx.x * (int64_t)lw + (wib - tw),
                     (int64_t)gridDim.x * lw);
    }
  }
  if (acc == 1.2345e300) *sink = acc;
}

__global__ void k_fill(int64_t m, int *col, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (uint64_t)(i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    col[i] = (int)(z % (uint64_t)n);
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                             const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                             const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

// fill col with m uniform ids in [0, n)
extern "C" void tg_fill(int64_t m, int *col, int64_t n, uint64_t seed) {
  k_fill<<<148 * 8, 256>>>(m, col, n, seed);
  cudaDeviceSynchronize();
}

// returns ms per pass (median of reps), or a negative error code
extern "C" float tg_run(int mode, int64_t m, const int *col, const double *x, int64_t n,
                        int ctas_per_sm, int threads, int tma_warps, double tma_frac, int l2promo,
                        int reps) {
  static EncodeFn enc = nullptr;
  if (!enc) {
    cudaDriverEntryPointQueryResult q;
    void *fp = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) !=
            cudaSuccess || !fp)
      return -1.f;
    enc = (EncodeFn)fp;
  }
  CUtensorMap tm;
  const cuuint64_t dims[2] = {4, (cuuint64_t)((n + 3) / 4)};
  const cuuint64_t strides[1] = {32};
  const cuuint32_t box[2] = {4, 1};
  const cuuint32_t es[2] = {1, 1};
  const CUtensorMapL2promotion pr =
      l2promo == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                   : (l2promo == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                   : CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)x, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, pr,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2.f - (float)r;
  const int64_t nchunks = m / kChunk;
  const int nw = threads / 32;
  const int tw = mode == 1 ? nw : (mode == 2 ? tma_warps : 0);
  const size_t smem = (size_t)tw * kS * (kChunk * 32 + 8);
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int grid = nsm * ctas_per_sm;
  const int64_t tcs = (int64_t)(tma_frac * (double)nchunks);
  double *sink = nullptr;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best[64];
  int nr = reps < 64 ? reps : 64;
  for (int i = 0; i < nr + 1; i++) {
    cudaEventRecord(a);
    k_probe<<<grid, threads, smem>>>(mode, nchunks, col, x, tm, tw, tcs, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    if (i > 0) best[i - 1] = t;
  }
  cudaError_t e = cudaGetLastError();
  cudaFree(sink);
  if (e != cudaSuccess) {
    fprintf(stderr, "tg_run: %s\n", cudaGetErrorString(e));
    return -100.f;
  }
  for (int i = 1; i < nr; i++)
    for (int j = i; j > 0 && best[j] < best[j - 1]; j--) {
      float t = best[j];
      best[j] = best[j - 1];
      best[j - 1] = t;
    }
  return best[nr / 2];
}
