// gather_bench.cu — ceilings of the pull sweep's gather pattern (diagnostics,
// not part of libfj): stream col (+w) and gather one fp64 x[col] per arc,
// with the H most popular columns (ids < H after relabelling) optionally
// served from a per-CTA shared-memory copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <stdint.h>

// VEC: 1 = scalar 4-byte stream loads, 4 = int4/float4 (4 consecutive arcs per lane)
template <int VEC, bool HOT>
__global__ void k_gb(int64_t m, const int *__restrict__ col, const float *__restrict__ w,
                     const double *__restrict__ x, int H, double *out) {
  extern __shared__ double hot[];
  if (HOT) {
    for (int i = threadIdx.x; i < H; i += blockDim.x) hot[i] = x[i];
    __syncthreads();
  }
  constexpr int U = 8 / VEC;  // loads in flight per lane: 8 arcs either way
  double acc = 0.0;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t mv = m / VEC;
  for (int64_t k0 = tid; k0 < mv; k0 += nthr * U) {
    int j[8];
    float wv[8];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t k = k0 + u * nthr;
      const bool ok = k < mv;
      const int64_t kk = ok ? k : 0;
      if (VEC == 4) {
        int4 c = __ldg(reinterpret_cast<const int4 *>(col) + kk);
        float4 ww = w ? __ldg(reinterpret_cast<const float4 *>(w) + kk) : make_float4(1, 1, 1, 1);
        j[4 * u] = c.x; j[4 * u + 1] = c.y; j[4 * u + 2] = c.z; j[4 * u + 3] = c.w;
        wv[4 * u] = ok ? ww.x : 0; wv[4 * u + 1] = ok ? ww.y : 0;
        wv[4 * u + 2] = ok ? ww.z : 0; wv[4 * u + 3] = ok ? ww.w : 0;
      } else {
        j[u] = __ldg(col + kk);
        wv[u] = ok ? (w ? __ldg(w + kk) : 1.f) : 0.f;
      }
    }
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (HOT && j[u] < H) v[u] = hot[j[u]];
      else v[u] = x[j[u]];
    }
#pragma unroll
    for (int u = 0; u < 8; u++) acc = fma((double)wv[u], v[u], acc);
  }
  if (acc == 1.2345e300) *out = acc;
}

extern "C" float gb_run(int vec, int hot, int64_t m, const int *col, const float *w,
                        const double *x, int H, int threads, int carveout, int reps, int extra) {
  const void *fn = vec == 4 ? (hot ? (const void *)k_gb<4, true> : (const void *)k_gb<4, false>)
                            : (hot ? (const void *)k_gb<1, true> : (const void *)k_gb<1, false>);
  const size_t smem = (hot ? (size_t)H * 8 : 0) + (size_t)extra;  // extra: emulated staging smem
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (carveout >= 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  int per_sm = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (per_sm < 1) return -1.f;
  const int grid = per_sm * sms;
  double *out = nullptr;
  cudaMalloc(&out, 8);
  void *args[] = {&m, &col, &w, &x, &H, &out};
  cudaLaunchKernel(fn, grid, threads, args, smem, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) cudaLaunchKernel(fn, grid, threads, args, smem, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return -2.f;
  return ms / reps;
}

extern "C" int gb_occupancy(int vec, int hot, int H, int threads) {
  const void *fn = vec == 4 ? (hot ? (const void *)k_gb<4, true> : (const void *)k_gb<4, false>)
                            : (hot ? (const void *)k_gb<1, true> : (const void *)k_gb<1, false>);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, hot ? (size_t)H * 8 : 0);
  return per_sm;
}
