// microbench.cu — bandwidth probes for the pull-sweep access pattern on the
// real layout CSR (diagnostics only, not part of libfj).
//   mode 0: stream col (+w) only              (DRAM roofline of the arc stream)
//   mode 1: gather z[col[k]] (fp64), sum      (stream + random gathers)
//   mode 2: sum w[k] * z[col[k]] (fp64)       (SpMV-like, no row structure)
//   mode 3: like 2 with fp32 z                (gather bytes halved)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
#include <cuda_runtime.h>
#include <stdint.h>

template <int MODE>
__global__ void __launch_bounds__(256) k_probe(int64_t m, const int *__restrict__ col,
                                                const float *__restrict__ w,
                                                const double *__restrict__ z,
                                                const float *__restrict__ zf, double *out) {
  constexpr int U = 8;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < m; k0 += stride * U) {
    int j[U];
    float wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t k = k0 + u * stride;
      bool ok = k < m;
      j[u] = ok ? __ldg(col + k) : 0;
      wv[u] = (ok && w) ? __ldg(w + k) : (ok ? 1.f : 0.f);
    }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < U; u++) acc += (double)j[u] + wv[u];
    } else if (MODE == 3) {
      float zz[U];
#pragma unroll
      for (int u = 0; u < U; u++) zz[u] = zf[j[u]];
#pragma unroll
      for (int u = 0; u < U; u++) acc += (double)(wv[u] * zz[u]);
    } else {
      double zz[U];
#pragma unroll
      for (int u = 0; u < U; u++) zz[u] = z[j[u]];
#pragma unroll
      for (int u = 0; u < U; u++) acc += (MODE == 1 ? zz[u] : (double)wv[u] * zz[u]);
    }
  }
  if (acc == 12345.678) *out = acc;  // keep the work alive
}

// K-wide gathers: z2 is double2[n * K/2] node-major
template <int K>
__global__ void __launch_bounds__(256) k_probe_k(int64_t m, const int *__restrict__ col,
                                                  const float *__restrict__ w,
                                                  const double2 *__restrict__ z2, double *out) {
  constexpr int U = 8;
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k0 < m; k0 += stride * U) {
    int j[U];
    float wv[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int64_t k = k0 + u * stride;
      bool ok = k < m;
      j[u] = ok ? __ldg(col + k) : 0;
      wv[u] = (ok && w) ? __ldg(w + k) : (ok ? 1.f : 0.f);
    }
    double2 zz[U][K / 2];
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int q = 0; q < K / 2; q++) zz[u][q] = z2[(int64_t)j[u] * (K / 2) + q];
#pragma unroll
    for (int u = 0; u < U; u++)
#pragma unroll
      for (int q = 0; q < K / 2; q++) acc += (double)wv[u] * (zz[u][q].x + zz[u][q].y);
  }
  if (acc == 12345.678) *out = acc;
}

extern "C" float fj_probe_k(int K, int64_t m, const int *col, const float *w, const double *z2,
                            int reps) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dim3 grid(sms * 4);
  auto launch = [&]() {
    if (K == 2) k_probe_k<2><<<grid, 256>>>(m, col, w, (const double2 *)z2, out);
    else if (K == 4) k_probe_k<4><<<grid, 256>>>(m, col, w, (const double2 *)z2, out);
    else k_probe_k<8><<<grid, 256>>>(m, col, w, (const double2 *)z2, out);
  };
  launch();
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms / reps;
}

extern "C" float fj_probe(int mode, int64_t m, const int *col, const float *w, const double *z,
                          const float *zf, int reps, int blocks_per_sm) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  dim3 grid(sms * blocks_per_sm);
  auto launch = [&]() {
    switch (mode) {
      case 0: k_probe<0><<<grid, 256>>>(m, col, w, z, zf, out); break;
      case 1: k_probe<1><<<grid, 256>>>(m, col, w, z, zf, out); break;
      case 2: k_probe<2><<<grid, 256>>>(m, col, w, z, zf, out); break;
      default: k_probe<3><<<grid, 256>>>(m, col, w, z, zf, out); break;
    }
  };
  launch();
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(out);
  return ms / reps;
}
