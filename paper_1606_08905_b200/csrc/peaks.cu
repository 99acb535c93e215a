// Roofline denominators that MEASURED_PEAKS.json does not carry: the FP64 FMA
// rate (the bound of the f64 configs 2 and 4) -- measured on the box by the
// benchmark itself rather than assumed from a datasheet, as the faster of the
// vector DFMA pipe and the FP64 tensor path (DMMA), in FMA/s.
#include <cuda_runtime.h>

#include "../../include/knor_b200.h"
#include "kernels.h"

namespace {

// 8 independent DFMA chains per thread; the chains never converge, so ptxas
// cannot fold them.  Each loop trip issues 8 DFMA per thread.
__global__ void __launch_bounds__(256) dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b);
    x1 = fma(x1, a, b);
    x2 = fma(x2, a, b);
    x3 = fma(x3, a, b);
    x4 = fma(x4, a, b);
    x5 = fma(x5, a, b);
    x6 = fma(x6, a, b);
    x7 = fma(x7, a, b);
  }
  const double s = ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7));
  if (s == 1234.5678) out[threadIdx.x] = s;  // never true; keeps the chains live
}

// FP64 tensor path: 8 independent m8n8k4 accumulators per warp (256 FMA per mma)
__global__ void __launch_bounds__(256) dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
}

__global__ void copy_kernel(const double4* __restrict__ src, double4* __restrict__ dst, long long n4) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace

extern "C" int knb_measure_peaks(int device, double* dfma_per_s, double* copy_bytes_per_s) {
  if (cudaSetDevice(device) != cudaSuccess) return KNB_E_CUDA;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return KNB_E_CUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* out = nullptr;
  if (cudaMalloc(&out, 4096) != cudaSuccess) return KNB_E_NOMEM;
  const int blocks = p.multiProcessorCount * 8, iters = 1 << 14;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;  // first launch is warm-up
  }
  double fma_rate = (double)blocks * 256.0 * 8.0 * iters / (best * 1e-3);
  best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dmma_kernel<<<p.multiProcessorCount * 4, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double mma_rate = (double)p.multiProcessorCount * 4 * 8 * 256.0 * 8 * iters / (best * 1e-3);
  // the FP64 roofline is the faster of the two FP64 pipes (vector FMA, DMMA tensor)
  if (dfma_per_s) *dfma_per_s = fma_rate > mma_rate ? fma_rate : mma_rate;
  const long long bytes = 1LL << 30;
  double *a = nullptr, *b = nullptr;
  int rc = KNB_OK;
  if (cudaMalloc(&a, bytes) == cudaSuccess && cudaMalloc(&b, bytes) == cudaSuccess) {
    cudaMemset(a, 0, bytes);
    best = 1e30f;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      copy_kernel<<<p.multiProcessorCount * 16, 256>>>((const double4*)a, (double4*)b, bytes / 32);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep && ms < best) best = ms;
    }
    if (copy_bytes_per_s) *copy_bytes_per_s = 2.0 * bytes / (best * 1e-3);
  } else {
    rc = KNB_E_NOMEM;
  }
  if (a) cudaFree(a);
  if (b) cudaFree(b);
  cudaFree(out);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (cudaGetLastError() != cudaSuccess) return KNB_E_CUDA;
  return rc;
}
