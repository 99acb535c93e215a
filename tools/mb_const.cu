// Microbenchmark: row-per-thread f64 scoring with centroids as uniform constant-bank
// operands (DFMA R, R, UR, R after LDCU), R rows per thread.  Reports FMA/s.
//
// Round-1 finding (B200): R = 2, d = 16, k = 100 reaches 14 T FMA/s (77% of the DFMA
// peak) here, but only while ptxas keeps the centroid walk on the uniform datapath
// (LDCU).  Inside the real K1 loop -- any other loop in the per-block body (mbarrier
// spin, row-ordered accumulation, exact rerank) -- ptxas falls back to per-thread
// LDC and the scorer ran 2x slower than the DMMA one, so K1 stays on DMMA.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ double c_cent[4096];
template <int DP, int R>
__global__ void __launch_bounds__(256) kern(const double* __restrict__ X, long long n, int kp, double* out) {
  const long long r0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * R;
  double x[R][DP];
#pragma unroll
  for (int q = 0; q < R; ++q)
#pragma unroll
    for (int e = 0; e < DP; ++e) x[q][e] = r0 + q < n ? X[(r0 + q) * DP + e] : 0.0;
  double best[R];
  int bi[R];
#pragma unroll
  for (int q = 0; q < R; ++q) { best[q] = -1e300; bi[q] = 0; }
  for (int jc = 0; jc < kp; jc += 4) {
#pragma unroll
    for (int jj = 0; jj < 4; ++jj) {
      double s[R];
#pragma unroll
      for (int q = 0; q < R; ++q) s[q] = c_cent[3000 + jc + jj];
#pragma unroll
      for (int e = 0; e < DP; ++e) {
        const double c = c_cent[(jc + jj) * DP + e];
#pragma unroll
        for (int q = 0; q < R; ++q) s[q] = fma(x[q][e], c, s[q]);
      }
#pragma unroll
      for (int q = 0; q < R; ++q) if (s[q] > best[q]) { best[q] = s[q]; bi[q] = jc + jj; }
    }
  }
#pragma unroll
  for (int q = 0; q < R; ++q) if (r0 + q < n) out[r0 + q] = best[q] + bi[q];
}
template <int DP, int R>
void run(const double* X, long long n, int kp, double* out) {
  const long long thr = (n + R - 1) / R;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  kern<DP, R><<<(thr + 255) / 256, 256>>>(X, n, kp, out);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) kern<DP, R><<<(thr + 255) / 256, 256>>>(X, n, kp, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("DP=%d R=%d kp=%d: %.3f ms  %.2f T FMA/s  %.1f GB/s\n", DP, R, kp, ms, (double)n * kp * DP / ms / 1e9,
         (double)n * DP * 8 / ms / 1e6);
}
int main() {
  const long long n = 1 << 24;
  double *X, *out;
  cudaMalloc(&X, n * 32 * 8); cudaMalloc(&out, n * 8);
  cudaMemset(X, 0, n * 32 * 8);
  static double h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = 0.001 * (i % 97);
  cudaMemcpyToSymbol(c_cent, h, sizeof(h));
  run<8, 1>(X, n, 12, out); run<8, 2>(X, n, 12, out);
  run<16, 1>(X, n, 100, out); run<16, 2>(X, n, 100, out); run<16, 4>(X, n, 100, out);
  run<32, 1>(X, n / 4, 32, out); run<32, 2>(X, n / 4, 32, out);
  run<16, 1>(X, n, 8, out); run<16, 2>(X, n, 8, out);
  return 0;
}
