// Microbenchmarks that decide the f64 distance-kernel design (run on the B200):
//   dfma   : 8 independent DFMA chains per thread (vector FP64 pipe)
//   dmma   : mma.sync.m8n8k4.f64 with 4/8 independent accumulators per warp (FP64 tensor path)
//   ldsb   : warp-uniform (broadcast) LDS.128 / LDS.64 issue cost
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_k(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

template <int NACC>
__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5 + threadIdx.x * 1e-4;
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void ldsb_k(double* out, int iters, int stride) {
  __shared__ double2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_double2(i, -i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 16; ++j) {
      double2 v = sm[(idx + j * 16 + (stride ? (threadIdx.x & 31) : 0)) & 1023];
      acc.x += v.x; acc.y += v.y;
    }
    idx += 17;
  }
  if (acc.x == 1234.5) out[0] = acc.x + acc.y;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  auto timeit = [&](auto launch) { float best = 1e30f; for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms; } return best; };
  int it = 1 << 14;
  for (int bpsm : {4, 8}) {
    float ms = timeit([&] { dfma_k<<<sms * bpsm, 256>>>(out, it); });
    double fmas = (double)sms * bpsm * 256 * 8 * it;
    printf("dfma  blocks/SM=%d: %.2f T FMA/s (%.1f TFLOP/s)\n", bpsm, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  for (int bpsm : {1}) {
    for (int thr : {128, 256}) {
      float ms = timeit([&] { dmma_k<8><<<sms * bpsm, thr>>>(out, it); });
      double fmas = (double)sms * bpsm * (thr / 32) * 256 * 8 * it;
      printf("dmma8 1 block/SM of %d threads (%d warps/SM): %.2f T FMA/s\n", thr, thr / 32, fmas / ms / 1e9);
      ms = timeit([&] { dmma_k<16><<<sms * bpsm, thr>>>(out, it); });
      fmas = (double)sms * bpsm * (thr / 32) * 256 * 16 * it;
      printf("dmma16 1 block/SM of %d threads (%d warps/SM): %.2f T FMA/s\n", thr, thr / 32, fmas / ms / 1e9);
    }
  }
  for (int bpsm : {2, 4, 8}) {
    float ms = timeit([&] { dmma_k<4><<<sms * bpsm, 256>>>(out, it); });
    double fmas = (double)sms * bpsm * 8 * 256 * 4 * it;
    printf("dmma4 blocks/SM=%d: %.2f T FMA/s (%.1f TFLOP/s)\n", bpsm, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
    ms = timeit([&] { dmma_k<8><<<sms * bpsm, 256>>>(out, it); });
    fmas = (double)sms * bpsm * 8 * 256 * 8 * it;
    printf("dmma8 blocks/SM=%d: %.2f T FMA/s (%.1f TFLOP/s)\n", bpsm, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  for (int stride : {0, 1}) {
    float ms = timeit([&] { ldsb_k<<<sms * 4, 256>>>(out, 1 << 12, stride); });
    double n = (double)sms * 4 * 8 * 16 * (1 << 12);  // warp-level LDS.128
    printf("lds128 %s: %.3f warp-LDS per clk per SM (at %d MHz)\n", stride ? "lane-distinct" : "broadcast",
           n / (ms * 1e-3) / sms / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
