// Cycle cost of score_block (mma_common.cuh) on smem-resident data, 8 warps/SM:
// isolates the DMMA + epilogue compute from TMA / global traffic.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1606_08905_b200/csrc/mma_common.cuh"
using namespace knb;

template <int DP>
__global__ void __launch_bounds__(256, 1) kern(const double* means, int k, int d, int reps, long long* cyc, int* sink) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int KS = DP / 4;
  const int kp = (k + 7) & ~7, ntile8 = kp >> 3;
  double* bf = reinterpret_cast<double*>(smem);
  double* chn = bf + kp * DP;
  unsigned char* tiles = smem + ((kp * DP + kp) * 8 + 1023) / 1024 * 1024;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kp * DP; i += blockDim.x) {
    const int l = i & 31, qs = i >> 5, q = qs / KS, s = qs - q * KS;
    const int jb = q * 8 + (l >> 2), eb = s * 4 + (l & 3);
    bf[i] = (jb < k && eb < d) ? means[jb * d + eb] : 0.0;
  }
  for (int j = threadIdx.x; j < kp; j += blockDim.x) {
    double s = 0; for (int e = 0; e < d; ++e) s += means[j * d + e] * means[j * d + e];
    chn[j] = j < k ? -0.5 * s : -1.0 / 0.0;
  }
  unsigned char* tb = tiles + warp * 32 * DP * 8;
  for (int i = lane; i < 32 * DP; i += 32) reinterpret_cast<double*>(tb)[i] = ((i * 7919) % 1000) * 1e-3;
  __syncthreads();
  int acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    Scored s = score_block<DP>(tb, bf, chn, ntile8, 1e-13, 100.0, lane);
    acc += s.id + (s.flag ? 1 : 0);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 8 + warp] = t1 - t0;
  if (acc == 123456789) sink[0] = acc;
}

int main() {
  const int k = 32, d = 32, reps = 200;
  double* means; long long* cyc; int* sink;
  cudaMalloc(&means, k * d * 8); cudaMalloc(&cyc, 148 * 8 * 8); cudaMalloc(&sink, 4);
  double h[k * d]; for (int i = 0; i < k * d; ++i) h[i] = ((i * 104729) % 997) * 1e-3;
  cudaMemcpy(means, h, sizeof(h), cudaMemcpyHostToDevice);
  size_t sm = ((k * d + k) * 8 + 1023) / 1024 * 1024 + 8 * 32 * d * 8;
  cudaFuncSetAttribute(kern<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int warps : {8, 4, 16}) {
    kern<32><<<148, warps * 32, sm>>>(means, k, d, reps, cyc, sink);
    cudaDeviceSynchronize();
    long long hc[148 * 8]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    double avg = 0; int nw = warps > 8 ? 8 : warps; for (int i = 0; i < nw; ++i) avg += hc[i]; avg /= nw;
    printf("warps/SM=%d: %.0f cycles per 32-row block per warp (%.0f per SMSP-block), DMMA-bound ideal %d\n",
           warps, avg / reps, avg / reps / (warps / 4.0), 128 * 16 / 1);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
