// score_block variants on smem-resident data (k = 32, d = 32), cycles per 32-row block.
// Build twice: -DKNB_EXPERIMENT=0 (full) and =1 (epilogue replaced by a max).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1606_08905_b200/csrc/mma_common.cuh"
using namespace knb;

template <int DP, bool LEAN, int NW>
__global__ void __launch_bounds__(NW * 32, 1) kern(const double* means, int k, int d, int reps, long long* cyc, int* sink) {
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
    Scored s = score_block<DP, false, LEAN>(tb, bf, chn, ntile8, 1e-13, 100.0, lane);
    acc += s.id + (s.flag ? 1 : 0);
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  if (acc == 123456789) sink[0] = acc;
}

template <bool LEAN, int NW>
void run(const double* means, long long* cyc, int* sink) {
  const int k = 32, d = 32, reps = 200;
  size_t sm = ((k * d + k) * 8 + 1023) / 1024 * 1024 + NW * 32 * d * 8;
  cudaFuncSetAttribute(kern<32, LEAN, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  kern<32, LEAN, NW><<<148, NW * 32, sm>>>(means, k, d, reps, cyc, sink);
  cudaDeviceSynchronize();
  long long hc[16]; cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < NW; ++i) avg += hc[i]; avg /= NW;
  printf("EXP=%d LEAN=%d warps/SM=%2d: %6.0f cyc/block/warp, %6.0f per SMSP-block: %.0f%% of DMMA peak\n",
         KNB_EXPERIMENT, (int)LEAN, NW, avg / reps, avg / reps / (NW / 4.0), 2048.0 / (avg / reps / (NW / 4.0)) * 100);
}

int main() {
  const int k = 32, d = 32;
  double* means; long long* cyc; int* sink;
  cudaMalloc(&means, k * d * 8); cudaMalloc(&cyc, 148 * 16 * 8); cudaMalloc(&sink, 4);
  double h[k * d]; for (int i = 0; i < k * d; ++i) h[i] = ((i * 104729) % 997) * 1e-3;
  cudaMemcpy(means, h, sizeof(h), cudaMemcpyHostToDevice);
  run<false, 4>(means, cyc, sink); run<false, 8>(means, cyc, sink); run<false, 12>(means, cyc, sink); run<false, 16>(means, cyc, sink);
  run<true, 4>(means, cyc, sink); run<true, 8>(means, cyc, sink); run<true, 12>(means, cyc, sink); run<true, 16>(means, cyc, sink);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
