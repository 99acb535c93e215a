// TMEM read (tcgen05.ld) throughput on one SM: W warps each read 7 x 16 columns of their
// lane quarter per round (the c4 epilogue's pattern), reduce them with a cheap op, repeat.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_tmem tools/mb_tmem.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int OPS>
__global__ void k_tmem(int rounds, unsigned* out, long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 128);
  unsigned acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
#pragma unroll
    for (int g = 0; g < 7; ++g) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(base + 16 * g)
          : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (OPS) {
#pragma unroll
        for (int e = 0; e < 16; ++e) acc = min(acc + r[e], acc ^ r[e]);
      } else {
        acc ^= r[0] ^ r[15];
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(512));
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int rounds = 4096;
  for (int ops = 0; ops < 2; ++ops)
    for (int w : {4, 8, 12, 16}) {
      for (int rep = 0; rep < 2; ++rep) {
        if (ops) k_tmem<1><<<148, 32 * w>>>(rounds, out, cyc);
        else k_tmem<0><<<148, 32 * w>>>(rounds, out, cyc);
      }
      cudaError_t e = cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)rounds * 7 * 16 * 32 * 4 * w;
      printf("ops=%d warps=%2d: %lld cycles, %.1f B/clk/SM, %.1f cycles per (128 rows x 112 cols) tile  %s\n", ops, w,
             c, bytes / c, (double)c / (rounds * w / 4.0), cudaGetErrorString(e));
    }
  return 0;
}
