// Device generation of numpy's `default_rng(seed).random(shape)` (PCG64 +
// XSL-RR output, random() = (next_uint64 >> 11) * 2^-53), bit-identical to the
// host stream from any starting draw -- config 4's 110 GB input (U[0,1)^16) is
// produced shard by shard in HBM instead of being generated and copied from the
// host.
//
// numpy PCG64: s <- s * M + inc (mod 2^128), then out = rotr64(hi(s) ^ lo(s), s >> 122).
// Jump-ahead by j: s_j = A_j s_0 + C_j with (A, C) composed from the table of
// (M^(2^i), c_i) for the bits of j.  Lane l of a warp starts at draw (chunk + l) and
// then steps 32 draws at a time with (A_32, C_32), so consecutive lanes write
// consecutive doubles.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "../../include/knor_b200.h"

namespace {

struct U128 {
  uint64_t lo, hi;
};

__host__ __device__ inline U128 mul128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo * b.lo;
#ifdef __CUDA_ARCH__
  r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
#else
  r.hi = (uint64_t)(((unsigned __int128)a.lo * b.lo) >> 64) + a.hi * b.lo + a.lo * b.hi;
#endif
  return r;
}

__host__ __device__ inline U128 add128(U128 a, U128 b) {
  U128 r;
  r.lo = a.lo + b.lo;
  r.hi = a.hi + b.hi + (r.lo < a.lo ? 1 : 0);
  return r;
}

struct Jump {
  U128 a, c;  // s -> a * s + c
};

__constant__ Jump c_pow2[64];  // jump by 2^i draws

__device__ inline U128 jump_from(U128 s, unsigned long long j) {
  U128 A{1, 0}, C{0, 0};
  for (int i = 0; j; ++i, j >>= 1) {
    if (j & 1) {
      A = mul128(A, c_pow2[i].a);
      C = add128(mul128(C, c_pow2[i].a), c_pow2[i].c);
    }
  }
  return add128(mul128(A, s), C);
}

__device__ inline double output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  const uint64_t o = (x >> rot) | (x << ((64 - rot) & 63));
  return (double)(o >> 11) * 1.1102230246251565e-16;  // * 2^-53 (exact)
}

// out[i] = draw (first + i), i < count.  Each warp fills chunks of 32 * R draws.
__global__ void __launch_bounds__(256) pcg64_fill_kernel(double* __restrict__ out, long long count,
                                                         unsigned long long first, U128 s0, Jump step1,
                                                         Jump step32) {
  constexpr int R = 64;
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const long long chunk = 32LL * R;
  for (long long base = warp * chunk; base < count; base += nwarps * chunk) {
    // state *before* draw (first + base + lane): the draw itself steps once more
    U128 s = jump_from(s0, first + base + lane);
#pragma unroll 4
    for (int r = 0; r < R; ++r) {
      const long long i = base + lane + 32LL * r;
      const U128 t = add128(mul128(step1.a, s), step1.c);  // the step that produces this draw
      if (i < count) out[i] = output(t);
      s = add128(mul128(step32.a, s), step32.c);
    }
  }
}

}  // namespace

extern "C" int knb_fill_uniform_pcg64(double* dev_out, int64_t count, int64_t first_draw, uint64_t state_hi,
                                      uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, void* stream) {
  if (!dev_out || count < 0 || first_draw < 0) return KNB_E_ARG;
  const U128 M{0x4385DF649FCCF645ULL, 0x2360ED051FC65DA4ULL};
  const U128 inc{inc_lo, inc_hi};
  Jump tab[64];
  U128 a = M, c = inc;
  for (int i = 0; i < 64; ++i) {
    tab[i].a = a;
    tab[i].c = c;
    c = mul128(c, add128(a, U128{1, 0}));  // c_{2j} = c_j (a_j + 1)
    a = mul128(a, a);
  }
  if (cudaMemcpyToSymbolAsync(c_pow2, tab, sizeof(tab), 0, cudaMemcpyHostToDevice,
                              static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return KNB_E_CUDA;
  Jump step1{M, inc}, step32 = tab[5];
  const U128 s0{state_lo, state_hi};
  const long long warps_needed = (count + 32LL * 64 - 1) / (32LL * 64);
  long long blocks = (warps_needed + 7) / 8;
  if (blocks > 148LL * 16) blocks = 148LL * 16;
  if (blocks < 1) blocks = 1;
  if (count) pcg64_fill_kernel<<<(int)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dev_out, count, (unsigned long long)first_draw, s0, step1, step32);
  return cudaGetLastError() == cudaSuccess ? KNB_OK : KNB_E_CUDA;
}
