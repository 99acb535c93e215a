// K8: device-side initialisation helpers, plus the test-mode oracle and the
// finite scan of check_matrix.
//
//   gather      forgy / kmeans++ rows: copy the requested global rows this shard
//               owns into a k x d buffer (rows owned elsewhere stay zero, so an
//               all-reduce(sum) across shards assembles the full set)
//   kpp update  d2 = min(d2, dist(x, c)^2) with the distance computed by the exact
//               recipe, sqrt THEN square as the reference does
//               (centroids.py:179, :187), plus fixed-order block sums
//   kpp search  Generator.choice(n, p=d2/total) draws u = random() and returns
//               searchsorted(cumsum(p) / cdf[-1], u, 'right'); the
//               host supplies the threshold u * cdf[-1] and the device finds the
//               first row whose running sum of d2/total exceeds it
//   validate    engine._validate_prune_state (engine.py:428-445): stored assignment
//               == exhaustive argmin and upper + 1e-9 max(1, d) >= d(v, c_a)
//   finite      matrix.check_matrix's non-finite scan (matrix.py:46-48): index of
//               the first row holding a NaN/inf
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

template <typename T>
__global__ void gather_rows_kernel(const T* __restrict__ X, long long n_local, long long row_lo,
                                   int d, const long long* __restrict__ ids, int count,
                                   double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)count * d;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(i / d), e = (int)(i - (long long)r * d);
    const long long g = ids[r] - row_lo;
    if (g >= 0 && g < n_local) out[i] = (double)X[g * d + e];
  }
}

// d2 update + per-block (KPP_BLOCK rows) sums of d2, fixed order inside a block
template <typename T>
__global__ void kpp_update_kernel(const T* __restrict__ X, long long n, int d,
                                  const double* __restrict__ c, double* __restrict__ d2, int first,
                                  double* __restrict__ block_sums) {
  __shared__ double sh[32];
  const long long b = blockIdx.x;
  const long long lo = b * KPP_BLOCK;
  double s = 0.0;
  // thread-strided rows: one sequential exact tree per row (this order also fixes the
  // block sum the probability walk uses)
  for (int i = threadIdx.x; i < KPP_BLOCK; i += blockDim.x) {
    const long long r = lo + i;
    if (r >= n) break;
    const double dist = sqrt(exact_sq_rt(X + r * d, c, d));
    const double cand = dist * dist;
    double v = first ? cand : fmin(d2[r], cand);
    d2[r] = v;
    s += v;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    block_sums[b] = t;
  }
}

// Same contract and summation order as kpp_update_kernel (thread i of a block handles
// rows lo + i, lo + i + 256, ...) for f64 rows with d <= DP, at memory speed: 256-row
// slabs stream into shared memory with coalesced 16-byte cp.async copies (consecutive
// threads, consecutive bytes; the next slab in flight while this one is scored), and
// every thread reads its row from there (row stride DP + 2 doubles: conflict-free
// 16-byte reads).
constexpr int KPP_SLAB = 256;
template <int DP>
__host__ __device__ constexpr size_t kpp_tile_bytes() { return 2ull * KPP_SLAB * (DP + 2) * 8; }

template <int DP>
__global__ void __launch_bounds__(KPP_SLAB) kpp_update_reg_kernel(const double* __restrict__ X, long long n, int d,
                                                                 const double* __restrict__ c,
                                                                 double* __restrict__ d2, int first,
                                                                 double* __restrict__ block_sums) {
  constexpr int RS = DP + 2;
  __shared__ double sh[32];
  __shared__ double cs[DP];
  extern __shared__ __align__(16) double tiles[];  // two slabs
  const int tid = threadIdx.x;
  for (int e = tid; e < DP; e += blockDim.x) cs[e] = e < d ? c[e] : 0.0;
  const long long lo = (long long)blockIdx.x * KPP_BLOCK;
  const int hd = d >> 1;
  const int nslab = (int)((n - lo < KPP_BLOCK ? n - lo : KPP_BLOCK) + KPP_SLAB - 1) / KPP_SLAB;
  const uint32_t t0 = smem_u32(tiles);
  auto issue = [&](int j) {
    const long long r0 = lo + (long long)j * KPP_SLAB;
    const int rows = n - r0 < KPP_SLAB ? (int)(n - r0) : KPP_SLAB;
    const double2* src = reinterpret_cast<const double2*>(X + r0 * d);
    const uint32_t dst = t0 + (uint32_t)((j & 1) * KPP_SLAB * RS * 8);
    for (int ch = tid; ch < rows * hd; ch += KPP_SLAB) {
      const int r = ch / hd, q = ch - r * hd;
      cp_async16_s(dst + (uint32_t)((r * RS + 2 * q) * 8), src + ch);
    }
    cp_async_commit();
  };
  double s = 0.0;
  if (nslab > 0) issue(0);
  for (int j = 0; j < nslab; ++j) {
    if (j + 1 < nslab) {
      issue(j + 1);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    const long long r0 = lo + (long long)j * KPP_SLAB;
    const int rows = n - r0 < KPP_SLAB ? (int)(n - r0) : KPP_SLAB;
    if (tid < rows) {
      const double old = first ? 0.0 : d2[r0 + tid];  // issued before the row's arithmetic
      const double* row = tiles + (j & 1) * KPP_SLAB * RS + tid * RS;
      double x[DP];
#pragma unroll
      for (int q = 0; q < DP / 2; ++q) {
        if (2 * q < d) {
          const double2 v = *reinterpret_cast<const double2*>(row + 2 * q);
          x[2 * q] = v.x;
          x[2 * q + 1] = v.y;
        } else {
          x[2 * q] = 0.0;
          x[2 * q + 1] = 0.0;
        }
      }
      const long long r = r0 + tid;
      const double dist = sqrt(exact_sq<DP>(x, cs, d));
      const double cand = dist * dist;
      const double v = first ? cand : fmin(old, cand);
      d2[r] = v;
      s += v;
    }
    __syncthreads();  // slab j's buffer is refilled by issue(j + 2)
  }
  s = warp_sum(s);
  if ((tid & 31) == 0) sh[tid >> 5] = s;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    block_sums[blockIdx.x] = t;
  }
}

template <int DP>
cudaError_t launch_kpp_tile(const double* X, long long n, int d, const double* c, double* d2, int first,
                            double* block_sums, int nblk, cudaStream_t s) {
  const size_t sm = kpp_tile_bytes<DP>();
  cudaError_t e = cudaFuncSetAttribute(kpp_update_reg_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  kpp_update_reg_kernel<DP><<<nblk, KPP_SLAB, sm, s>>>(X, n, d, c, d2, first, block_sums);
  return cudaGetLastError();
}

// block sums of p = d2 / total
__global__ void kpp_psums_kernel(const double* __restrict__ d2, long long n, double total,
                                 double* __restrict__ block_sums) {
  __shared__ double sh[32];
  const long long lo = blockIdx.x * (long long)KPP_BLOCK;
  double s = 0.0;
  for (int i = threadIdx.x; i < KPP_BLOCK; i += blockDim.x) {
    const long long r = lo + i;
    if (r >= n) break;
    s += d2[r] / total;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    block_sums[blockIdx.x] = t;
  }
}

// block sums of p = d2 / total with total read from device memory (device loop)
__global__ void kpp_psums_dev_kernel(const double* __restrict__ d2, long long n, const double* total_p,
                                     double* __restrict__ block_sums) {
  __shared__ double sh[32];
  const double total = *total_p;
  const long long lo = blockIdx.x * (long long)KPP_BLOCK;
  double s = 0.0;
  for (int i = threadIdx.x; i < KPP_BLOCK; i += blockDim.x) {
    const long long r = lo + i;
    if (r >= n) break;
    s += d2[r] / total;
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    block_sums[blockIdx.x] = t;
  }
}

// copy row idx[0] of the shard into dst (device-side index)
template <typename T>
__global__ void gather_row_dev_kernel(const T* __restrict__ X, int d, const long long* idx, double* __restrict__ dst) {
  const long long r = *idx;
  for (int e = threadIdx.x; e < d; e += blockDim.x) dst[e] = (double)X[r * d + e];
}

// one warp: lane l adds blocks l, l + 32, ... in order, then a fixed butterfly
__global__ void sum_blocks_kernel(const double* __restrict__ bs, int nblk, double* out) {
  const int lane = threadIdx.x & 31;
  if (threadIdx.x >= 32) return;
  double t = 0.0;
  for (int i = lane; i < nblk; i += 32) t += bs[i];
  t = warp_sum(t);
  if (lane == 0) *out = t;
}

// single CTA: walk block sums, then scan inside the crossing block.  Device-loop
// form: total, the cumulative end and the uniform draw come from device memory
// (thr = u * cdf_end, the host's arithmetic); total == 0 flags a degenerate step.
__device__ void kpp_search_body(const double* __restrict__ d2, long long n, double total,
                                const double* __restrict__ bs, int nblk, double thr, long long* out);

__global__ void kpp_search_dev_kernel(const double* __restrict__ d2, long long n, const double* total_p,
                                      const double* __restrict__ bs, int nblk, const double* cdf_p,
                                      const double* u, long long* out, int* degenerate) {
  const double total = *total_p;
  if (!(total > 0.0)) {
    if (threadIdx.x == 0) {
      *degenerate = 1;
      *out = 0;
    }
    return;
  }
  kpp_search_body(d2, n, total, bs, nblk, *u * *cdf_p, out);
}

__global__ void kpp_search_kernel(const double* __restrict__ d2, long long n, double total,
                                  const double* __restrict__ bs, int nblk, double thr, long long* out) {
  kpp_search_body(d2, n, total, bs, nblk, thr, out);
}

// inclusive scan of one value per thread over the CTA (fixed shape: warp shuffles, then
// the warp totals), plus the CTA total; blockDim.x == 1024
__device__ __forceinline__ double cta_scan(double v, double* wsum, double* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    double z = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  const double r = v + (w ? wsum[w - 1] : 0.0);
  *total = wsum[31];
  __syncthreads();
  return r;
}

// The pick: the first row whose running sum of p = d2 / total exceeds thr, found in
// two parallel scans (block sums, 1024 at a time with a carried base; then the 2048
// rows of the crossing block, two per thread).  Fixed arithmetic order, so the pick
// is deterministic; it differs from a sequential walk only by rounding.
__device__ void kpp_search_body(const double* __restrict__ d2, long long n, double total,
                                const double* __restrict__ bs, int nblk, double thr, long long* out) {
  __shared__ double wsum[32];
  __shared__ double incl_sh[1024];
  __shared__ int found_sh;
  const int tid = threadIdx.x;
  double base = 0.0;  // sum of the blocks before the current chunk
  int blk = -1;
  for (int c0 = 0; c0 < nblk; c0 += 1024) {
    const int b = c0 + tid;
    if (tid == 0) found_sh = 0x7fffffff;
    double tot;
    const double incl = base + cta_scan(b < nblk ? bs[b] : 0.0, wsum, &tot);
    incl_sh[tid] = incl;
    if (b < nblk && incl > thr) atomicMin(&found_sh, tid);
    __syncthreads();
    const int f = found_sh;
    if (f != 0x7fffffff) {
      blk = c0 + f;
      base = f ? incl_sh[f - 1] : base;
      break;
    }
    base += tot;
    __syncthreads();
  }
  if (blk < 0) {  // rounding at the very end: the last bin, like searchsorted
    blk = nblk - 1;
    base -= bs[nblk - 1];
  }
  __syncthreads();
  const long long lo = (long long)blk * KPP_BLOCK;
  // two rows per thread, in order
  const long long r0 = lo + 2LL * tid, r1 = r0 + 1;
  const double p0 = r0 < n ? d2[r0] / total : 0.0;
  const double p1 = r1 < n ? d2[r1] / total : 0.0;
  if (tid == 0) found_sh = 0x7fffffff;
  double tot;
  const double incl = base + cta_scan(p0 + p1, wsum, &tot);
  incl_sh[tid] = incl;
  __syncthreads();
  const double before = tid ? incl_sh[tid - 1] : base;
  if (r0 < n) {
    if (before + p0 > thr) atomicMin(&found_sh, 2 * tid);
    else if (r1 < n && incl > thr) atomicMin(&found_sh, 2 * tid + 1);
  }
  __syncthreads();
  if (tid == 0) {
    long long f = found_sh == 0x7fffffff ? lo + KPP_BLOCK - 1 : lo + found_sh;  // (rounding: the block's end)
    if (f >= n) f = n - 1;
    *out = f;
  }
}

__global__ void validate_kernel(const double* __restrict__ X, long long n, int d, int k,
                                const int32_t* __restrict__ assign, const double* __restrict__ upper,
                                const double* __restrict__ means, long long* bad) {
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n;
       r += (long long)gridDim.x * blockDim.x) {
    const double* x = X + r * d;
    double bd = CUDART_INF;
    int bi = 0;
    for (int j = 0; j < k; ++j) {
      const double dj = sqrt(exact_sq_rt(x, means + (long long)j * d, d));
      if (dj < bd) { bd = dj; bi = j; }
    }
    const int a = assign[r];
    if (a != bi) atomicMin(reinterpret_cast<unsigned long long*>(&bad[0]), (unsigned long long)r);
    const double td = sqrt(exact_sq_rt(x, means + (long long)a * d, d));
    const double slack = 1e-9 * fmax(1.0, td);
    if (upper[r] + slack < td) atomicMin(reinterpret_cast<unsigned long long*>(&bad[1]), (unsigned long long)r);
  }
}

template <typename T>
__global__ void check_finite_kernel(const T* __restrict__ X, long long total, int d, long long* first_bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    if (!isfinite(X[i])) atomicMin(reinterpret_cast<unsigned long long*>(first_bad), (unsigned long long)(i / d));
  }
}

}  // namespace

cudaError_t launch_gather_rows(const void* X, int elem, long long n_local, long long row_lo, int d,
                               const long long* ids, int count, double* out, cudaStream_t s) {
  long long tot = (long long)count * d;
  int blocks = (int)((tot + 255) / 256);
  if (blocks < 1) blocks = 1;
  if (blocks > 4096) blocks = 4096;
  if (elem == 4)
    gather_rows_kernel<<<blocks, 256, 0, s>>>(static_cast<const float*>(X), n_local, row_lo, d, ids, count, out);
  else
    gather_rows_kernel<<<blocks, 256, 0, s>>>(static_cast<const double*>(X), n_local, row_lo, d, ids, count, out);
  return cudaGetLastError();
}

cudaError_t launch_kpp_update(const void* X, int elem, long long n, int d, const double* c, double* d2, int first,
                              double* block_sums, int nblk, cudaStream_t s) {
  const bool vec = elem == 8 && (d % 2 == 0) && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  const double* Xd = static_cast<const double*>(X);
  if (vec && d <= 8)
    return launch_kpp_tile<8>(Xd, n, d, c, d2, first, block_sums, nblk, s);
  else if (vec && d <= 16)
    return launch_kpp_tile<16>(Xd, n, d, c, d2, first, block_sums, nblk, s);
  else if (vec && d <= 32)
    return launch_kpp_tile<32>(Xd, n, d, c, d2, first, block_sums, nblk, s);
  else if (elem == 4)
    kpp_update_kernel<<<nblk, 256, 0, s>>>(static_cast<const float*>(X), n, d, c, d2, first, block_sums);
  else
    kpp_update_kernel<<<nblk, 256, 0, s>>>(Xd, n, d, c, d2, first, block_sums);
  return cudaGetLastError();
}

cudaError_t launch_kpp_psums(const double* d2, long long n, double total, double* block_sums, int nblk,
                             cudaStream_t s) {
  kpp_psums_kernel<<<nblk, 256, 0, s>>>(d2, n, total, block_sums);
  return cudaGetLastError();
}

cudaError_t launch_sum_blocks(const double* block_sums, int nblk, double* out, cudaStream_t s) {
  sum_blocks_kernel<<<1, 32, 0, s>>>(block_sums, nblk, out);
  return cudaGetLastError();
}

cudaError_t launch_kpp_search(const double* d2, long long n, double total, const double* block_sums, int nblk,
                              double threshold, long long* out, cudaStream_t s) {
  kpp_search_kernel<<<1, 1024, 0, s>>>(d2, n, total, block_sums, nblk, threshold, out);
  return cudaGetLastError();
}

cudaError_t launch_kpp_psums_dev(const double* d2, long long n, const double* total, double* block_sums, int nblk,
                                 cudaStream_t s) {
  kpp_psums_dev_kernel<<<nblk, 256, 0, s>>>(d2, n, total, block_sums);
  return cudaGetLastError();
}

cudaError_t launch_kpp_search_dev(const double* d2, long long n, const double* total, const double* block_sums,
                                  int nblk, const double* cdf_end, const double* u, long long* out, int* degenerate,
                                  cudaStream_t s) {
  kpp_search_dev_kernel<<<1, 1024, 0, s>>>(d2, n, total, block_sums, nblk, cdf_end, u, out, degenerate);
  return cudaGetLastError();
}

cudaError_t launch_gather_row_dev(const void* X, int elem, int d, const long long* idx, double* dst, cudaStream_t s) {
  if (elem == 4) gather_row_dev_kernel<<<1, 256, 0, s>>>(static_cast<const float*>(X), d, idx, dst);
  else gather_row_dev_kernel<<<1, 256, 0, s>>>(static_cast<const double*>(X), d, idx, dst);
  return cudaGetLastError();
}

cudaError_t launch_validate(const double* X, long long n, int d, int k, const int32_t* assign,
                            const double* upper, const double* means, long long* bad, cudaStream_t s) {
  validate_kernel<<<592, 256, 0, s>>>(X, n, d, k, assign, upper, means, bad);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const void* X, int elem, long long n, int d, long long* first_bad, cudaStream_t s) {
  if (elem == 4)
    check_finite_kernel<<<1184, 256, 0, s>>>(static_cast<const float*>(X), n * d, d, first_bad);
  else
    check_finite_kernel<<<1184, 256, 0, s>>>(static_cast<const double*>(X), n * d, d, first_bad);
  return cudaGetLastError();
}

}  // namespace knb
