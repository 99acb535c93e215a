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

// Same contract and summation order as kpp_update_kernel for f64 rows with d <= DP:
// the row is loaded into registers with 16-byte loads and the centroid is read from
// shared memory, so the pass runs at memory speed.
template <int DP>
__global__ void kpp_update_reg_kernel(const double* __restrict__ X, long long n, int d, const double* __restrict__ c,
                                      double* __restrict__ d2, int first, double* __restrict__ block_sums) {
  __shared__ double sh[32];
  __shared__ double cs[DP];
  for (int e = threadIdx.x; e < DP; e += blockDim.x) cs[e] = e < d ? c[e] : 0.0;
  __syncthreads();
  const long long b = blockIdx.x;
  const long long lo = b * KPP_BLOCK;
  double s = 0.0;
  for (int i = threadIdx.x; i < KPP_BLOCK; i += blockDim.x) {
    const long long r = lo + i;
    if (r >= n) break;
    double x[DP];
    const double2* xr = reinterpret_cast<const double2*>(X + r * d);
#pragma unroll
    for (int q = 0; q < DP / 2; ++q) {
      if (2 * q < d) {
        const double2 v = xr[q];
        x[2 * q] = v.x;
        x[2 * q + 1] = v.y;
      } else {
        x[2 * q] = 0.0;
        x[2 * q + 1] = 0.0;
      }
    }
    const double dist = sqrt(exact_sq<DP>(x, cs, d));
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

__device__ void kpp_search_body(const double* __restrict__ d2, long long n, double total,
                                const double* __restrict__ bs, int nblk, double thr, long long* out) {
  __shared__ double run_sh;
  __shared__ int blk_sh;
  __shared__ double part[1024];
  if (threadIdx.x == 0) {
    double run = 0.0;
    int b = 0;
    for (; b < nblk; ++b) {
      if (run + bs[b] > thr) break;
      run += bs[b];
    }
    if (b == nblk) b = nblk - 1;  // rounding at the very end: clamp like searchsorted's last bin
    blk_sh = b;
    // recompute the base as the sum of the preceding blocks (already in run)
    run_sh = run;
  }
  __syncthreads();
  const long long lo = (long long)blk_sh * KPP_BLOCK;
  const int per = KPP_BLOCK / blockDim.x;  // rows per thread (contiguous)
  double s = 0.0;
  for (int i = 0; i < per; ++i) {
    const long long r = lo + threadIdx.x * per + i;
    if (r < n) s += d2[r] / total;
  }
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = run_sh;
    long long found = -1;
    for (int t = 0; t < (int)blockDim.x && found < 0; ++t) {
      if (run + part[t] > thr) {
        for (int i = 0; i < per; ++i) {
          const long long r = lo + (long long)t * per + i;
          if (r >= n) break;
          run += d2[r] / total;
          if (run > thr) { found = r; break; }
        }
        if (found < 0) found = lo + (long long)t * per + per - 1;
      } else {
        run += part[t];
      }
    }
    if (found < 0) found = n - 1;
    if (found >= n) found = n - 1;
    *out = found;
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
    kpp_update_reg_kernel<8><<<nblk, 256, 0, s>>>(Xd, n, d, c, d2, first, block_sums);
  else if (vec && d <= 16)
    kpp_update_reg_kernel<16><<<nblk, 256, 0, s>>>(Xd, n, d, c, d2, first, block_sums);
  else if (vec && d <= 32)
    kpp_update_reg_kernel<32><<<nblk, 256, 0, s>>>(Xd, n, d, c, d2, first, block_sums);
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
  kpp_search_kernel<<<1, 256, 0, s>>>(d2, n, total, block_sums, nblk, threshold, out);
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
  kpp_search_dev_kernel<<<1, 256, 0, s>>>(d2, n, total, block_sums, nblk, cdf_end, u, out, degenerate);
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
