// K1 generic path and the dispatch between the K1 variants.
//
// The fast path for d <= 64 is the FP64 tensor-core kernel in assign_mma.cu.  This
// file keeps the generic kernel (d > 64, or centroids too large for shared memory):
// every distance is the exact recipe (distance.py:28-39), the ascending strict-less
// scan of distance.py:94-116, and the same mask-based deterministic accumulation
// with the CTA partial kept in global memory (one owner thread per (cluster, dim)).
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Generic path (d > 64, or k too large for shared memory): exact recipe for every
// distance, points and centroids read through L1/L2, CTA partial kept in global
// memory (each (cluster, dim) pair has a single owner thread, so no atomics).
__global__ void __launch_bounds__(KNB_NT) dense_generic_kernel(const DenseArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* masks = reinterpret_cast<uint32_t*>(smem);             // KNB_WARPS * k
  double* xsq = reinterpret_cast<double*>(smem + align_up((size_t)KNB_WARPS * k * 4, 16));
  double* red = xsq + KNB_NT;
  const long long Lg = acc_len(k, d);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  for (long long i = tid; i < Lg; i += KNB_NT) out[i] = 0.0;
  const bool labels = a.labels_only != 0;
  const long long ntiles = (a.n + KNB_NT - 1) / KNB_NT;
  long long reassigned = 0, rows_done = 0;
  double wcss = 0.0;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int i = tid; i < KNB_WARPS * k; i += KNB_NT) masks[i] = 0u;
    const long long row = tile * KNB_NT + tid;
    const bool valid = row < a.n;
    int bid = -1, oldid = -1;
    if (valid) {
      const double* x = a.X + row * d;
      if (labels) {
        bid = a.assign[row];
      } else {
        oldid = a.assign[row];
        double bd = CUDART_INF, lo = CUDART_INF, hi = CUDART_INF;
        int bi = 0;
        for (int j = 0; j < k; ++j) {
          const double s2 = exact_sq_rt(x, a.means + (long long)j * d, d);
          bool less = s2 < lo;
          if (!less && !(s2 > hi)) less = sqrt(s2) < bd;
          if (less) {
            bd = sqrt(s2);
            bi = j;
            const double b2 = bd * bd;
            lo = b2 * (1.0 - 8.9e-16);
            hi = b2 * (1.0 + 8.9e-16);
          }
        }
        bid = bi;
        const int old = a.assign[row];
        a.assign[row] = bi;
        reassigned += (old != bi);
        if (a.mti_seed) {
          a.upper[row] = bd;
          a.tight[row] = 1;
          xsq[tid] = exact_self_rt(x, d);
        } else {
          wcss += bd * bd;
        }
      }
      ++rows_done;
    }
    const long long row0 = tile * KNB_NT;
    // full passes add every row; later dense passes add moved rows to their new
    // cluster (sign +1) and remove them from the old one (sign -1)
    const bool moved = valid && !labels && bid != oldid;
    for (int pass = 0; pass < (a.delta ? 2 : 1); ++pass) {
      const double sign = pass ? -1.0 : 1.0;
      const int accid = !a.delta ? bid : (moved ? (pass ? oldid : bid) : -1);
      __syncthreads();
      if (pass) for (int i = tid; i < KNB_WARPS * k; i += KNB_NT) masks[i] = 0u;
      __syncthreads();
      {
        const unsigned peers = __match_any_sync(0xffffffffu, accid);
        if (accid >= 0 && lane == __ffs(peers) - 1) masks[warp * k + accid] = peers;
      }
      __syncthreads();
      for (long long pi = tid; pi < (long long)k * d; pi += KNB_NT) {
        const int j = (int)(pi / d), e = (int)(pi - (long long)j * d);
        double s = 0.0, c = 0.0, q = 0.0;
        for (int w = 0; w < KNB_WARPS; ++w) {
          unsigned m = masks[w * k + j];
          if (e == 0) c += __popc(m);
          while (m) {
            const int l = __ffs(m) - 1;
            m &= m - 1;
            const int r = w * 32 + l;
            s += a.X[(row0 + r) * d + e];
            if (e == 0 && a.mti_seed) q += xsq[r];
          }
        }
        out[pi] += sign * s;
        if (e == 0) {
          out[(long long)k * d + j] += sign * c;
          out[(long long)k * d + k + j] += sign * q;
        }
      }
    }
    __syncthreads();
  }
  const double r_re = (double)warp_sum_ll(reassigned);
  const double r_w = warp_sum(wcss);
  const double r_rows = (double)warp_sum_ll(rows_done);
  if (lane == 0) { red[warp * 4 + 0] = r_re; red[warp * 4 + 1] = r_w; red[warp * 4 + 2] = r_rows; }
  __syncthreads();
  if (tid == 0) {
    double t_re = 0, t_w = 0, t_rows = 0;
    for (int w = 0; w < KNB_WARPS; ++w) { t_re += red[w * 4]; t_w += red[w * 4 + 1]; t_rows += red[w * 4 + 2]; }
    double* sc = out + (long long)k * d + 2LL * k;
    sc[S_REASSIGNED] = t_re;
    sc[S_WCSS] = t_w;
    sc[S_COMPUTED] = labels ? 0.0 : t_rows * (double)k;
    sc[S_ROWS] = t_rows;
  }
}

}  // namespace

int dense_tile_dp(int d) { return dense_mma_dp(d); }

int dense_rows_per_tile(int DP) { return DP ? dense_mma_rows() : KNB_NT; }

size_t dense_tile_smem(int DP, int k, int d) { return dense_mma_smem(DP, k, d); }

int dense_tile_grid(int DP, int k, int d, int sms) {
  const size_t sm = dense_tile_smem(DP, k, d);
  int per = (int)((227u * 1024u) / (sm + 1024));
  if (per < 1) per = 1;
  if (per > 2) per = 2;  // register-bound: at most two CTAs' warps per SM
  return sms * per;
}

cudaError_t launch_dense(const CUtensorMap* tmap, const DenseArgs& a, int DP, int grid, cudaStream_t s) {
  if (DP == 0) {
    const size_t sm = (size_t)KNB_WARPS * a.k * 4 + 16 + (KNB_NT + KNB_WARPS * 4) * 8;
    cudaError_t e = cudaFuncSetAttribute(dense_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dense_generic_kernel<<<grid, KNB_NT, sm, s>>>(a);
    return cudaGetLastError();
  }
  return launch_dense_mma(tmap, a, DP, grid, s);
}

}  // namespace knb
