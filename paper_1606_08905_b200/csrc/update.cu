// K3 stage 2 + K4 + K5 + K9: fixed-order reduction of CTA partials, centroid
// finalize, WCSS/statistics, convergence test and MTI geometry -- the barrier
// action of numakmeans (engine.py:358-426) on device.
//
//   reduce      sum the G CTA partials element by element in CTA order (fixed
//               order -> bit-reproducible for a fixed grid; centroids.py:88-107
//               merges per-task accumulators in task order for the same reason)
//   finalize    pruned runs add the (all-reduced) deltas into running totals
//               (engine.py:371-375); means = sums / counts for occupied
//               clusters, empty clusters keep their previous mean; drift is the
//               exact-recipe distance old -> new, 0 when empty
//               (centroids.py:110-128); per-cluster WCSS terms for pruned runs
//               (engine.py:385-388)
//   stats       Sigma counts == n check (engine.py:378-380), WCSS, the
//               IterationStats row, converged = reassigned <= tolerance, stop
//               when converged or t + 1 >= max_iters (engine.py:413-416)
//   geometry    half_dist[a][b] = 0.5 * d(c_a, c_b) (exact recipe) and the row
//               minima off the diagonal, +inf for k == 1 (pruning.py:48-61)
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

constexpr int GEO_PAIRS_MAX_K = 256;  // beyond: one warp per row (k^2 warps would be many)

// LPE lanes per element: lane q sums CTA partials [q*S, (q+1)*S) in CTA order
// (S = ceil(G/LPE), loads batched 16 deep), then the LPE sums combine in a fixed
// butterfly -- a fixed order for a given (G, L), so runs are bit-reproducible.  Short
// vectors (the usual case: k*d + 2k + 8 doubles) take 32 lanes per element so that
// every partial's load is in flight at once; the pass is one memory round trip.
template <int LPE>
__global__ void reduce_kernel(const double* __restrict__ partials, int G, long long L,
                              double* __restrict__ out, const Ctrl* ctrl) {
  pdl_enter();
  if (ctrl->stop && !ctrl->ignore_stop) return;
  constexpr int EPW = 32 / LPE;  // elements per warp
  const int q = threadIdx.x & (LPE - 1);
  const int S = (G + LPE - 1) / LPE;
  const int b0 = q * S, b1 = b0 + S < G ? b0 + S : G;
  for (long long e0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / LPE; e0 < ((L + EPW - 1) / EPW) * EPW;
       e0 += ((long long)gridDim.x * blockDim.x) / LPE) {
    const long long e = e0 < L ? e0 : L - 1;
    double s = 0.0;
    int b = b0;
    for (; b + 16 <= b1; b += 16) {
      double v[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) v[t] = partials[(long long)(b + t) * L + e];
#pragma unroll
      for (int t = 0; t < 16; ++t) s += v[t];
    }
    double v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = b + t < b1 ? partials[(long long)(b + t) * L + e] : 0.0;
#pragma unroll
    for (int t = 0; t < 16; ++t)
      if (b + t < b1) s += v[t];
#pragma unroll
    for (int o = 1; o < LPE; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (q == 0 && e0 < L) out[e] = s;
  }
}

__device__ void finalize_centroid(const FinalArgs& f, int j);
__device__ void stats_body(const FinalArgs& f);
__device__ void geometry_row(const FinalArgs& f, int a);

// One warp per centroid; the last CTA to finish then runs the statistics row (one
// launch instead of two; the MTI geometry stays a separate, wider kernel).
__global__ void finalize_kernel(const FinalArgs f) {
  pdl_enter();
  if (f.ctrl->stop && !f.ctrl->ignore_stop) return;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j < f.k) finalize_centroid(f, j);
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(f.sync, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  stats_body(f);
  if (threadIdx.x == 0) *f.sync = 0u;  // ready for the next iteration (graph replays)
}

__device__ void finalize_centroid(const FinalArgs& f, int j) {
  const int k = f.k, d = f.d;
  const int lane = threadIdx.x & 31;
  const long long kd = (long long)k * d;
  double* sums = f.exch + (long long)j * d;
  double cntj = f.exch[kd + j];
  double sqj = f.exch[kd + k + j];
  {  // running totals += this iteration's merged vector: full totals on the first pass,
     // signed deltas of moved rows afterwards (pruned runs: engine.py:371-375)
    double* rs = f.run + (long long)j * d;
    for (int e = lane; e < d; e += 32) rs[e] += sums[e];
    __syncwarp();
    if (lane == 0) {
      f.run[kd + j] += cntj;
      f.run[kd + k + j] += sqj;
    }
    __syncwarp();
    sums = rs;
    cntj = f.run[kd + j];
    sqj = f.run[kd + k + j];
  }
  double* m = f.means + (long long)j * d;
  double* pv = f.prev + (long long)j * d;
  const bool occ = cntj > 0.0;
  if (f.wcss_mode == 2) {
    // unpruned WCSS against the centroids the pass assigned with (engine.py:331-333),
    // from the running totals of the new assignment: sum ||x - c||^2 over the
    // cluster = Q - 2 c.S + count ||c||^2 (tensor-core pass: no per-row exact distance)
    double cs = 0.0, cc = 0.0;
    for (int e = lane; e < d; e += 32) {
      const double o = m[e];
      cs += o * sums[e];
      cc += o * o;
    }
    cs = warp_sum(cs);
    cc = warp_sum(cc);
    if (lane == 0) f.wterm[j] = occ ? sqj - 2.0 * cs + cntj * cc : 0.0;
    __syncwarp();
  }
  for (int e = lane; e < d; e += 32) {
    const double old = m[e];
    pv[e] = old;
    if (occ) m[e] = sums[e] / cntj;
  }
  __syncwarp();
  // (lane 0's sequential trees: measured faster here than warp_exact_sq's shuffle chain)
  if (lane == 0) {
    if (f.pruning && k <= GEO_PAIRS_MAX_K) {  // the pair-wise geometry fills in the rest
      f.half_min[j] = CUDART_INF;
      f.half[(long long)j * k + j] = 0.0;
    }
    f.drift[j] = occ ? sqrt(exact_sq_rt(m, pv, d)) : 0.0;
    f.counts[j] = cntj;
    const double n2 = exact_self_rt(m, d);
    f.cn2[j] = n2;
    f.chn[j] = -0.5 * n2;
    if (f.wcss_mode == 1) {  // sq - ||sums||^2 / count, clamped at 0 (engine.py:385-388)
      double s2 = 0.0;
      for (int e = 0; e < d; ++e) s2 += sums[e] * sums[e];
      const double term = sqj - s2 / cntj;
      f.wterm[j] = occ ? (term > 0.0 ? term : 0.0) : 0.0;
    }
  }
}

// the statistics row + convergence test, by one CTA after every centroid is final
__device__ void stats_body(const FinalArgs& f) {
  Ctrl* c = f.ctrl;
  __shared__ double sw[32];
  __shared__ double sc[32];
  __shared__ double sm[32];
  const int k = f.k, d = f.d, tid = threadIdx.x;
  double cs = 0.0, ws = 0.0, mx = 0.0;
  for (int j = tid; j < k; j += blockDim.x) {
    cs += f.counts[j];
    if (f.wcss_mode) ws += f.wterm[j];
    mx = fmax(mx, f.cn2[j]);
  }
  cs = warp_sum(cs);
  ws = warp_sum(ws);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) { sc[tid >> 5] = cs; sw[tid >> 5] = ws; sm[tid >> 5] = mx; }
  __syncthreads();
  if (tid == 0) {
    double C = 0.0, W = 0.0, M = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { C += sc[w]; W += sw[w]; M = fmax(M, sm[w]); }
    const double* scal = f.exch + (long long)k * d + 2LL * k;
    const long long t = c->t;
    IterStatsDev st;
    st.t = t;
    st.reassignments = (long long)scal[S_REASSIGNED];
    st.wcss = f.wcss_mode ? W : scal[S_WCSS];
    st.dist_comps = (long long)scal[S_COMPUTED];
    st.skips = (long long)scal[S_SKIPS];
    st.pruned_stale = (long long)scal[S_PSTALE];
    st.pruned_tight = (long long)scal[S_PTIGHT];
    st.count_total = (long long)C;
    if ((long long)C != f.n) c->count_error = 1;
    c->count_seen = (long long)C;
    const int conv = (double)st.reassignments <= c->tolerance;
    const int stop = conv || (t + 1 >= c->max_iters);
    st.converged = conv;
    st.stop = stop;
    if (t < c->max_iters) f.stats[t] = st;
    c->converged = conv;
    c->stop = stop;
    // adaptive MTI kernel for the next pass: streaming every block only beats
    // compacting the survivors when clause 1 skips almost nothing (measured: c2 with
    // 49% skips 0.46 vs 0.28 ms, c4 with 0% skips 183 vs 190 ms)
    c->mti_choice = (double)st.skips < 0.01 * c->block_pct * (double)f.n ? 1 : 0;
    c->cmax2 = M;
    c->full_pass = 0;
    c->t = t + 1;
  }
}


// one warp per row a of the half-distance matrix
__device__ void geometry_row(const FinalArgs& f, int a) {
  const int k = f.k, d = f.d, lane = threadIdx.x & 31;
  const double* ca = f.means + (long long)a * d;
  double mn = CUDART_INF;
  for (int b = lane; b < k; b += 32) {
    double h = 0.0;
    if (b != a) {
      // rowwise_distances(means[a+1:], means[a]) * 0.5 for a < b; the subtract's
      // sign cannot change a square, so the matrix is exactly symmetric
      const double* lo = a < b ? f.means + (long long)b * d : ca;
      const double* hi = a < b ? ca : f.means + (long long)b * d;
      h = sqrt(exact_sq_rt(lo, hi, d)) * 0.5;
      mn = fmin(mn, h);
    }
    f.half[(long long)a * k + b] = h;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if (lane == 0) f.half_min[a] = mn;  // +inf when k == 1
}

// k <= GEO_PAIRS_MAX_K: one warp per centroid pair a < b (warp-wide exact tree), the
// row minima by atomicMin on the bit patterns (non-negative doubles order like their
// bits; min is order-free, so the result is deterministic).  finalize reset half_min
// to +inf and the diagonal to 0.
__global__ void geometry_pairs_kernel(const FinalArgs f) {
  pdl_enter();
  const Ctrl* c = f.ctrl;
  if (c->stop && !c->ignore_stop) return;
  const int k = f.k, d = f.d, lane = threadIdx.x & 31;
  const long long p = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (p >= (long long)k * k) return;
  const int a = (int)(p / k), b = (int)(p - (long long)a * k);
  if (b <= a) return;  // warp-uniform
  // rowwise_distances(means[a+1:], means[a]) * 0.5: x = means[b], c = means[a]
  const double h = sqrt(warp_exact_sq(f.means + (long long)b * d, f.means + (long long)a * d, d, lane)) * 0.5;
  if (lane == 0) {
    f.half[(long long)a * k + b] = h;
    f.half[(long long)b * k + a] = h;
    const unsigned long long hb = (unsigned long long)__double_as_longlong(h);
    atomicMin(reinterpret_cast<unsigned long long*>(f.half_min + a), hb);
    atomicMin(reinterpret_cast<unsigned long long*>(f.half_min + b), hb);
  }
}

// The whole barrier action in one CTA for small k (k <= FUSED_MAX_K): every centroid's
// finalize (a warp each), the statistics row and convergence test, then -- pruned runs --
// the pair-wise geometry, with __syncthreads between the phases instead of a grid-wide
// arrival counter and a separate geometry launch (c1: 22.8 -> 21.8 us per iteration).
// (Folding the reduction of the CTA partials in as well, one CTA instead of a grid, was
// slower: c1 28.9 us.)
#ifndef KNB_NO_FUSED_FINISH
#define KNB_NO_FUSED_FINISH 0
#endif
constexpr int FUSED_MAX_K = KNB_NO_FUSED_FINISH ? 0 : 16;
__global__ void __launch_bounds__(512) finish_small_kernel(const FinalArgs f) {
  pdl_enter();
  if (f.ctrl->stop && !f.ctrl->ignore_stop) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int j = warp; j < f.k; j += nw) finalize_centroid(f, j);
  __syncthreads();
  stats_body(f);
  if (!f.pruning) return;
  __syncthreads();
  const int k = f.k, d = f.d;
  for (int p = warp; p < k * k; p += nw) {
    const int a = p / k, b = p - a * k;
    if (b <= a) continue;  // warp-uniform
    const double h = sqrt(warp_exact_sq(f.means + (long long)b * d, f.means + (long long)a * d, d, lane)) * 0.5;
    if (lane == 0) {
      f.half[(long long)a * k + b] = h;
      f.half[(long long)b * k + a] = h;
      const unsigned long long hb = (unsigned long long)__double_as_longlong(h);
      atomicMin(reinterpret_cast<unsigned long long*>(f.half_min + a), hb);
      atomicMin(reinterpret_cast<unsigned long long*>(f.half_min + b), hb);
    }
  }
}

__global__ void geometry_kernel(const FinalArgs f) {
  pdl_enter();
  const Ctrl* c = f.ctrl;
  if (c->stop && !c->ignore_stop) return;
  const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (a >= f.k) return;
  geometry_row(f, a);
}

// Install initial centroids (given / forgy / kmeans++ rows, or random-partition
// group sums) and derive the per-centroid quantities the kernels need.
__global__ void set_means_kernel(const double* src, int k, int d, const FinalArgs f, int from_partition,
                                 long long n) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= k) return;
  double* m = f.means + (long long)j * d;
  double* pv = f.prev + (long long)j * d;
  if (!from_partition) {
    for (int e = lane; e < d; e += 32) m[e] = pv[e] = src[(long long)j * d + e];
  } else {
    // src holds group sums/counts in the accumulator layout; an empty group takes
    // the global mean (centroids.py:164-173)
    const long long kd = (long long)k * d;
    const double cj = src[kd + j];
    for (int e = lane; e < d; e += 32) {
      double v;
      if (cj > 0.0) {
        v = src[(long long)j * d + e] / cj;
      } else {
        double tot = 0.0;
        for (int g = 0; g < k; ++g) tot += src[(long long)g * d + e];
        v = tot / (double)n;
      }
      m[e] = pv[e] = v;
    }
  }
  __syncwarp();
  if (lane == 0) {
    f.drift[j] = 0.0;
    f.counts[j] = 0.0;
    const double n2 = exact_self_rt(m, d);
    f.cn2[j] = n2;
    f.chn[j] = -0.5 * n2;
  }
}

__global__ void cmax_kernel(const FinalArgs f) {
  __shared__ double sm[32];
  double mx = 0.0;
  for (int j = threadIdx.x; j < f.k; j += blockDim.x) mx = fmax(mx, f.cn2[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double M = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) M = fmax(M, sm[w]);
    f.ctrl->cmax2 = M;
  }
}

}  // namespace

cudaError_t launch_reduce(const double* partials, int G, long long L, double* out, const Ctrl* ctrl,
                          cudaStream_t s) {
  if (L <= 8192) {  // latency-bound: every partial in flight
    const long long blocks = (L * 32 + 127) / 128;
    return launch_pdl(reduce_kernel<32>, dim3((unsigned)blocks), dim3(128), 0, s, partials, G, L, out, ctrl);
  } else {
    long long blocks = (L * 8 + 127) / 128;
    if (blocks > 4096) blocks = 4096;
    return launch_pdl(reduce_kernel<8>, dim3((unsigned)blocks), dim3(128), 0, s, partials, G, L, out, ctrl);
  }
}

cudaError_t launch_finalize(const FinalArgs& f, cudaStream_t s) {
  if (f.k <= FUSED_MAX_K) return launch_pdl(finish_small_kernel, dim3(1), dim3(512), 0, s, f);
  const int wpb = 8;
  return launch_pdl(finalize_kernel, dim3((f.k + wpb - 1) / wpb), dim3(wpb * 32), 0, s, f);
}

cudaError_t launch_geometry(const FinalArgs& f, cudaStream_t s) {
  if (f.k <= FUSED_MAX_K) return cudaSuccess;  // (finish_small_kernel did it)
  if (f.k <= GEO_PAIRS_MAX_K) {
    const long long warps = (long long)f.k * f.k;
    return launch_pdl(geometry_pairs_kernel, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0, s, f);
  }
  const int wpb = 8;
  return launch_pdl(geometry_kernel, dim3((f.k + wpb - 1) / wpb), dim3(wpb * 32), 0, s, f);
}

cudaError_t launch_set_means(const double* src, int k, int d, FinalArgs f, int from_partition, long long n,
                             cudaStream_t s) {
  const int wpb = 8;
  set_means_kernel<<<(k + wpb - 1) / wpb, wpb * 32, 0, s>>>(src, k, d, f, from_partition, n);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  cmax_kernel<<<1, 1024, 0, s>>>(f);
  return cudaGetLastError();
}

}  // namespace knb
