// K1: dense point -> centroid assignment fused with the centroid-sum accumulation.
//
// Replaces numakmeans engine._task_full (engine.py:285-319) and the streaming
// nearest-centroid kernel it calls (distance.py:94-116):
//   * argmin over centroids in ascending id order, strict-less (lowest id wins ties);
//   * reassignment count against the previous assignment (engine.py:303-304);
//   * on the full pass of a pruned run, seeds upper = nearest distance, tight = 1
//     and the per-cluster squared-norm sums (engine.py:305-308); otherwise the
//     dense WCSS term sum(nearest^2) (engine.py:310);
//   * per-cluster counts and sums (engine.py:311-318).
//
// Register path (d <= 64): point tiles stream HBM -> shared memory through a
// double-buffered 2-D TMA (hardware 128/64/32-byte swizzle) or, when the row
// stride is not 16-byte aligned, through cp.async into the same layout.  Each
// thread keeps P points in registers and scores centroids staged in shared
// memory with the norm form  s_j = x.c_j - ||c_j||^2/2  (one DFMA per
// point-centroid-dim).  Every comparison also maintains a near-tie flag with
// integer ops only; a point is "certified" when no other centroid scored within
// tol = (8d+32) 2^-53 (||x||^2 + max||c||^2) of the winner, which bounds the
// rounding of both the norm form and the reference's subtract-square recipe, so
// the certified winner IS the reference's argmin.  Uncertified points (near
// ties; practically never) are re-ranked with the exact recipe over all k.
// The winner's distance is then recomputed with the exact recipe (bit-identical
// to the oracle where the host BLAS tree matches).
//
// Accumulation is deterministic without atomics: per 32-row group a warp
// publishes one member mask per cluster (match.any), then thread (dim e,
// group g) owns clusters j = g mod NG and adds members' values in row order
// into CTA-private shared-memory sums.  The CTA writes one partial; a fixed-
// order reduction (update.cu) combines partials -- the GPU analogue of the
// per-task accumulators and task-ordered merge (engine.py:10-13,
// centroids.py:88-107).
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

template <int DP, int P>
struct DenseCfg {
  static constexpr int R = KNB_NT * P;  // rows per tile
  static constexpr int RG = R / 32;     // 32-row groups per tile
  using TL = TileLayout<DP>;
  static constexpr int TILE_BYTES = TL::tile_bytes(R);
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// shared-memory carve-up, identical on host (sizing) and device
struct DenseSmem {
  size_t xb0, xb1, C, chn, acc, cnt, sq, xsq, masks, mbar, red, total;
  __host__ __device__ DenseSmem(int tile_bytes, int R, int RG, int DP, int k) {
    const int kp = (k + 1) & ~1;
    size_t o = 0;
    xb0 = o; o += tile_bytes;
    xb1 = o; o += tile_bytes;
    C = o;   o += (size_t)kp * DP * 8;
    chn = o; o += (size_t)kp * 8;
    acc = o; o += (size_t)k * DP * 8;
    cnt = o; o += (size_t)k * 8;
    sq = o;  o += (size_t)k * 8;
    xsq = o; o += (size_t)R * 8;
    masks = o; o += (size_t)RG * k * 4;
    o = align_up(o, 16);
    mbar = o; o += 16;
    red = o;  o += KNB_WARPS * 4 * 8;
    total = o;
  }
};

__device__ __forceinline__ void score_update(double& best, int& bid, bool& flag, double s, int j,
                                             int tolhi) {
  const double diff = __dsub_rn(s, best);
  const int h = __double2hiint(diff);
  const bool better = h > 0;
  const bool near = (h & 0x7fffffff) <= tolhi;
  flag = near | (flag & !better);
  best = better ? s : best;
  bid = better ? j : bid;
}

// Issue the load of tile `tile` into buffer `dst` (TMA: one thread; cp.async: all threads).
template <int DP, int P>
__device__ __forceinline__ void issue_tile(const CUtensorMap* tmap, uint64_t* bar, unsigned char* dst,
                                           long long tile, const DenseArgs& a, bool tma) {
  using Cfg = DenseCfg<DP, P>;
  using TL = typename Cfg::TL;
  constexpr int R = Cfg::R;
  const long long row0 = tile * R;
  if (tma) {
    if (threadIdx.x == 0) {
      constexpr int BR = R < 256 ? R : 256;  // TMA box rows are capped at 256
      mbar_arrive_expect_tx(bar, Cfg::TILE_BYTES);
#pragma unroll
      for (int p = 0; p < TL::NPANEL; ++p)
#pragma unroll
        for (int h = 0; h < R / BR; ++h)
          tma_load_2d(dst + p * R * TL::RB + h * BR * TL::RB, tmap, bar, p * TL::PW, (int)(row0 + h * BR));
    }
  } else {
    const long long rows_ll = a.n - row0 < R ? a.n - row0 : R;
    const int rows = (int)rows_ll;
    const int d = a.d;
    const double* src = a.X + row0 * d;
    if (((d & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0)) {
      const int hd = d >> 1;
      const int total = rows * hd;
      for (int i = threadIdx.x; i < total; i += KNB_NT) {
        const int r = i / hd, q = i - r * hd;
        cp_async16(dst + TL::chunk_off(r, q, R), src + 2LL * i);
      }
    } else {
      const int total = rows * d;
      for (int i = threadIdx.x; i < total; i += KNB_NT) {
        const int r = i / d, e = i - r * d;
        cp_async8(dst + TL::elem_off(r, e, R), src + i);
      }
    }
    cp_async_commit();
  }
}

template <int DP, int P>
__global__ void __launch_bounds__(KNB_NT, 1)
    dense_tile_kernel(const __grid_constant__ CUtensorMap tmap, const DenseArgs a) {
  using Cfg = DenseCfg<DP, P>;
  using TL = typename Cfg::TL;
  constexpr int R = Cfg::R, RG = Cfg::RG;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;

  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kp = (k + 1) & ~1;
  const DenseSmem L(Cfg::TILE_BYTES, R, RG, DP, k);
  unsigned char* xb[2] = {smem + L.xb0, smem + L.xb1};
  double* C = reinterpret_cast<double*>(smem + L.C);
  double* chn = reinterpret_cast<double*>(smem + L.chn);
  double* acc = reinterpret_cast<double*>(smem + L.acc);
  double* cnt = reinterpret_cast<double*>(smem + L.cnt);
  double* sqa = reinterpret_cast<double*>(smem + L.sq);
  double* xsq = reinterpret_cast<double*>(smem + L.xsq);
  uint32_t* masks = reinterpret_cast<uint32_t*>(smem + L.masks);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  double* red = reinterpret_cast<double*>(smem + L.red);
  const bool tma = a.use_tma != 0;
  const bool labels = a.labels_only != 0;

  // stage centroids (zero-padded to DP dims; an odd k gets a dummy that never wins)
  for (int i = tid; i < kp * DP; i += KNB_NT) {
    const int j = i / DP, e = i - j * DP;
    C[i] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
  }
  for (int j = tid; j < kp; j += KNB_NT) chn[j] = j < k ? a.chn[j] : -CUDART_INF;
  for (int i = tid; i < k * DP; i += KNB_NT) acc[i] = 0.0;
  for (int j = tid; j < k; j += KNB_NT) { cnt[j] = 0.0; sqa[j] = 0.0; }
  if (!tma) {  // padded columns stay zero for the whole kernel
    if (d < DP) {
      for (int b = 0; b < 2; ++b)
        for (int i = tid; i < R * DP; i += KNB_NT) {
          const int r = i / DP, e = i - r * DP;
          if (e >= d) *reinterpret_cast<double*>(xb[b] + TL::elem_off(r, e, R)) = 0.0;
        }
    }
  }
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
    if (tma) prefetch_tmap(&tmap);
  }
  __syncthreads();

  const double cmax2 = a.ctrl->cmax2;
  const double tolk = (8.0 * d + 32.0) * 1.1102230246251565e-16;  // (8d+32) * 2^-53
  const long long ntiles = (a.n + R - 1) / R;
  long long reassigned = 0;
  double wcss = 0.0;
  long long rows_done = 0;
  uint32_t phase[2] = {0u, 0u};
  int buf = 0;

  if ((long long)blockIdx.x < ntiles) issue_tile<DP, P>(&tmap, &bar[0], xb[0], blockIdx.x, a, tma);

  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long next = tile + gridDim.x;
    if (next < ntiles) issue_tile<DP, P>(&tmap, &bar[buf ^ 1], xb[buf ^ 1], next, a, tma);
    for (int i = tid; i < RG * k; i += KNB_NT) masks[i] = 0u;
    if (tma) {
      mbar_wait(&bar[buf], phase[buf]);
      phase[buf] ^= 1u;
    } else {
      if (next < ntiles) cp_async_wait_1(); else cp_async_wait_all();
    }
    __syncthreads();
    const unsigned char* tb = xb[buf];
    const long long row0 = tile * R;

    int bid[P];
    bool valid[P];
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int r = p * KNB_NT + tid;
      const long long row = row0 + r;
      valid[p] = row < a.n;
      bid[p] = 0;
    }

    if (!labels) {
      double x[P][DP];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int r = p * KNB_NT + tid;
#pragma unroll
        for (int q = 0; q < DP / 2; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, q, R));
          x[p][2 * q] = v.x;
          x[p][2 * q + 1] = v.y;
        }
      }
      double best[P];
      bool flag[P];
      int tolhi[P];
#pragma unroll
      for (int p = 0; p < P; ++p) {
        double xn2 = 0.0;
#pragma unroll
        for (int e = 0; e < DP; ++e) xn2 = fma(x[p][e], x[p][e], xn2);
        tolhi[p] = __double2hiint(tolk * (xn2 + cmax2));
        best[p] = -CUDART_INF;
        flag[p] = false;
      }
#pragma unroll 1
      for (int j = 0; j < kp; j += 2) {
        const double* c0 = C + j * DP;
        const double* c1 = c0 + DP;
        double s0[P], s1[P];
#pragma unroll
        for (int p = 0; p < P; ++p) { s0[p] = chn[j]; s1[p] = chn[j + 1]; }
#pragma unroll
        for (int q = 0; q < DP / 2; ++q) {
          const double2 a0 = *reinterpret_cast<const double2*>(c0 + 2 * q);
          const double2 a1 = *reinterpret_cast<const double2*>(c1 + 2 * q);
#pragma unroll
          for (int p = 0; p < P; ++p) {
            s0[p] = fma(x[p][2 * q], a0.x, s0[p]);
            s1[p] = fma(x[p][2 * q], a1.x, s1[p]);
            s0[p] = fma(x[p][2 * q + 1], a0.y, s0[p]);
            s1[p] = fma(x[p][2 * q + 1], a1.y, s1[p]);
          }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
          score_update(best[p], bid[p], flag[p], s0[p], j, tolhi[p]);
          score_update(best[p], bid[p], flag[p], s1[p], j + 1, tolhi[p]);
        }
      }
#pragma unroll
      for (int p = 0; p < P; ++p) {
        const int r = p * KNB_NT + tid;
        double nd;
        if (flag[p]) {  // near tie: exact re-rank over every centroid (distance.py:106-116)
          double bd = CUDART_INF;
          int bi = 0;
          for (int j = 0; j < k; ++j) {
            const double dj = sqrt(exact_sq<DP>(x[p], C + j * DP, d));
            if (dj < bd) { bd = dj; bi = j; }
          }
          bid[p] = bi;
          nd = bd;
        } else {
          nd = sqrt(exact_sq<DP>(x[p], C + bid[p] * DP, d));
        }
        if (valid[p]) {
          const long long row = row0 + r;
          const int old = a.assign[row];
          a.assign[row] = bid[p];
          reassigned += (old != bid[p]);
          if (a.mti_seed) {
            a.upper[row] = nd;
            a.tight[row] = 1;
            xsq[r] = exact_sq<DP>(x[p], Zero{}, d);
          } else {
            wcss += nd * nd;
          }
          ++rows_done;
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < P; ++p)
        if (valid[p]) { bid[p] = a.assign[row0 + p * KNB_NT + tid]; ++rows_done; }
    }
    __syncthreads();  // masks zeroed by everyone before publication
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int id = valid[p] ? bid[p] : -1;
      const unsigned peers = __match_any_sync(0xffffffffu, id);
      if (id >= 0 && lane == __ffs(peers) - 1) masks[(p * KNB_WARPS + warp) * k + id] = peers;
    }
    __syncthreads();
    {  // deterministic segmented accumulation, members in row order
      constexpr int NG = KNB_NT / DP;
      const int e = tid % DP, g = tid / DP;
      if (e < d) {
        for (int j = g; j < k; j += NG) {
          double s = 0.0, c = 0.0, q = 0.0;
          for (int rg = 0; rg < RG; ++rg) {
            unsigned m = masks[rg * k + j];
            if (e == 0) c += __popc(m);
            while (m) {
              const int l = __ffs(m) - 1;
              m &= m - 1;
              const int r = rg * 32 + l;
              s += *reinterpret_cast<const double*>(tb + TL::elem_off(r, e, R));
              if (e == 0 && a.mti_seed) q += xsq[r];
            }
          }
          acc[j * DP + e] += s;
          if (e == 0) { cnt[j] += c; sqa[j] += q; }
        }
      }
    }
    __syncthreads();  // tile buffer and masks free for reuse
    buf ^= 1;
  }

  // CTA partial (every CTA writes one, even with no tiles, so the reduce is uniform)
  const long long Lg = acc_len(k, d);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  for (int i = tid; i < k * d; i += KNB_NT) {
    const int j = i / d, e = i - j * d;
    out[i] = acc[j * DP + e];
  }
  for (int j = tid; j < k; j += KNB_NT) {
    out[(long long)k * d + j] = cnt[j];
    out[(long long)k * d + k + j] = sqa[j];
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
    for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
    sc[S_REASSIGNED] = t_re;
    sc[S_WCSS] = t_w;
    sc[S_COMPUTED] = labels ? 0.0 : t_rows * (double)k;
    sc[S_ROWS] = t_rows;
  }
}

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
    int bid = -1;
    if (valid) {
      const double* x = a.X + row * d;
      if (labels) {
        bid = a.assign[row];
      } else {
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
    __syncthreads();
    {
      const unsigned peers = __match_any_sync(0xffffffffu, bid);
      if (bid >= 0 && lane == __ffs(peers) - 1) masks[warp * k + bid] = peers;
    }
    __syncthreads();
    const long long row0 = tile * KNB_NT;
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
      out[pi] += s;
      if (e == 0) {
        out[(long long)k * d + j] += c;
        out[(long long)k * d + k + j] += q;
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

template <int DP, int P>
cudaError_t launch_tile(const CUtensorMap* tmap, const DenseArgs& a, int grid, cudaStream_t s) {
  using Cfg = DenseCfg<DP, P>;
  const DenseSmem L(Cfg::TILE_BYTES, Cfg::R, Cfg::RG, DP, a.k);
  auto fn = dense_tile_kernel<DP, P>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  fn<<<grid, KNB_NT, L.total, s>>>(*tmap, a);
  return cudaGetLastError();
}

}  // namespace

// points per thread for each padded width (register budget vs shared-memory reuse)
#define KNB_DENSE_CASES(X) X(2, 2) X(4, 2) X(8, 2) X(16, 2) X(32, 1) X(64, 1)

int dense_tile_dp(int d) {
  if (d <= 2) return 2;
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  if (d <= 64) return 64;
  return 0;
}

static int points_per_thread(int DP) {
#define X(dp, p) if (DP == dp) return p;
  KNB_DENSE_CASES(X)
#undef X
  return 1;
}

int dense_rows_per_tile(int DP) { return DP ? KNB_NT * points_per_thread(DP) : KNB_NT; }

size_t dense_tile_smem(int DP, int k) {
  const int P = points_per_thread(DP);
  const int R = KNB_NT * P;
  const DenseSmem L(R * DP * 8, R, R / 32, DP, k);
  return L.total;
}

int dense_tile_grid(int DP, int k, int sms) {
  const size_t sm = dense_tile_smem(DP, k);
  int per = (int)((227u * 1024u) / (sm + 1024));
  if (per < 1) per = 1;
  if (per > 4) per = 4;
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
#define X(dp, p) if (DP == dp) return launch_tile<dp, p>(tmap, a, grid, s);
  KNB_DENSE_CASES(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace knb
