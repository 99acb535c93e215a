// K6+K7: minimal-triangle-inequality (MTI) pruned iteration.
//
// Replaces numakmeans engine._task_pruned (engine.py:321-354) together with
// inflate_bounds (pruning.py:152-160) and scan_block / scan_point
// (pruning.py:113-149, 163-204), with the same semantics and counters:
//   prologue  u += drift[a]; tight &= (drift[a] == 0)        (bound inflation, fused)
//   clause 1  skip the point when u <= half_min[a]            (inclusive, no row read)
//   tighten   loose bound -> exact distance to a, computed += 1
//   scan      x = 0..k-1 ascending, skipping cur and orig; gap = half_dist[cur][x];
//             u <= gap prunes (stale if the entry bound was already <= gap, else
//             tight); otherwise compute d(v, c_x), computed += 1, switch on strict <
//   deltas    moved points add their row to the new cluster and subtract it from
//             the old one (sums, counts, squared norms), engine.py:345-353.
//
// Layout: a CTA filters a tile of F*NT rows reading only the 13 B/point state
// (assign int32, upper f64, tight u8); survivors are compacted in row order
// with warp ballots and processed NT at a time, one survivor per thread (row
// gathered straight from HBM -- skipped rows are never read).  Every distance
// the scan evaluates uses the exact recipe, so bounds and pruning decisions are
// the reference's own.  sqrt is only evaluated when the squared distance is
// within a few ulps of u^2 or on a switch.  Signed deltas go to CTA-private
// shared-memory accumulators through per-cluster member masks (row order,
// deterministic) and leave as one partial per CTA.
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

constexpr int MTI_F = 4;  // filter rows per thread per tile

__host__ __device__ inline size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct MtiSmem {
  size_t C, hmin, drift, half, acc, cnt, sq, surv, wcnt, mvx, mvsq, mto, mfrom, red, total;
  __host__ __device__ MtiSmem(int DP, int k, int half_in_smem) {
    size_t o = 0;
    C = o;     o += (size_t)k * DP * 8;
    hmin = o;  o += (size_t)k * 8;
    drift = o; o += (size_t)k * 8;
    half = o;  o += half_in_smem ? (size_t)k * k * 8 : 0;
    acc = o;   o += (size_t)k * DP * 8;
    cnt = o;   o += (size_t)k * 8;
    sq = o;    o += (size_t)k * 8;
    mvx = o;   o += (size_t)KNB_NT * (DP + 1) * 8;
    mvsq = o;  o += (size_t)KNB_NT * 8;
    red = o;   o += (size_t)KNB_WARPS * 8 * 8;
    surv = o;  o += (size_t)MTI_F * KNB_NT * 4;
    wcnt = o;  o += (size_t)(MTI_F * KNB_WARPS + 1) * 4;
    o = al(o, 16);
    mto = o;   o += (size_t)KNB_WARPS * k * 4;
    mfrom = o; o += (size_t)KNB_WARPS * k * 4;
    total = al(o, 16);
  }
};

template <int DP>
__global__ void __launch_bounds__(KNB_NT) mti_tile_kernel(const MtiArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const MtiSmem L(DP, k, a.half_in_smem);
  double* C = reinterpret_cast<double*>(smem + L.C);
  double* hmin = reinterpret_cast<double*>(smem + L.hmin);
  double* drift = reinterpret_cast<double*>(smem + L.drift);
  const double* half = a.half_in_smem ? reinterpret_cast<double*>(smem + L.half) : a.half;
  double* acc = reinterpret_cast<double*>(smem + L.acc);
  double* cnt = reinterpret_cast<double*>(smem + L.cnt);
  double* sqa = reinterpret_cast<double*>(smem + L.sq);
  double* mvx = reinterpret_cast<double*>(smem + L.mvx);
  double* mvsq = reinterpret_cast<double*>(smem + L.mvsq);
  double* red = reinterpret_cast<double*>(smem + L.red);
  int* surv = reinterpret_cast<int*>(smem + L.surv);
  int* wcnt = reinterpret_cast<int*>(smem + L.wcnt);
  uint32_t* mto = reinterpret_cast<uint32_t*>(smem + L.mto);
  uint32_t* mfrom = reinterpret_cast<uint32_t*>(smem + L.mfrom);

  for (int i = tid; i < k * DP; i += KNB_NT) {
    const int j = i / DP, e = i - j * DP;
    C[i] = e < d ? a.means[(long long)j * d + e] : 0.0;
    acc[i] = 0.0;
  }
  for (int j = tid; j < k; j += KNB_NT) {
    hmin[j] = a.half_min[j];
    drift[j] = a.drift[j];
    cnt[j] = 0.0;
    sqa[j] = 0.0;
  }
  if (a.half_in_smem) {
    double* hs = reinterpret_cast<double*>(smem + L.half);
    for (int i = tid; i < k * k; i += KNB_NT) hs[i] = a.half[i];
  }
  __syncthreads();

  long long skips = 0, computed = 0, pstale = 0, ptight = 0, reassigned = 0;
  constexpr int TR = MTI_F * KNB_NT;
  const long long ntiles = (a.n + TR - 1) / TR;
  const bool even = ((d & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);

  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long row0 = tile * TR;
    // ---- filter: inflate bounds, clause 1, compaction in row order
    bool live[MTI_F];
    unsigned bal[MTI_F];
#pragma unroll
    for (int f = 0; f < MTI_F; ++f) {
      const long long row = row0 + f * KNB_NT + tid;
      live[f] = false;
      if (row < a.n) {
        const int aa = a.assign[row];
        double u = a.upper[row];
        const double dr = drift[aa];
        if (dr != 0.0) {  // u + 0.0 == u and tight & true == tight: no store needed
          u = u + dr;
          a.upper[row] = u;
          a.tight[row] = 0;
        }
        if (u <= hmin[aa]) ++skips;
        else live[f] = true;
      }
      bal[f] = __ballot_sync(0xffffffffu, live[f]);
      if (lane == 0) wcnt[f * KNB_WARPS + warp] = __popc(bal[f]);
    }
    __syncthreads();
    if (tid == 0) {  // exclusive scan in (f, warp, lane) == row order
      int s = 0;
      for (int i = 0; i < MTI_F * KNB_WARPS; ++i) { const int c = wcnt[i]; wcnt[i] = s; s += c; }
      wcnt[MTI_F * KNB_WARPS] = s;
    }
    __syncthreads();
#pragma unroll
    for (int f = 0; f < MTI_F; ++f)
      if (live[f]) surv[wcnt[f * KNB_WARPS + warp] + __popc(bal[f] & ((1u << lane) - 1u))] = f * KNB_NT + tid;
    __syncthreads();
    const int ns = wcnt[MTI_F * KNB_WARPS];

    // ---- survivors: NT per round, one per thread
    for (int base = 0; base < ns; base += KNB_NT) {
      for (int i = tid; i < KNB_WARPS * k; i += KNB_NT) { mto[i] = 0u; mfrom[i] = 0u; }
      __syncthreads();
      const int si = base + tid;
      int to = -1, from = -1;
      if (si < ns) {
        const long long row = row0 + surv[si];
        const int orig = a.assign[row];
        double u = a.upper[row];
        const bool tg = a.tight[row] != 0;
        double x[DP];
        const double* xp = a.X + row * d;
        if (even) {
#pragma unroll
          for (int q = 0; q < DP / 2; ++q) {
            if (2 * q < d) {
              const double2 v = *reinterpret_cast<const double2*>(xp + 2 * q);
              x[2 * q] = v.x;
              x[2 * q + 1] = v.y;
            } else {
              x[2 * q] = 0.0;
              x[2 * q + 1] = 0.0;
            }
          }
        } else {
#pragma unroll
          for (int e = 0; e < DP; ++e) x[e] = e < d ? xp[e] : 0.0;
        }
        const double stale = u;
        if (!tg) {
          u = sqrt(exact_sq<DP>(x, C + orig * DP, d));
          ++computed;
        }
        int cur = orig;
        double u2lo = u * u * (1.0 - 8.9e-16), u2hi = u * u * (1.0 + 8.9e-16);
        for (int j = 0; j < k; ++j) {
          if (j == cur || j == orig) continue;
          const double gap = half[cur * k + j];
          if (u <= gap) {
            if (stale <= gap) ++pstale; else ++ptight;
            continue;
          }
          const double s2 = exact_sq<DP>(x, C + j * DP, d);
          ++computed;
          bool less = s2 < u2lo;
          if (!less && !(s2 > u2hi)) less = sqrt(s2) < u;
          if (less) {
            cur = j;
            u = sqrt(s2);
            u2lo = u * u * (1.0 - 8.9e-16);
            u2hi = u * u * (1.0 + 8.9e-16);
          }
        }
        a.upper[row] = u;
        if (!tg) a.tight[row] = 1;
        if (cur != orig) {
          a.assign[row] = cur;
          ++reassigned;
          to = cur;
          from = orig;
#pragma unroll
          for (int e = 0; e < DP; ++e) mvx[tid * (DP + 1) + e] = x[e];
          mvsq[tid] = exact_sq<DP>(x, Zero{}, d);
        }
      }
      {
        const unsigned pt = __match_any_sync(0xffffffffu, to);
        if (to >= 0 && lane == __ffs(pt) - 1) mto[warp * k + to] = pt;
        const unsigned pf = __match_any_sync(0xffffffffu, from);
        if (from >= 0 && lane == __ffs(pf) - 1) mfrom[warp * k + from] = pf;
      }
      __syncthreads();
      {
        constexpr int NG = KNB_NT / DP;
        const int e = tid % DP, g = tid / DP;
        if (e < d) {
          for (int j = g; j < k; j += NG) {
            double sa = 0.0, ss = 0.0, ca = 0.0, qa = 0.0, qs = 0.0;
            bool any = false;
            for (int w = 0; w < KNB_WARPS; ++w) {
              unsigned m = mto[w * k + j];
              if (m) any = true;
              if (e == 0) ca += __popc(m);
              while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                sa += mvx[(w * 32 + l) * (DP + 1) + e];
                if (e == 0) qa += mvsq[w * 32 + l];
              }
            }
            for (int w = 0; w < KNB_WARPS; ++w) {
              unsigned m = mfrom[w * k + j];
              if (m) any = true;
              if (e == 0) ca -= __popc(m);
              while (m) {
                const int l = __ffs(m) - 1;
                m &= m - 1;
                ss += mvx[(w * 32 + l) * (DP + 1) + e];
                if (e == 0) qs += mvsq[w * 32 + l];
              }
            }
            if (any) {
              acc[j * DP + e] = (acc[j * DP + e] + sa) - ss;
              if (e == 0) { cnt[j] += ca; sqa[j] = (sqa[j] + qa) - qs; }
            }
          }
        }
      }
      __syncthreads();
    }
    __syncthreads();
  }

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
  const long long v0 = warp_sum_ll(reassigned), v1 = warp_sum_ll(computed), v2 = warp_sum_ll(skips),
                  v3 = warp_sum_ll(pstale), v4 = warp_sum_ll(ptight);
  __syncthreads();
  if (lane == 0) {
    red[warp * 8 + 0] = (double)v0;
    red[warp * 8 + 1] = (double)v1;
    red[warp * 8 + 2] = (double)v2;
    red[warp * 8 + 3] = (double)v3;
    red[warp * 8 + 4] = (double)v4;
  }
  __syncthreads();
  if (tid == 0) {
    double t[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < KNB_WARPS; ++w)
      for (int i = 0; i < 5; ++i) t[i] += red[w * 8 + i];
    double* sc = out + (long long)k * d + 2LL * k;
    for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
    sc[S_REASSIGNED] = t[0];
    sc[S_COMPUTED] = t[1];
    sc[S_SKIPS] = t[2];
    sc[S_PSTALE] = t[3];
    sc[S_PTIGHT] = t[4];
  }
}


// Generic path (d > 64 or large k): same semantics, points/centroids through
// L1/L2, CTA partial in global memory with one owner thread per (cluster, dim).
__global__ void __launch_bounds__(KNB_NT) mti_generic_kernel(const MtiArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* mto = reinterpret_cast<uint32_t*>(smem);
  uint32_t* mfrom = mto + KNB_WARPS * k;
  double* mvsq = reinterpret_cast<double*>(smem + al((size_t)2 * KNB_WARPS * k * 4, 16));
  long long* mrow = reinterpret_cast<long long*>(mvsq + KNB_NT);
  double* red = reinterpret_cast<double*>(mrow + KNB_NT);
  const long long Lg = acc_len(k, d);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  for (long long i = tid; i < Lg; i += KNB_NT) out[i] = 0.0;
  long long skips = 0, computed = 0, pstale = 0, ptight = 0, reassigned = 0;
  const long long ntiles = (a.n + KNB_NT - 1) / KNB_NT;
  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int i = tid; i < KNB_WARPS * k; i += KNB_NT) { mto[i] = 0u; mfrom[i] = 0u; }
    __syncthreads();
    const long long row = tile * KNB_NT + tid;
    int to = -1, from = -1;
    if (row < a.n) {
      const int orig = a.assign[row];
      double u = a.upper[row];
      bool tg = a.tight[row] != 0;
      const double dr = a.drift[orig];
      if (dr != 0.0) { u = u + dr; tg = false; a.upper[row] = u; a.tight[row] = 0; }
      if (u <= a.half_min[orig]) {
        ++skips;
      } else {
        const double* x = a.X + row * d;
        const double stale = u;
        if (!tg) { u = sqrt(exact_sq_rt(x, a.means + (long long)orig * d, d)); ++computed; }
        int cur = orig;
        double u2lo = u * u * (1.0 - 8.9e-16), u2hi = u * u * (1.0 + 8.9e-16);
        for (int j = 0; j < k; ++j) {
          if (j == cur || j == orig) continue;
          const double gap = a.half[(long long)cur * k + j];
          if (u <= gap) { if (stale <= gap) ++pstale; else ++ptight; continue; }
          const double s2 = exact_sq_rt(x, a.means + (long long)j * d, d);
          ++computed;
          bool less = s2 < u2lo;
          if (!less && !(s2 > u2hi)) less = sqrt(s2) < u;
          if (less) { cur = j; u = sqrt(s2); u2lo = u * u * (1.0 - 8.9e-16); u2hi = u * u * (1.0 + 8.9e-16); }
        }
        a.upper[row] = u;
        a.tight[row] = 1;
        if (cur != orig) {
          a.assign[row] = cur;
          ++reassigned;
          to = cur;
          from = orig;
          mvsq[tid] = exact_self_rt(x, d);
        }
      }
    }
    mrow[tid] = row;
    {
      const unsigned pt = __match_any_sync(0xffffffffu, to);
      if (to >= 0 && lane == __ffs(pt) - 1) mto[warp * k + to] = pt;
      const unsigned pf = __match_any_sync(0xffffffffu, from);
      if (from >= 0 && lane == __ffs(pf) - 1) mfrom[warp * k + from] = pf;
    }
    __syncthreads();
    for (long long pi = tid; pi < (long long)k * d; pi += KNB_NT) {
      const int j = (int)(pi / d), e = (int)(pi - (long long)j * d);
      double sa = 0.0, ss = 0.0, ca = 0.0, qa = 0.0, qs = 0.0;
      bool any = false;
      for (int w = 0; w < KNB_WARPS; ++w) {
        unsigned m = mto[w * k + j];
        if (m) any = true;
        if (e == 0) ca += __popc(m);
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          sa += a.X[mrow[w * 32 + l] * d + e];
          if (e == 0) qa += mvsq[w * 32 + l];
        }
      }
      for (int w = 0; w < KNB_WARPS; ++w) {
        unsigned m = mfrom[w * k + j];
        if (m) any = true;
        if (e == 0) ca -= __popc(m);
        while (m) {
          const int l = __ffs(m) - 1;
          m &= m - 1;
          ss += a.X[mrow[w * 32 + l] * d + e];
          if (e == 0) qs += mvsq[w * 32 + l];
        }
      }
      if (any) {
        out[pi] = (out[pi] + sa) - ss;
        if (e == 0) {
          out[(long long)k * d + j] += ca;
          out[(long long)k * d + k + j] = (out[(long long)k * d + k + j] + qa) - qs;
        }
      }
    }
    __syncthreads();
  }
  const long long v0 = warp_sum_ll(reassigned), v1 = warp_sum_ll(computed), v2 = warp_sum_ll(skips),
                  v3 = warp_sum_ll(pstale), v4 = warp_sum_ll(ptight);
  if (lane == 0) {
    red[warp * 8 + 0] = (double)v0;
    red[warp * 8 + 1] = (double)v1;
    red[warp * 8 + 2] = (double)v2;
    red[warp * 8 + 3] = (double)v3;
    red[warp * 8 + 4] = (double)v4;
  }
  __syncthreads();
  if (tid == 0) {
    double t[5] = {0, 0, 0, 0, 0};
    for (int w = 0; w < KNB_WARPS; ++w)
      for (int i = 0; i < 5; ++i) t[i] += red[w * 8 + i];
    double* sc = out + (long long)k * d + 2LL * k;
    sc[S_REASSIGNED] = t[0];
    sc[S_COMPUTED] = t[1];
    sc[S_SKIPS] = t[2];
    sc[S_PSTALE] = t[3];
    sc[S_PTIGHT] = t[4];
  }
}

}  // namespace

size_t mti_tile_smem(int DP, int k, int half_in_smem) { return MtiSmem(DP, k, half_in_smem).total; }

int mti_tile_grid(int DP, int k, int half_in_smem, int sms) {
  const size_t sm = mti_tile_smem(DP, k, half_in_smem);
  int per = (int)((227u * 1024u) / (sm + 1024));
  if (per < 1) per = 1;
  if (per > 4) per = 4;
  return sms * per;
}

template <int DP>
static cudaError_t launch_mti_dp(const MtiArgs& a, int grid, cudaStream_t s) {
  const size_t sm = mti_tile_smem(DP, a.k, a.half_in_smem);
  cudaError_t e = cudaFuncSetAttribute(mti_tile_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  mti_tile_kernel<DP><<<grid, KNB_NT, sm, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_mti(const MtiArgs& a, int DP, int grid, cudaStream_t s) {
  if (DP == 0) {
    const size_t sm = al((size_t)2 * KNB_WARPS * a.k * 4, 16) + (size_t)KNB_NT * 16 + KNB_WARPS * 64;
    cudaError_t e = cudaFuncSetAttribute(mti_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    mti_generic_kernel<<<grid, KNB_NT, sm, s>>>(a);
    return cudaGetLastError();
  }
  switch (DP) {
    case 2: return launch_mti_dp<2>(a, grid, s);
    case 4: return launch_mti_dp<4>(a, grid, s);
    case 8: return launch_mti_dp<8>(a, grid, s);
    case 16: return launch_mti_dp<16>(a, grid, s);
    case 32: return launch_mti_dp<32>(a, grid, s);
    case 64: return launch_mti_dp<64>(a, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace knb
