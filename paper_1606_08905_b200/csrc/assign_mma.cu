// K1 on the FP64 tensor cores: dense point -> centroid assignment fused with the
// centroid-sum accumulation, for d <= 64 and centroids that fit shared memory.
//
// Replaces numakmeans engine._task_full (engine.py:285-319) and the streaming
// nearest-centroid scan it calls (distance.py:94-116).
//
// Why DMMA: the contraction s = X C^T is a small dense GEMM per tile.  On B200 the
// FP64 tensor path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) and the vector FP64 FMA
// pipe have the same peak (measured 18.5 vs 18.2 T FMA/s, tools/microbench.cu), but a
// DMMA does 256 FMAs from register fragments, whereas vector DFMA needs a centroid
// operand per FMA from a warp-uniform LDS (measured 0.45 LDS.128 / clk / SM), which
// caps the vector kernel near a quarter of peak.  tcgen05 has no f64 kind.
//
// Tile: a CTA of 8 warps owns 256 rows; each warp computes a 32-row x 32-centroid
// block as 4 x 4 DMMA tiles over d/4 k-steps.  Point fragments come from the
// swizzled TMA tile (conflict-free), centroid fragments from a shared-memory copy
// pre-permuted into fragment order, and each accumulator starts at -||c_j||^2 / 2,
// so the tensor core produces s_ij = x_i.c_j - ||c_j||^2/2 directly (argmax s ==
// argmin distance).  The epilogue folds 8 columns per lane into a running best /
// argbest plus the near-tie flag (integer ops only), then combines the 4 lanes of
// each row quad with shuffles.  A point is certified when no other centroid scored
// within tol = (8d+32) 2^-53 (||x||^2 + max||c||^2) of the winner -- a bound on the
// rounding of both this contraction (any summation order) and the reference's
// subtract-square recipe -- so the certified winner is exactly the reference's
// argmin; uncertified points (near ties) are re-ranked with the exact recipe.  The
// winner's distance is recomputed with the exact recipe (bit-identical to the
// oracle on the reference's BLAS tree).
//
// Accumulation: per 32-row group one member mask per cluster (match.any), then
// thread (dim e, group g) owns clusters j = g mod NG and adds members' values in
// row order into CTA-private shared-memory sums -- deterministic, no atomics.  One
// partial per CTA leaves for the fixed-order reduction (update.cu).
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

constexpr int MR = KNB_NT;  // rows per tile: 32 per warp

__host__ __device__ inline size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct MmaSmem {
  size_t xb0, xb1, bf, crow, chn, acc, cnt, sq, xsq, masks, mbar, red, total;
  __host__ __device__ MmaSmem(int DP, int k) {
    const int kp = (k + 7) & ~7;
    const size_t tile = (size_t)MR * DP * 8;
    size_t o = 0;
    xb0 = o;  o += tile;
    xb1 = o;  o += tile;
    bf = o;   o += (size_t)kp * DP * 8;
    crow = o; o += (size_t)kp * DP * 8;
    chn = o;  o += (size_t)kp * 8;
    acc = o;  o += (size_t)k * DP * 8;
    cnt = o;  o += (size_t)k * 8;
    sq = o;   o += (size_t)k * 8;
    xsq = o;  o += (size_t)MR * 8;
    masks = o; o += (size_t)(MR / 32) * k * 4;
    o = al(o, 16);
    mbar = o; o += 16;
    red = o;  o += KNB_WARPS * 4 * 8;
    total = o;
  }
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void score_update(double& best, int& bid, bool& flag, double s, int j, int tolhi) {
  const double diff = __dsub_rn(s, best);
  const int h = __double2hiint(diff);
  const bool better = h > 0;
  const bool near = (h & 0x7fffffff) <= tolhi;
  flag = near | (flag & !better);
  best = better ? s : best;
  bid = better ? j : bid;
}

// Merge a disjoint partial (best, id, flag) from another lane of the same row.
__device__ __forceinline__ void combine(double& best, int& bid, bool& flag, int tolhi, int lanemask) {
  const double ob = __shfl_xor_sync(0xffffffffu, best, lanemask);
  const int oi = __shfl_xor_sync(0xffffffffu, bid, lanemask);
  const bool of = __shfl_xor_sync(0xffffffffu, (int)flag, lanemask) != 0;
  const double diff = __dsub_rn(ob, best);
  const int h = __double2hiint(diff);
  const bool near = (h & 0x7fffffff) <= tolhi;
  const bool other = h > 0 || (diff == 0.0 && oi < bid);
  flag = near | (other ? of : flag);
  best = other ? ob : best;
  bid = other ? oi : bid;
}

template <int DP>
__device__ __forceinline__ void issue_tile(const CUtensorMap* tmap, uint64_t* bar, unsigned char* dst,
                                           long long tile, const DenseArgs& a, bool tma) {
  using TL = TileLayout<DP>;
  const long long row0 = tile * MR;
  if (tma) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(bar, TL::tile_bytes(MR));
#pragma unroll
      for (int p = 0; p < TL::NPANEL; ++p) tma_load_2d(dst + p * MR * TL::RB, tmap, bar, p * TL::PW, (int)row0);
    }
  } else {
    const int rows = (int)(a.n - row0 < MR ? a.n - row0 : MR);
    const int d = a.d;
    const double* src = a.X + row0 * d;
    if (((d & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0)) {
      const int hd = d >> 1;
      for (int i = threadIdx.x; i < rows * hd; i += KNB_NT) {
        const int r = i / hd, q = i - r * hd;
        cp_async16(dst + TL::chunk_off(r, q, MR), src + 2LL * i);
      }
    } else {
      for (int i = threadIdx.x; i < rows * d; i += KNB_NT) {
        const int r = i / d, e = i - r * d;
        cp_async8(dst + TL::elem_off(r, e, MR), src + i);
      }
    }
    cp_async_commit();
  }
}

template <int DP>
__global__ void __launch_bounds__(KNB_NT, 1)
    dense_mma_kernel(const __grid_constant__ CUtensorMap tmap, const DenseArgs a) {
  using TL = TileLayout<DP>;
  constexpr int KS = DP / 4;            // k-steps of 4 dims
  constexpr bool ACACHE = DP <= 32;     // point fragments stay in registers
  constexpr int RG = MR / 32;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;

  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int kp = (k + 7) & ~7, ntile8 = kp >> 3;
  const MmaSmem L(DP, k);
  unsigned char* const xb0 = smem + L.xb0;
  unsigned char* const xb1 = smem + L.xb1;
  double* bf = reinterpret_cast<double*>(smem + L.bf);
  double* crow = reinterpret_cast<double*>(smem + L.crow);
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

  // centroids: row layout (exact recipe) and DMMA B-fragment order
  //   bf[((q*KS + s)*32 + l)] = C[q*8 + l/4][s*4 + l%4]
  for (int i = tid; i < kp * DP; i += KNB_NT) {
    const int j = i / DP, e = i - j * DP;
    crow[i] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
  }
  for (int i = tid; i < kp * DP; i += KNB_NT) {
    const int l = i & 31, qs = i >> 5, q = qs / KS, s = qs - q * KS;
    const int j = q * 8 + (l >> 2), e = s * 4 + (l & 3);
    bf[i] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
  }
  for (int j = tid; j < kp; j += KNB_NT) chn[j] = j < k ? a.chn[j] : -CUDART_INF;
  for (int i = tid; i < k * DP; i += KNB_NT) acc[i] = 0.0;
  for (int j = tid; j < k; j += KNB_NT) { cnt[j] = 0.0; sqa[j] = 0.0; }
  if (!tma && d < DP) {  // cp.async never writes the padded columns: zero them once
    for (int b = 0; b < 2; ++b)
      for (int i = tid; i < MR * DP; i += KNB_NT) {
        const int r = i / DP, e = i - r * DP;
        if (e >= d) *reinterpret_cast<double*>((b ? xb1 : xb0) + TL::elem_off(r, e, MR)) = 0.0;
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
  const long long ntiles = (a.n + MR - 1) / MR;
  long long reassigned = 0, rows_done = 0;
  double wcss = 0.0;
  uint32_t ph0 = 0u, ph1 = 0u;
  int buf = 0;
  if ((long long)blockIdx.x < ntiles) issue_tile<DP>(&tmap, &bar[0], xb0, blockIdx.x, a, tma);

  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long long next = tile + gridDim.x;
    if (next < ntiles) issue_tile<DP>(&tmap, buf ? &bar[0] : &bar[1], buf ? xb0 : xb1, next, a, tma);
    for (int i = tid; i < RG * k; i += KNB_NT) masks[i] = 0u;
    if (tma) {
      if (buf) { mbar_wait(&bar[1], ph1); ph1 ^= 1u; } else { mbar_wait(&bar[0], ph0); ph0 ^= 1u; }
    } else {
      if (next < ntiles) cp_async_wait_1(); else cp_async_wait_all();
    }
    __syncthreads();
    const unsigned char* tb = buf ? xb1 : xb0;
    const long long row0 = tile * MR;
    // this lane's own point after the quad combine: row (t4 * 8 + g) of the warp's 32
    const int my_r = warp * 32 + t4 * 8 + g;
    const bool valid = row0 + my_r < a.n;
    int my_id = 0;

    if (!labels) {
      // ---- point fragments: A[m][kk] = x[warp*32 + pg*8 + g][s*4 + t4]
      double afr[4][ACACHE ? KS : 1];
      double xn2[4];
#pragma unroll
      for (int pg = 0; pg < 4; ++pg) {
        const int r = warp * 32 + pg * 8 + g;
        double s2 = 0.0;
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          const double v = *reinterpret_cast<const double*>(tb + TL::elem_off(r, s * 4 + t4, MR));
          if constexpr (ACACHE) afr[pg][s] = v;
          s2 = fma(v, v, s2);
        }
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
        xn2[pg] = s2;
      }
      double best[4];
      int bid[4], tolhi[4];
      bool flag[4];
#pragma unroll
      for (int pg = 0; pg < 4; ++pg) {
        tolhi[pg] = __double2hiint(tolk * (xn2[pg] + cmax2));
        best[pg] = -CUDART_INF;
        bid[pg] = 0;
        flag[pg] = false;
      }
      // ---- centroid blocks of up to 32 (4 n-tiles of 8)
#pragma unroll 1
      for (int cb = 0; cb < ntile8; cb += 4) {
        const int nq = ntile8 - cb < 4 ? ntile8 - cb : 4;
        double c[4][4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double2 h = q < nq ? *reinterpret_cast<const double2*>(chn + (cb + q) * 8 + 2 * t4)
                                   : make_double2(0.0, 0.0);
#pragma unroll
          for (int pg = 0; pg < 4; ++pg) { c[pg][q][0] = h.x; c[pg][q][1] = h.y; }
        }
#pragma unroll
        for (int s = 0; s < KS; ++s) {
          double av[4];
#pragma unroll
          for (int pg = 0; pg < 4; ++pg) {
            if constexpr (ACACHE) av[pg] = afr[pg][s];
            else av[pg] = *reinterpret_cast<const double*>(tb + TL::elem_off(warp * 32 + pg * 8 + g, s * 4 + t4, MR));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (q < nq) {
              const double bv = bf[(((cb + q) * KS + s) << 5) + lane];
#pragma unroll
              for (int pg = 0; pg < 4; ++pg) dmma(c[pg][q], av[pg], bv);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (q < nq) {
            const int j0 = (cb + q) * 8 + 2 * t4;
#pragma unroll
            for (int pg = 0; pg < 4; ++pg) {
              score_update(best[pg], bid[pg], flag[pg], c[pg][q][0], j0, tolhi[pg]);
              score_update(best[pg], bid[pg], flag[pg], c[pg][q][1], j0 + 1, tolhi[pg]);
            }
          }
        }
      }
      // ---- combine the 4 lanes of each row quad
#pragma unroll
      for (int pg = 0; pg < 4; ++pg) {
        combine(best[pg], bid[pg], flag[pg], tolhi[pg], 1);
        combine(best[pg], bid[pg], flag[pg], tolhi[pg], 2);
      }
      // lane takes point group pg == t4 (row t4*8 + g)
      int id = bid[0];
      bool fl = flag[0];
#pragma unroll
      for (int pg = 1; pg < 4; ++pg)
        if (t4 == pg) { id = bid[pg]; fl = flag[pg]; }
      // ---- exact recipe on the lane's own point
      double x[DP];
#pragma unroll
      for (int q2 = 0; q2 < DP / 2; ++q2) {
        const double2 v = *reinterpret_cast<const double2*>(tb + TL::chunk_off(my_r, q2, MR));
        x[2 * q2] = v.x;
        x[2 * q2 + 1] = v.y;
      }
      double nd;
      if (fl) {  // near tie: exact re-rank over every centroid, ascending, strict <
        double bd = CUDART_INF;
        int bi = 0;
        for (int j = 0; j < k; ++j) {
          const double dj = sqrt(exact_sq<DP>(x, crow + j * DP, d));
          if (dj < bd) { bd = dj; bi = j; }
        }
        id = bi;
        nd = bd;
      } else {
        nd = sqrt(exact_sq<DP>(x, crow + id * DP, d));
      }
      my_id = id;
      if (valid) {
        const long long row = row0 + my_r;
        const int old = a.assign[row];
        a.assign[row] = id;
        reassigned += (old != id);
        if (a.mti_seed) {
          a.upper[row] = nd;
          a.tight[row] = 1;
          xsq[my_r] = exact_sq<DP>(x, Zero{}, d);
        } else {
          wcss += nd * nd;
        }
        ++rows_done;
      }
    } else if (valid) {
      my_id = a.assign[row0 + my_r];
      ++rows_done;
    }
    // ---- member masks in natural row order: bit p <-> row warp*32 + p
    {
      const int src = ((lane & 7) << 2) | (lane >> 3);  // lane owning row offset `lane`
      const int idn = __shfl_sync(0xffffffffu, valid ? my_id : -1, src);
      const unsigned peers = __match_any_sync(0xffffffffu, idn);
      if (idn >= 0 && lane == __ffs(peers) - 1) masks[warp * k + idn] = peers;
    }
    __syncthreads();
    {  // deterministic segmented accumulation, members in row order
      constexpr int NG = KNB_NT / DP;
      const int e = tid % DP, gg = tid / DP;
      if (e < d) {
        for (int j = gg; j < k; j += NG) {
          double s = 0.0, cc = 0.0, q = 0.0;
#pragma unroll
          for (int rg = 0; rg < RG; ++rg) {
            unsigned m = masks[rg * k + j];
            if (e == 0) cc += __popc(m);
            while (m) {
              const int l = __ffs(m) - 1;
              m &= m - 1;
              const int r = rg * 32 + l;
              s += *reinterpret_cast<const double*>(tb + TL::elem_off(r, e, MR));
              if (e == 0 && a.mti_seed) q += xsq[r];
            }
          }
          acc[j * DP + e] += s;
          if (e == 0) { cnt[j] += cc; sqa[j] += q; }
        }
      }
    }
    __syncthreads();  // tile buffer and masks free for reuse
    buf ^= 1;
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

template <int DP>
cudaError_t launch_mma_dp(const CUtensorMap* tmap, const DenseArgs& a, int grid, cudaStream_t s) {
  const MmaSmem L(DP, a.k);
  cudaError_t e = cudaFuncSetAttribute(dense_mma_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  dense_mma_kernel<DP><<<grid, KNB_NT, L.total, s>>>(*tmap, a);
  return cudaGetLastError();
}

}  // namespace

int dense_mma_dp(int d) {
  if (d <= 4) return 4;
  if (d <= 8) return 8;
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  if (d <= 64) return 64;
  return 0;
}

size_t dense_mma_smem(int DP, int k) { return MmaSmem(DP, k).total; }

int dense_mma_rows() { return MR; }

cudaError_t launch_dense_mma(const CUtensorMap* tmap, const DenseArgs& a, int DP, int grid, cudaStream_t s) {
  switch (DP) {
    case 4: return launch_mma_dp<4>(tmap, a, grid, s);
    case 8: return launch_mma_dp<8>(tmap, a, grid, s);
    case 16: return launch_mma_dp<16>(tmap, a, grid, s);
    case 32: return launch_mma_dp<32>(tmap, a, grid, s);
    case 64: return launch_mma_dp<64>(tmap, a, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace knb
