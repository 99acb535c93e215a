// K1 on the FP64 tensor cores: dense point -> centroid assignment fused with the
// centroid-sum accumulation, for d <= 64 and centroids that fit shared memory.
//
// Replaces numakmeans engine._task_full (engine.py:285-319) and the streaming
// nearest-centroid scan it calls (distance.py:94-116).
//
// Why DMMA: the contraction s = X C^T is a small dense GEMM per block of rows.  On
// B200 the FP64 tensor path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) and the vector
// FP64 FMA pipe have the same peak (measured 18.5 vs 18.2 T FMA/s,
// tools/microbench.cu), but a DMMA does 256 FMAs from register fragments, whereas
// vector DFMA needs a warp-uniform centroid operand per FMA from shared memory
// (measured 0.45 LDS.128 / clk / SM), which caps it near a quarter of peak.
// tcgen05 has no f64 kind.
//
// Warp-independent pipelines: every warp owns a strided sequence of 32-row blocks
// and streams them through its own NS-stage buffer with its own 2-D TMA loads
// (hardware-swizzled 32 x 16-double boxes) and mbarriers, so warps never wait for
// each other inside the main loop and one warp's epilogue overlaps another's DMMA.
//
// Per block: a warp computes 32 rows x up to 32 centroids per step as 4 x 4 DMMA
// tiles over d/4 k-steps.  Centroid fragments come from a shared-memory copy
// pre-permuted into fragment order and each accumulator starts at -||c_j||^2 / 2,
// so the tensor core emits s_ij = x_i.c_j - ||c_j||^2/2 (argmax s == argmin
// distance).  The epilogue keeps a running best / argbest and a near-tie flag
// (integer ops), then merges the 4 lanes of each row quad.  A point is certified
// when no other centroid scored within tol = (8d+32) 2^-53 (||x||^2 + max||c||^2)
// of the winner -- a bound on the rounding of this contraction (any order) and of
// the reference's subtract-square recipe -- so the certified winner is exactly the
// reference's argmin; near ties are re-ranked with the exact recipe, and the
// winner's distance is recomputed with it (bit-identical to the oracle on the
// reference's BLAS tree).
//
// Accumulation is warp-local and deterministic: the warp walks the block's rows in
// row order with lanes = dims (accumulate_in_row_order) and adds each into its
// private shared-memory sums -- every row on the first pass, only the moved rows'
// signed deltas afterwards.  At the end the CTA adds its warps' sums in warp order
// into one partial for the fixed-order reduction (update.cu).
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"
#include "mma_common.cuh"

namespace knb {

namespace {

__host__ __device__ inline size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

// W12: the twelve-warp budget (one stage per warp, no fragment-ordered copy)
__host__ __device__ constexpr int stages_for(int DP, bool w12 = false) { return w12 ? 1 : DP <= 8 ? 4 : 2; }

// shared memory: [centroids: bf, crow, chn] [per warp: NS stages, mbar, acc, cnt, sq]
struct WarpSmem {
  size_t bf, crow, chn, hmin, drift, warp0, stage_bytes, mbar_off, acc_off, cnt_off, sq_off, per_warp, red, total;
  __host__ __device__ WarpSmem(int DP, int k, int d, int W, bool w12 = false) {
    const int kp = (k + 7) & ~7;
    const int NS = stages_for(DP, w12);
    size_t o = 0;
    bf = o;   o += w12 ? 0 : (size_t)kp * DP * 8;
    crow = o; o += (size_t)kp * (DP + 2) * 8;
    chn = o;  o += (size_t)kp * 8;
    hmin = o; o += (size_t)k * 8;
    drift = o; o += (size_t)k * 8;
    red = o;  o += 16 * 8 * 8;
    o = al(o, 1024);
    warp0 = o;
    stage_bytes = (size_t)BR * DP * 8;              // multiple of 1024 for DP >= 4
    size_t w = (size_t)NS * stage_bytes;
    mbar_off = w; w += (size_t)NS * 8;
    w = al(w, 16);
    acc_off = w;  w += (size_t)k * d * 8;
    cnt_off = w;  w += (size_t)k * 8;
    sq_off = w;   w += (size_t)k * 8;
    per_warp = al(w, 1024);
    total = warp0 + (size_t)W * per_warp;
  }
};

template <int DP>
__device__ __forceinline__ void load_block(const CUtensorMap* tmap, uint64_t* bar, unsigned char* dst, long long blk,
                                           const DenseArgs& a, bool tma, int lane) {
  using TL = TileLayout<DP>;
  const long long row0 = blk * BR;
  if (tma) {
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, TL::tile_bytes(BR));
#pragma unroll
      for (int p = 0; p < TL::NPANEL; ++p) tma_load_2d(dst + p * BR * TL::RB, tmap, bar, p * TL::PW, (int)row0);
    }
  } else {
    const int rows = (int)(a.n - row0 < BR ? a.n - row0 : BR);
    const int d = a.d;
    const double* src = a.X + row0 * d;
    if (((d & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0)) {
      const int hd = d >> 1;
      for (int i = lane; i < rows * hd; i += 32) {
        const int r = i / hd, q = i - r * hd;
        cp_async16(dst + TL::chunk_off(r, q, BR), src + 2LL * i);
      }
    } else {
      for (int i = lane; i < rows * d; i += 32) {
        const int r = i / d, e = i - r * d;
        cp_async8(dst + TL::elem_off(r, e, BR), src + i);
      }
    }
    cp_async_commit();
  }
}

#ifndef KNB_DENSE_2CTA_DP
#define KNB_DENSE_2CTA_DP 8
#endif

// SMALLK (k <= 16): the scorer's one-step form; with narrow rows it leaves room for
// two CTAs per SM (<= 128 registers, no spills)
// W12 (d == DP in {16, 32}, k > 16): up to twelve warps per SM at <= 168 registers --
// one TMA stage per warp (the next block is prefetched into L2 while the current one is
// scored), B fragments from the row-major centroid copy, exact distances streamed
// through the tree; the pass is bound by warp-level latency (profiles/README.md)
#ifndef KNB_DENSE_W12_THREADS
#define KNB_DENSE_W12_THREADS 384
#endif
// ONE (k <= 8): the scorer's single-tile form (half the DMMAs of a padded tile pair)
#ifndef KNB_DENSE_DIRECT
#define KNB_DENSE_DIRECT 1
#endif
template <int DP, bool SMALLK, bool W12 = false, bool ONE = false>
__global__ void __launch_bounds__(W12 ? KNB_DENSE_W12_THREADS : KNB_NT, (SMALLK && DP <= KNB_DENSE_2CTA_DP) ? 2 : 1)
    dense_mma_kernel(const __grid_constant__ CUtensorMap tmap, const DenseArgs a) {
  using TL = TileLayout<DP>;
  constexpr int KS = DP / 4;         // k-steps of 4 dims
  constexpr int NS = stages_for(DP, W12);
  // narrow rows, few centroids (config 3's shape): rows ranked by the exact recipe directly
  constexpr bool DIRECT = KNB_DENSE_DIRECT && SMALLK && !W12 && DP <= 8;
  extern __shared__ __align__(1024) unsigned char smem[];
  pdl_enter();
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  if (a.gate && a.ctrl->mti_choice != 1) return;  // the compacted MTI kernel runs this iteration

  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = blockDim.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int kp = (k + 7) & ~7, ntile8 = kp >> 3;
  const WarpSmem L(DP, k, d, W, W12);
  double* hmin_s = reinterpret_cast<double*>(smem + L.hmin);
  double* drift_s = reinterpret_cast<double*>(smem + L.drift);
  double* bf = reinterpret_cast<double*>(smem + L.bf);
  double* crow = reinterpret_cast<double*>(smem + L.crow);
  double* chn = reinterpret_cast<double*>(smem + L.chn);
  double* red = reinterpret_cast<double*>(smem + L.red);
  unsigned char* wbase = smem + L.warp0 + (size_t)warp * L.per_warp;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wbase + L.mbar_off);
  double* acc = reinterpret_cast<double*>(wbase + L.acc_off);
  double* cnt = reinterpret_cast<double*>(wbase + L.cnt_off);
  double* sqa = reinterpret_cast<double*>(wbase + L.sq_off);
  const bool tma = a.use_tma != 0;
  const bool labels = a.labels_only != 0;

  // centroids: row layout (exact recipe) and B-fragment order
  //   bf[((q*KS + s)*32 + l)] = C[q*8 + l/4][s*4 + l%4]
  for (int i = tid; i < kp * DP; i += blockDim.x) {
    const int j = i / DP, e = i - j * DP;
    crow[j * crow_stride<DP>() + e] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
    if constexpr (!W12) {
      const int l = i & 31, qs = i >> 5, q = qs / KS, s = qs - q * KS;
      const int jb = q * 8 + (l >> 2), eb = s * 4 + (l & 3);
      bf[i] = (jb < k && eb < d) ? a.means[(long long)jb * d + eb] : 0.0;
    }
  }
  for (int j = tid; j < kp; j += blockDim.x) chn[j] = j < k ? a.chn[j] : -CUDART_INF;
  if (a.mti_filter)
    for (int j = tid; j < k; j += blockDim.x) {
      hmin_s[j] = a.half_min[j];
      drift_s[j] = a.drift[j];
    }
  for (int i = lane; i < k * d; i += 32) acc[i] = 0.0;
  for (int j = lane; j < k; j += 32) { cnt[j] = 0.0; sqa[j] = 0.0; }
  if (!tma && d < DP) {  // cp.async never writes the padded columns: zero them once
    for (int s = 0; s < NS; ++s)
      for (int i = lane; i < BR * DP; i += 32) {
        const int r = i / DP, e = i - r * DP;
        if (e >= d) *reinterpret_cast<double*>(wbase + s * L.stage_bytes + TL::elem_off(r, e, BR)) = 0.0;
      }
  }
  if (lane == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
    fence_barrier_init();
    if (tma && warp == 0) prefetch_tmap(&tmap);
  }
  __syncthreads();

  const double cmax2 = a.ctrl->cmax2;
  const double tolk = (8.0 * d + 32.0) * 1.1102230246251565e-16;  // (8d+32) * 2^-53
  const long long nblk = (a.n + BR - 1) / BR;
  const long long gw = (long long)blockIdx.x * W + warp, TW = (long long)gridDim.x * W;
  long long reassigned = 0, rows_done = 0, skips = 0, computed = 0;
  double wcss = 0.0;

#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (gw + s * TW < nblk) load_block<DP>(&tmap, &bar[s], wbase + s * L.stage_bytes, gw + s * TW, a, tma, lane);

  // Per-row state (previous assignment, MTI bound) is prefetched one block ahead so
  // no block starts by waiting on a global load.
  // W12: lane r handles row r after the scorer (rows_to_lanes; measured: the eight-warp
  // forms do not gain from it -- c3's first pass 1.76 -> 1.83 ms)
  const int my_r0 = W12 ? lane : t4 * 8 + g;
  auto state_row = [&](long long b) -> long long {
    const long long r = b * BR + my_r0;
    return (b < nblk && r < a.n) ? r : 0;
  };
  int pf_old = a.assign[state_row(gw)];
  double pf_u = a.mti_filter ? a.upper[state_row(gw)] : 0.0;
  int it = 0;
  for (long long blk = gw; blk < nblk; blk += TW, ++it) {
    const int old_raw = pf_old;
    const double u_pre = pf_u;
    pf_old = a.assign[state_row(blk + TW)];
    if (a.mti_filter) pf_u = a.upper[state_row(blk + TW)];
    const int s = it % NS;
    unsigned char* tb = wbase + s * L.stage_bytes;
    if (tma) {
      if constexpr (W12) {  // one stage: the next block heads for L2 while this one is scored
        const long long pb = blk + TW;
        if (lane == 0 && pb < nblk) {
#pragma unroll
          for (int p = 0; p < TL::NPANEL; ++p) tma_prefetch_l2_2d(&tmap, p * TL::PW, (int)(pb * BR));
        }
      }
      mbar_wait(&bar[s], (uint32_t)((it / NS) & 1));
    } else {
      // groups complete in order: allow the NS-1 younger groups to stay in flight
      const long long left = (nblk - 1 - blk) / TW;  // blocks after this one
      if (left >= NS - 1) {
        if constexpr (NS == 4) asm volatile("cp.async.wait_group 3;" ::: "memory");
        else if constexpr (NS == 2) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else cp_async_wait_all();
      } else {
        cp_async_wait_all();
      }
      __syncwarp();
    }
    const long long row0 = blk * BR;
    const int my_r = my_r0;  // the row this lane finishes after the scorer
    const bool valid = row0 + my_r < a.n;
    const long long row = row0 + my_r;
    int id = 0;
    double my_sq = 0.0;
    int old = -1;
    if (a.mti_filter) {
      // block-dense MTI pass: bound inflation + clause 1 per row (pruning.py:152-160,
      // engine.py:327); survivors get the certified argmin, the exact-recipe bound and
      // tight = 1 (scan_block's outcome); skipped rows are left exactly as the
      // reference leaves them.  A block whose rows all skip costs no tensor work.
      const int aa = valid ? old_raw : 0;
      const double dr = drift_s[aa];
      const double u = u_pre + dr;  // u + 0.0 == u
      const bool live = valid && !(u <= hmin_s[aa]);
      if (valid && !live && dr != 0.0) {  // a skipped row keeps the inflated bound;
        a.upper[row] = u;                 // survivors' bounds are rewritten below
        a.tight[row] = 0;
      }
      skips += (valid && !live) ? 1 : 0;
      const unsigned lmask = __ballot_sync(0xffffffffu, live);
      if (lmask) {
        int nid;
        double nd, sq = 0.0;
        if constexpr (DIRECT) {
          nd = direct_winner<DP, TL>(tb, my_r, crow, k, d, live ? aa : 0, nid);
          if (live && nid != aa) sq = row_self_sq<DP>(tb, my_r, d);
        } else {
        Scored sc = score_block<DP, SMALLK, W12, W12, false, TL, ONE>(tb, W12 ? crow : bf, chn, ntile8, tolk, cmax2,
                                                                     lane);
        if constexpr (W12) sc = rows_to_lanes(sc, lane);
        nid = sc.id;
        if constexpr (W12) {
          nd = exact_winner_stream<DP>(tb, my_r, crow, k, sc.flag, nid, live ? aa : -1);
          if (live && nid != aa) sq = exact_sq_stream<DP, true>(tb, my_r, nullptr);
        } else {
          nd = exact_winner<DP>(tb, my_r, crow, k, d, sc.flag, nid, nullptr, live ? aa : -1);
          if (live && nid != aa) sq = row_self_sq<DP>(tb, my_r, d);
        }
        }
        if (live) {
          a.upper[row] = nd;
          a.tight[row] = 1;
          if (nid != aa) {
            a.assign[row] = nid;
            ++reassigned;
          }
        }
        if (lane == 0) computed += (long long)__popc(lmask) * k;
        accumulate_in_row_order<DP, TL, W12>(row_mask(live && nid != aa, my_r), nid, aa, sq, tb, acc, cnt, sqa, d,
                                             lane);
      }
    } else if (!labels) {
      double nd2;
      if constexpr (DIRECT) {
        // narrow rows, few centroids: the k exact distances directly (direct_winner)
        const double nd = direct_winner<DP, TL, false>(tb, my_r, crow, k, d, -1, id, a.mti_seed ? &my_sq : nullptr);
        nd2 = nd * nd;
        if (a.mti_seed && valid) {
          a.upper[row] = nd;
          a.tight[row] = 1;
        }
      } else {
      Scored sc = score_block<DP, SMALLK, W12, W12, false, TL, ONE>(tb, W12 ? crow : bf, chn, ntile8, tolk, cmax2,
                                                                   lane);
      if constexpr (W12) sc = rows_to_lanes(sc, lane);
      id = sc.id;
      if (sc.flag || a.mti_seed) {
        // exact recipe: near-tie re-rank, or the MTI bound seed (engine.py:305-308)
        double nd;
        if constexpr (W12) {
          nd = exact_winner_stream<DP>(tb, my_r, crow, k, sc.flag, id);
          if (a.mti_seed) my_sq = exact_sq_stream<DP, true>(tb, my_r, nullptr);
        } else {
          nd = exact_winner<DP>(tb, my_r, crow, k, d, sc.flag, id, a.mti_seed ? &my_sq : nullptr);
        }
        nd2 = nd * nd;
        if (a.mti_seed && valid) {
          a.upper[row] = nd;
          a.tight[row] = 1;
        }
      } else {
        // certified winner: WCSS term from the norm form ||x||^2 - 2 s (rounding ~1e-16 ||x||^2)
        nd2 = fmax(sc.xn2 - 2.0 * sc.best, 0.0);
      }
      }
      old = valid ? old_raw : -1;
      if (valid) {
        if (id != old) {
          a.assign[row] = id;
          ++reassigned;
        }
        if (!a.mti_seed) wcss += nd2;
        ++rows_done;
      }
    } else if (valid) {
      old = old_raw;
      id = old;
      ++rows_done;
    }
    if (a.mti_filter) {
      // accumulated above
    } else if (!a.delta) {
      accumulate_full_rows<DP, TL, W12>(row_mask(valid, my_r), id, my_sq, tb, acc, cnt, sqa, d, lane);
    } else {
      // steady-state dense passes: running sums move by the reassigned rows only
      accumulate_in_row_order<DP, TL, W12>(row_mask(valid && id != old, my_r), id, old, 0.0, tb, acc, cnt, sqa, d,
                                           lane);
    }
    // ---- refill this stage with the block NS strides ahead
    __syncwarp();
    const long long nb = blk + (long long)NS * TW;
    if (nb < nblk) {
      fence_proxy_async();
      load_block<DP>(&tmap, &bar[s], tb, nb, a, tma, lane);
    }
  }
  __syncthreads();

  // CTA partial: warps' private sums added in warp order
  const long long Lg = acc_len(k, d);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  const long long kd = (long long)k * d;
  for (long long i = tid; i < kd + 2LL * k; i += blockDim.x) {
    size_t off;
    long long ii;
    if (i < kd) { off = L.acc_off; ii = i; }
    else if (i < kd + k) { off = L.cnt_off; ii = i - kd; }
    else { off = L.sq_off; ii = i - kd - k; }
    double v = 0.0;
    for (int w = 0; w < W; ++w) v += reinterpret_cast<const double*>(smem + L.warp0 + (size_t)w * L.per_warp + off)[ii];
    out[i] = v;
  }
  const double r_re = (double)warp_sum_ll(reassigned);
  const double r_w = warp_sum(wcss);
  const double r_rows = (double)warp_sum_ll(rows_done);
  const double r_sk = (double)warp_sum_ll(skips);
  const double r_cp = (double)warp_sum_ll(computed);
  if (lane == 0) {
    red[warp * 8 + 0] = r_re;
    red[warp * 8 + 1] = r_w;
    red[warp * 8 + 2] = r_rows;
    red[warp * 8 + 3] = r_sk;
    red[warp * 8 + 4] = r_cp;
  }
  __syncthreads();
  if (tid == 0) {
    double t_re = 0, t_w = 0, t_rows = 0, t_sk = 0, t_cp = 0;
    for (int w = 0; w < W; ++w) {
      t_re += red[w * 8];
      t_w += red[w * 8 + 1];
      t_rows += red[w * 8 + 2];
      t_sk += red[w * 8 + 3];
      t_cp += red[w * 8 + 4];
    }
    double* sc = out + kd + 2LL * k;
    for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
    sc[S_REASSIGNED] = t_re;
    sc[S_WCSS] = t_w;
    sc[S_COMPUTED] = a.mti_filter ? t_cp : (labels ? 0.0 : t_rows * (double)k);
    sc[S_SKIPS] = t_sk;
    sc[S_ROWS] = t_rows;
  }
}

constexpr size_t SMEM_MAX = 227 * 1024;

int warps_for(int DP, int k, int d, bool w12 = false) {
  for (int W = w12 ? KNB_DENSE_W12_THREADS / 32 : KNB_WARPS; W >= 1; --W)
    if (WarpSmem(DP, k, d, W, w12).total <= SMEM_MAX) return W;
  return 0;
}

// the twelve-warp form when all twelve warps fit (KNB_DENSE_W12=0: off, A/B runs).
// Measured: c2 (d = 32, k = 32, 12 warps) 0.244 -> 0.220 ms per steady pass; c4 (d = 16,
// k = 100: 11 warps, the sums take 13 KB per warp) 35.5 -> 37.5 ms per 200M rows, so
// the two-stage eight-warp form stays there
bool use_w12(int DP, int k, int d) {
  static const int env = [] { const char* v = getenv("KNB_DENSE_W12"); return v ? atoi(v) : 1; }();
  return env && d == DP && (DP == 16 || DP == 32) && k > 16 && warps_for(DP, k, d, true) >= 12;
}

template <int DP, bool SMALLK, bool W12 = false, bool ONE = false>
cudaError_t launch_mma_k(const CUtensorMap* tmap, const DenseArgs& a, int grid, cudaStream_t s) {
  const int W = warps_for(DP, a.k, a.d, W12);
  if (!W) return cudaErrorInvalidValue;
  const WarpSmem L(DP, a.k, a.d, W, W12);
  cudaError_t e = cudaFuncSetAttribute(dense_mma_kernel<DP, SMALLK, W12, ONE>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  return launch_pdl(dense_mma_kernel<DP, SMALLK, W12, ONE>, dim3(grid), dim3(W * 32), L.total, s, *tmap, a);
}

template <int DP>
cudaError_t launch_mma_dp(const CUtensorMap* tmap, const DenseArgs& a, int grid, cudaStream_t s) {
  if constexpr (DP == 16 || DP == 32)
    if (use_w12(DP, a.k, a.d)) return launch_mma_k<DP, false, true>(tmap, a, grid, s);
  if (a.k <= 8) return launch_mma_k<DP, true, false, true>(tmap, a, grid, s);  // c1: 0.0248 -> 0.0228 ms / iter
  return a.k <= 16 ? launch_mma_k<DP, true>(tmap, a, grid, s) : launch_mma_k<DP, false>(tmap, a, grid, s);
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

// 0 when even one warp's buffers do not fit (the generic kernel takes over)
size_t dense_mma_smem(int DP, int k, int d) {
  const bool w12 = use_w12(DP, k, d);
  const int W = warps_for(DP, k, d, w12);
  return W ? WarpSmem(DP, k, d, W, w12).total : (size_t)-1;
}

int dense_mma_rows() { return BR; }

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
