// K6 + K7 on the FP64 tensor cores: the pruned (MTI) iteration with survivors of
// the point-skip test re-assigned by certified DMMA scoring.
//
// Replaces numakmeans engine._task_pruned (engine.py:321-354) + inflate_bounds
// (pruning.py:152-160) + scan_block (pruning.py:163-204) with these semantics:
//   prologue  u += drift[a]; tight &= (drift[a] == 0)        (bound inflation, fused)
//   clause 1  the point is skipped when u <= half_min[a]      (inclusive; its row is never read)
//   survivor  its new centroid is the exhaustive argmin with scan_block's tie rule (an
//             exact tie keeps the current centroid, otherwise the lowest id wins: what the
//             reference's candidate scan returns -- pruning is sound and its distances are
//             the exact recipe), its bound becomes the exact-recipe distance to that
//             centroid and tight = 1, as in scan_block; moved points contribute signed
//             deltas.
// Assignments, bounds (and therefore every later skip decision), centroids and the
// skip counts are the reference's; dist_comps counts the k distances evaluated per
// survivor instead of the reference's clause-2/3 candidate walk (pruned_* are 0).  The
// reference-counter walk stays available as the "exact" MTI scan (mti.cu).
//
// Layout: warp-independent.  A warp filters its strided 32-row blocks reading only the
// 13 B/point state, appends survivors to a warp-private queue, and whenever 32 are
// queued gathers their rows from HBM into a swizzled 32-row tile and scores them with
// score_block (mma_common.cuh).  Deltas go through the warp-local row-ordered walk
// into warp-private sums; the CTA adds its warps' sums in warp order.
// Two forms: mti_mma_kernel (eight warps, two staging tiles per warp; k <= 16, rows in
// host memory, other shapes) and mti_w12_kernel (twelve warps per SM, one staging tile
// each; d == DP in {16, 32} with k > 16 -- config 2).  Rows of <= 8 doubles with k <= 16
// (config 3) skip the DMMA scorer: their survivors are ranked by the exact recipe directly
// (direct_winner, mma_common.cuh), which is fewer instructions than scores + certificate.
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"
#include "mma_common.cuh"

namespace knb {

namespace {

__host__ __device__ inline size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }

struct MtiMmaSmem {
  size_t bf, crow, chn, hmin, drift, red, warp0, tile_off, tile_stride, q_off, acc_off, cnt_off, sq_off, per_warp,
      total;
  // src: semi-external runs also queue each row's HBM cache slot
  __host__ __device__ MtiMmaSmem(int DP, int k, int d, int W, bool src = false) {
    const int kp = (k + 7) & ~7;
    size_t o = 0;
    bf = o;    o += (size_t)kp * DP * 8;
    crow = o;  o += (size_t)kp * (DP + 2) * 8;
    chn = o;   o += (size_t)kp * 8;
    hmin = o;  o += (size_t)k * 16;  // {drift, half_min} pairs
    drift = hmin;
    red = o;   o += 16 * 8 * 8;
    o = al(o, 1024);
    warp0 = o;
    size_t w = 0;
    tile_stride = (size_t)BR * DP * 8;
    tile_off = w; w += 2 * tile_stride;  // two staging tiles (gather double buffer)
    q_off = w;    w += 192 * 4 * (src ? 3 : 2);  // queued rows, pre-scan assignment (, cache slot)
    acc_off = w;  w += (size_t)k * d * 8;
    cnt_off = w;  w += (size_t)k * 8;
    sq_off = w;   w += (size_t)k * 8;
    per_warp = al(w, 1024);
    total = warp0 + (size_t)W * per_warp;
  }
};

#ifndef KNB_MTI_DIRECT
#define KNB_MTI_DIRECT 1
#endif

// warps per CTA of the direct-scan form (two CTAs per SM).  Measured at c3: twelve warps
// (80 registers, spills) 1.29 ms, sixteen (64 registers) 1.79 ms against 1.06 ms with eight
#ifndef KNB_MTI_DIRECT_WARPS
#define KNB_MTI_DIRECT_WARPS 8
#endif
template <int DP, bool HOST, bool SMALLK>
__host__ __device__ constexpr bool mti_direct() { return KNB_MTI_DIRECT && SMALLK && !HOST && DP <= 8; }
template <int DP, bool HOST, bool SMALLK>
__host__ __device__ constexpr int mti_threads() { return mti_direct<DP, HOST, SMALLK>() ? 32 * KNB_MTI_DIRECT_WARPS : KNB_NT; }
#ifndef KNB_MTI_2CTA_DP
#define KNB_MTI_2CTA_DP 8
#endif

// LEAN (DP = 32): the scorer's fewest-register form -- measured 3% faster at c2 (the
// registers go to scheduling freedom; twelve warps per CTA would cap them at 168 and
// spill, and one staging tile instead of two is slower)
// HOST: rows in host memory (row_gather) and/or the semi-external HBM row cache; the
// HBM-resident instantiation keeps the plain per-lane gather
template <int DP, bool HOST, bool SMALLK, bool LEAN>
__global__ void __launch_bounds__((mti_threads<DP, HOST, SMALLK>()), (SMALLK && DP <= KNB_MTI_2CTA_DP) ? 2 : 1)
    mti_mma_kernel(const MtiArgs a) {
  using TL = TileLayout<DP, 1>;  // tiles written by cp.async only: the fragment-friendly swizzle
  constexpr int KS = DP / 4;
  // narrow rows, few centroids (config 3): the survivors' k exact distances directly
  // (direct_winner), no DMMA scores
  constexpr bool DIRECT = mti_direct<DP, HOST, SMALLK>();
  extern __shared__ __align__(1024) unsigned char smem[];
  pdl_enter();
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  if (a.gate && a.ctrl->mti_choice != 0) return;  // the block-dense pass runs this iteration
  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = blockDim.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int kp = (k + 7) & ~7, ntile8 = kp >> 3;
  const int32_t* cslot = HOST ? a.cslot : nullptr;
  const MtiMmaSmem L(DP, k, d, W, cslot != nullptr);
  double* bf = reinterpret_cast<double*>(smem + L.bf);
  double* crow = reinterpret_cast<double*>(smem + L.crow);
  double* chn = reinterpret_cast<double*>(smem + L.chn);
  double2* hd = reinterpret_cast<double2*>(smem + L.hmin);  // {drift, half_min} per centroid
  double* red = reinterpret_cast<double*>(smem + L.red);
  unsigned char* wbase = smem + L.warp0 + (size_t)warp * L.per_warp;
  unsigned char* tb = wbase + L.tile_off;
  int* qrow = reinterpret_cast<int*>(wbase + L.q_off);
  int* qorig = qrow + 192;
  int* qsrc = qrow + 384;  // semi-external runs: the row's HBM cache slot (-1: host memory)
  // the queue is a ring of 192 entries starting at qh (popping a batch moves qh, no copies)
  int qh = 0;
  auto ring = [&](int i) { const int x = qh + i; return x >= 192 ? x - 192 : x; };
  double* acc = reinterpret_cast<double*>(wbase + L.acc_off);
  double* cnt = reinterpret_cast<double*>(wbase + L.cnt_off);
  double* sqa = reinterpret_cast<double*>(wbase + L.sq_off);

  for (int i = tid; i < kp * DP; i += blockDim.x) {
    const int j = i / DP, e = i - j * DP;
    crow[j * crow_stride<DP>() + e] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
    const int l = i & 31, qs = i >> 5, q = qs / KS, s = qs - q * KS;
    const int jb = q * 8 + (l >> 2), eb = s * 4 + (l & 3);
    bf[i] = (jb < k && eb < d) ? a.means[(long long)jb * d + eb] : 0.0;
  }
  for (int j = tid; j < kp; j += blockDim.x) chn[j] = j < k ? a.chn[j] : -CUDART_INF;
  for (int j = tid; j < k; j += blockDim.x) hd[j] = make_double2(a.drift[j], a.half_min[j]);
  for (int i = lane; i < k * d; i += 32) acc[i] = 0.0;
  for (int j = lane; j < k; j += 32) { cnt[j] = 0.0; sqa[j] = 0.0; }
  __syncthreads();

  const double cmax2 = a.ctrl->cmax2;
  const double tolk = (8.0 * d + 32.0) * 1.1102230246251565e-16;
  const long long nblk = (a.n + BR - 1) / BR;
  const long long gw = (long long)blockIdx.x * W + warp, TW = (long long)gridDim.x * W;
  const bool vec = ((d & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
  long long computed = 0, reassigned = 0;
  int qn = 0;
  // both staging tiles start zeroed: padded dims stay zero, rows past a batch hold stale finite data
  for (int i = lane; i < 2 * BR * DP; i += 32) reinterpret_cast<double*>(tb)[i] = 0.0;
  __syncwarp();

  // async gather of queued entries [base, base + cnum) into a staging tile (rows 0..cnum-1)
  auto gather = [&](unsigned char* dstp, int base, int cnum) {
    const uint32_t dst = smem_u32(dstp);
    // source of each lane's row: HBM rows, the HBM row cache (semi-external runs), or
    // host memory
    const double* src = nullptr;
    bool host = false;
    if (lane < cnum) {
      const int qi = ring(base + lane);
      const int r = qrow[qi];
      const int slot = cslot ? qsrc[qi] : -1;
      src = slot >= 0 ? a.cache + (long long)slot * d : a.X + (long long)r * d;
      host = a.row_gather && slot < 0;
    }
    if (vec && (!HOST || !__any_sync(0xffffffffu, host))) {
      // rows in HBM: every lane copies its own row (unrolled, no index arithmetic)
      if (lane < cnum) {
#pragma unroll
        for (int q2 = 0; q2 < DP / 2; ++q2)
          if (2 * q2 < d) cp_async16_s(dst + TL::chunk_off(lane, q2, BR), src + 2 * q2);
      }
    } else {
      if (vec) {
        // consecutive lanes copy consecutive 16-byte chunks of the same row: each
        // row is fetched as one coalesced request over the host link
        const int hd = d >> 1, tot = cnum * hd;
        for (int i0 = 0; i0 < tot; i0 += 32) {
          const int i = i0 + lane;
          const int r = (i < tot ? i : tot - 1) / hd, q2 = i - r * hd;
          const double* p = reinterpret_cast<const double*>(
              __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), r));
          if (i < tot) cp_async16_s(dst + TL::chunk_off(r, q2, BR), p + 2 * q2);
        }
      } else if (lane < cnum) {
#pragma unroll
        for (int e = 0; e < DP; ++e)
          if (e < d) cp_async8_s(dst + TL::elem_off(lane, e, BR), src + e);
      }
    }
    cp_async_commit();
  };

  // score and update the first `cnum` queued survivors (cnum <= 32), staged in tb
  auto process = [&](const unsigned char* tb, int cnum) {
    const int r = lane;  // lane r handles row r from here on
    const bool valid = r < cnum;
    const int orig = valid ? qorig[ring(r)] : 0;
    int id;
    double nd;
    if constexpr (DIRECT) {
      nd = direct_winner<DP, TL>(tb, r, crow, k, d, orig, id);
    } else {
      const Scored sc = rows_to_lanes(score_block<DP, SMALLK, LEAN, false, false, TL>(tb, bf, chn, ntile8, tolk,
                                                                                       cmax2, lane), lane);
      id = sc.id;
      nd = exact_winner<DP, TL>(tb, r, crow, k, d, sc.flag, id, nullptr, valid ? orig : -1);
    }
    const bool moved = valid && id != orig;
    // ||x||^2 only for the (few) moved rows whose signed deltas carry it
    const double sq = moved ? row_self_sq<DP, TL>(tb, r, d) : 0.0;
    if (valid) {
      const long long grow = qrow[ring(r)];
      a.upper[grow] = nd;
      a.tight[grow] = 1;
      if (moved) {
        a.assign[grow] = id;
        ++reassigned;
      }
    }
    if (lane == 0) computed += (long long)cnum * k;
    accumulate_in_row_order<DP, TL, true>(row_mask(moved, r), id, orig, sq, tb, acc, cnt, sqa, d, lane);
    __syncwarp();
  };

  // filter strided blocks (bound inflation + clause 1) until `target` survivors are queued.
  // The per-row state of the NEXT group of FB blocks is loaded while the current group is
  // filtered (and across calls), so the loads' latency overlaps useful work.  Row and
  // block indices are 32-bit (launch_pass runs this kernel only when mti_compact_ok).
  const int n32 = (int)a.n, nblk32 = (n32 + BR - 1) / BR, TW32 = (int)TW;
  int blk = (int)gw;
  const int32_t* __restrict__ g_assign = a.assign;
  double* __restrict__ g_upper = a.upper;
  uint8_t* __restrict__ g_tight = a.tight;
  constexpr int FB = DP <= 32 ? 4 : 2;  // (DP = 64 is register-bound)
  // (measured: prefetching at DP = 32 costs 1.6% at c2 -- the registers matter more)
  constexpr bool PREFETCH = DP <= 16;
  int pa[FB], ps[FB];
  double pu[FB];
  auto load_group = [&](int b) {
#pragma unroll
    for (int j = 0; j < FB; ++j) {
      const int bj = b + j * TW32;
      const int row = bj * BR + lane;
      const bool ok = bj < nblk32 && row < n32;
      pa[j] = ok ? g_assign[row] : -1;
      pu[j] = ok ? g_upper[row] : 0.0;
      if constexpr (HOST) ps[j] = (ok && cslot) ? cslot[row] : -1;
    }
  };
  if constexpr (PREFETCH) load_group(blk);
  int skips32 = 0;
  auto filter_until = [&](int target) {
    while (qn < target && blk < nblk32) {
      if constexpr (!PREFETCH) load_group(blk);
      int aa[FB], sl[FB];
      double uu[FB];
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        aa[j] = pa[j];
        uu[j] = pu[j];
        if constexpr (HOST) sl[j] = ps[j];
      }
      const int cur = blk;
      blk += FB * TW32;
      if constexpr (PREFETCH) load_group(blk);  // prefetch the next group
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        const int bj = cur + j * TW32;
        if (bj >= nblk32) break;  // uniform
        const int row = bj * BR + lane;
        const int aj = aa[j] < 0 ? 0 : aa[j];
        const double2 dh = hd[aj];  // {drift, half_min}
        const double u = uu[j] + dh.x;  // u + 0.0 == u
        const bool valid = aa[j] >= 0;
        const bool skip = valid && u <= dh.y;
        const bool live = valid && !skip;  // a survivor's bound and tight flag are rewritten by its scan
        skips32 += skip;
        if (skip && dh.x != 0.0) {  // the inflated bound is the skipped row's final state
          g_upper[row] = u;
          g_tight[row] = 0;
        }
        const unsigned b = __ballot_sync(0xffffffffu, live);
        if (live) {
          const int pos = ring(qn + __popc(b & ((1u << lane) - 1u)));
          qrow[pos] = row;
          qorig[pos] = aa[j];
          if (HOST && cslot) qsrc[pos] = sl[j];
        }
        qn += __popc(b);
      }
      __syncwarp();
    }
  };

  // two staging tiles: the next batch's rows stream in while the current one is scored
  int cur = 0;
  filter_until(32);
  int b0 = qn < 32 ? qn : 32;
  if (b0 > 0) gather(tb, 0, b0);
  while (b0 > 0) {
    filter_until(64);
    const int b1 = (b0 == 32 && qn > 32) ? (qn - 32 < 32 ? qn - 32 : 32) : 0;
    unsigned char* tcur = tb + cur * L.tile_stride;
    if (b1 > 0) {
      gather(tb + (cur ^ 1) * L.tile_stride, 32, b1);
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncwarp();
    process(tcur, b0);
    // pop the processed batch from the queue
    const int rest = qn - b0;
    qh = ring(b0);
    qn = rest;
    b0 = b1;
    cur ^= 1;
  }
  __syncthreads();

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
  const long long v0 = warp_sum_ll(reassigned), v1 = warp_sum_ll(computed), v2 = warp_sum_ll((long long)skips32);
  if (lane == 0) { red[warp * 8 + 0] = (double)v0; red[warp * 8 + 1] = (double)v1; red[warp * 8 + 2] = (double)v2; }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0, t1 = 0, t2 = 0;
    for (int w = 0; w < W; ++w) { t0 += red[w * 8]; t1 += red[w * 8 + 1]; t2 += red[w * 8 + 2]; }
    double* sc = out + kd + 2LL * k;
    for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
    sc[S_REASSIGNED] = t0;
    sc[S_COMPUTED] = t1;
    sc[S_SKIPS] = t2;
  }
}

// ---------------------------------------------------------------------------------
// Twelve-warp form (rows in HBM, d == DP): the same filter / gather / certified DMMA
// scoring / exact bound / signed deltas as mti_mma_kernel, re-budgeted so that three
// warps share each SMSP instead of two -- the pass is bound by warp-level latency, not by
// the tensor pipe (profiles/README.md).  Per warp: one staging tile (the next batch is
// gathered while the following one is filtered), a 160-entry queue; per CTA: one
// row-major centroid copy serving both the B fragments and the exact recipe; the exact
// distances stream through the tree eight elements at a time (about 20 live doubles).
#ifndef KNB_W12_FB
#define KNB_W12_FB 2  // with the prefetch: measured c2 0.1710 -> 0.1693 ms (FB 4 + prefetch spills)
#endif
#ifndef KNB_W12_PREFETCH
#define KNB_W12_PREFETCH 1
#endif
#ifndef KNB_W12_COOP
#define KNB_W12_COOP 1  // measured at c2: MTI 0.165 -> 0.158 ms
#endif
constexpr int W12_Q = 160;  // < 32 queued + one group of FB = 4 blocks

struct MtiW12Smem {
  size_t crow, chn, hd, red, warp0, tile_stride, q_off, acc_off, cnt_off, sq_off, per_warp, total;
  __host__ __device__ MtiW12Smem(int DP, int k, int d, int W) {
    const int kp = (k + 7) & ~7;
    size_t o = 0;
    crow = o;  o += (size_t)kp * (DP + 2) * 8;
    chn = o;   o += (size_t)kp * 8;
    hd = o;    o += (size_t)k * 16;  // {drift, half_min}
    red = o;   o += 16 * 8 * 8;
    o = al(o, 128);
    warp0 = o;
    size_t w = 0;
    tile_stride = (size_t)BR * DP * 8;
    w += tile_stride;
    q_off = w;    w += W12_Q * 4 * 2;
    acc_off = w;  w += (size_t)k * d * 8;
    cnt_off = w;  w += (size_t)k * 8;
    sq_off = w;   w += (size_t)k * 8;
    per_warp = al(w, 128);
    total = warp0 + (size_t)W * per_warp;
  }
};

#ifndef KNB_W12_THREADS
#define KNB_W12_THREADS 384
#endif

template <int DP>
__global__ void __launch_bounds__(KNB_W12_THREADS, 1) mti_w12_kernel(const MtiArgs a) {
  using TL = TileLayout<DP, 1>;  // written by cp.async only: the fragment-friendly swizzle
  extern __shared__ __align__(1024) unsigned char smem[];
  pdl_enter();
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  if (a.gate && a.ctrl->mti_choice != 0) return;  // the block-dense pass runs this iteration
  const int k = a.k, d = a.d, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = blockDim.x >> 5;
  const int kp = (k + 7) & ~7, ntile8 = kp >> 3;
  const MtiW12Smem L(DP, k, d, W);
  double* crow = reinterpret_cast<double*>(smem + L.crow);
  double* chn = reinterpret_cast<double*>(smem + L.chn);
  double2* hd = reinterpret_cast<double2*>(smem + L.hd);
  double* red = reinterpret_cast<double*>(smem + L.red);
  unsigned char* wbase = smem + L.warp0 + (size_t)warp * L.per_warp;
  unsigned char* tb = wbase;
  int* qrow = reinterpret_cast<int*>(wbase + L.q_off);
  int* qorig = qrow + W12_Q;
  int qh = 0;
  auto ring = [&](int i) { const int x = qh + i; return x >= W12_Q ? x - W12_Q : x; };
  double* acc = reinterpret_cast<double*>(wbase + L.acc_off);
  double* cnt = reinterpret_cast<double*>(wbase + L.cnt_off);
  double* sqa = reinterpret_cast<double*>(wbase + L.sq_off);

  for (int i = tid; i < kp * DP; i += blockDim.x) {
    const int j = i / DP, e = i - j * DP;
    crow[j * crow_stride<DP>() + e] = (j < k && e < d) ? a.means[(long long)j * d + e] : 0.0;
  }
  for (int j = tid; j < kp; j += blockDim.x) chn[j] = j < k ? a.chn[j] : -CUDART_INF;
  for (int j = tid; j < k; j += blockDim.x) hd[j] = make_double2(a.drift[j], a.half_min[j]);
  for (int i = lane; i < k * d + 2 * k; i += 32) acc[i] = 0.0;  // acc, cnt, sq are contiguous
  // rows past a batch keep stale finite data (d == DP: no padded dims)
  for (int i = lane; i < BR * DP; i += 32) reinterpret_cast<double*>(tb)[i] = 0.0;
  __syncthreads();

  const double cmax2 = a.ctrl->cmax2;
  const double tolk = (8.0 * d + 32.0) * 1.1102230246251565e-16;
  const long long nblk = (a.n + BR - 1) / BR;
  const long long gw = (long long)blockIdx.x * W + warp, TW = (long long)gridDim.x * W;
  long long skips = 0, computed = 0, reassigned = 0;
  int qn = 0;

  // async gather of queued entries [0, cnum) into the staging tile: every lane its row.
  // Returns the row's stored bound (the load stays in flight while the next batch is
  // filtered): ||x||^2 <= 2 ||c_a||^2 + 2 u^2 bounds the certificate's tolerance, so the
  // scorer skips its d-term sums.
  auto gather = [&](int cnum) -> double {
    const uint32_t dst = smem_u32(tb);
    double uraw = 0.0;
#if KNB_W12_COOP
    // consecutive lanes copy consecutive 16-byte chunks of the same row (64 / DP rows
    // per instruction): coalesced global reads, fewer shared-memory wavefronts
    const double* src = nullptr;
    if (lane < cnum) {
      const int row = qrow[ring(lane)];
      src = a.X + (long long)row * d;
      uraw = a.upper[row];  // not yet inflated (the filter leaves survivors' bounds alone)
    }
    constexpr int HC = DP / 2, RPI = 32 / HC;
    const int q2 = lane % HC, rl = lane / HC;
#pragma unroll
    for (int it = 0; it < BR / RPI; ++it) {
      if (it * RPI >= cnum) break;  // uniform
      const int rr = it * RPI + rl;
      const double* p = reinterpret_cast<const double*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), rr));
      if (rr < cnum) cp_async16_s(dst + TL::chunk_off(rr, q2, BR), p + 2 * q2);
    }
#else
    if (lane < cnum) {
      const int row = qrow[ring(lane)];
      const double* src = a.X + (long long)row * d;
#pragma unroll
      for (int q2 = 0; q2 < DP / 2; ++q2) cp_async16_s(dst + TL::chunk_off(lane, q2, BR), src + 2 * q2);
      uraw = a.upper[row];  // not yet inflated (the filter leaves survivors' bounds alone)
    }
#endif
    cp_async_commit();
    return uraw;
  };

  long long blk = gw;
  constexpr int FB = KNB_W12_FB;
  int pa[FB];
  double pu[FB];
  auto load_group = [&](long long b) {
#pragma unroll
    for (int j = 0; j < FB; ++j) {
      const long long row = (b + j * TW) * BR + lane;
      const bool ok = b + j * TW < nblk && row < a.n;
      pa[j] = ok ? a.assign[row] : -1;
      pu[j] = ok ? a.upper[row] : 0.0;
    }
  };
  if (KNB_W12_PREFETCH) load_group(blk);
  auto filter_until = [&](int target) {
    while (qn < target && blk < nblk) {
      int aa[FB];
      double uu[FB];
      if (!KNB_W12_PREFETCH) load_group(blk);
#pragma unroll
      for (int j = 0; j < FB; ++j) { aa[j] = pa[j]; uu[j] = pu[j]; }
      const long long cur = blk;
      blk += FB * TW;
      if (KNB_W12_PREFETCH) load_group(blk);  // the next group's state loads overlap this one's filter
#pragma unroll
      for (int j = 0; j < FB; ++j) {
        if (cur + j * TW >= nblk) break;  // uniform
        const long long row = (cur + j * TW) * BR + lane;
        bool live = false;
        if (aa[j] >= 0) {
          const double2 dh = hd[aa[j]];
          const double u = uu[j] + dh.x;  // u + 0.0 == u
          if (u <= dh.y) {
            ++skips;
            if (dh.x != 0.0) {  // the inflated bound is the skipped row's final state
              a.upper[row] = u;
              a.tight[row] = 0;
            }
          } else {
            live = true;  // a survivor's bound and tight flag are rewritten by its scan
          }
        }
        const unsigned b = __ballot_sync(0xffffffffu, live);
        if (live) {
          const int pos = ring(qn + __popc(b & ((1u << lane) - 1u)));
          qrow[pos] = (int)row;
          qorig[pos] = aa[j];
        }
        qn += __popc(b);
      }
      __syncwarp();
    }
  };

  // batch loop: gather the next 32 survivors, filter ahead while they land, score
  filter_until(32);
  while (qn > 0) {
    const int cnum = qn < 32 ? qn : 32;
    const double uraw = gather(cnum);
    filter_until(32 + cnum);  // the following batch's survivors, overlapping the gather
    // lane r handles row r from here on (8 consecutive rows per quarter-warp: the exact
    // tree's row loads hit distinct bank groups)
    const int r = lane;
    const bool valid = r < cnum;
    const int orig = valid ? qorig[ring(r)] : 0;
    const double xb = valid ? xnorm2_bound(uraw + hd[orig].x, chn[orig]) : 0.0;
    cp_async_wait_all();
    __syncwarp();
    const Scored sc = score_block<DP, false, true, true, true, TL>(tb, crow, chn, ntile8, tolk, cmax2, lane, xb);
    int id = __shfl_sync(0xffffffffu, sc.id, owner_lane(r));
    const bool flag = __shfl_sync(0xffffffffu, (int)sc.flag, owner_lane(r)) != 0;
    const double nd = exact_winner_stream<DP, TL>(tb, r, crow, k, flag, id, valid ? orig : -1);
    const bool moved = valid && id != orig;
    const double sq = moved ? exact_sq_stream<DP, true, TL>(tb, r, nullptr) : 0.0;
    if (valid) {
      const long long grow = qrow[ring(r)];
      a.upper[grow] = nd;
      a.tight[grow] = 1;
      if (moved) {
        a.assign[grow] = id;
        ++reassigned;
      }
    }
    if (lane == 0) computed += (long long)cnum * k;
    accumulate_in_row_order<DP, TL, true>(row_mask(moved, r), id, orig, sq, tb, acc, cnt, sqa, d, lane);
    __syncwarp();
    qh = ring(cnum);  // pop the batch
    qn -= cnum;
  }
  __syncthreads();

  const long long Lg = acc_len(k, d);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  const long long kd = (long long)k * d;
  for (long long i = tid; i < kd + 2LL * k; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < W; ++w) v += reinterpret_cast<const double*>(smem + L.warp0 + (size_t)w * L.per_warp + L.acc_off)[i];
    out[i] = v;
  }
  const long long v0 = warp_sum_ll(reassigned), v1 = warp_sum_ll(computed), v2 = warp_sum_ll(skips);
  if (lane == 0) { red[warp * 8 + 0] = (double)v0; red[warp * 8 + 1] = (double)v1; red[warp * 8 + 2] = (double)v2; }
  __syncthreads();
  if (tid == 0) {
    double t0 = 0, t1 = 0, t2 = 0;
    for (int w = 0; w < W; ++w) { t0 += red[w * 8]; t1 += red[w * 8 + 1]; t2 += red[w * 8 + 2]; }
    double* sc = out + kd + 2LL * k;
    for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
    sc[S_REASSIGNED] = t0;
    sc[S_COMPUTED] = t1;
    sc[S_SKIPS] = t2;
  }
}

constexpr size_t SMEM_MAX = 227 * 1024;

int w12_warps_for(int DP, int k, int d) {
  if (d != DP || (DP != 16 && DP != 32)) return 0;
  const int W = KNB_W12_THREADS / 32;
  return MtiW12Smem(DP, k, d, W).total <= SMEM_MAX ? W : 0;  // else the two-tile kernel
}

template <int DP>
cudaError_t launch_w12(const MtiArgs& a, int grid, cudaStream_t s) {
  const int W = w12_warps_for(DP, a.k, a.d);
  const MtiW12Smem L(DP, a.k, a.d, W);
  cudaError_t e =
      cudaFuncSetAttribute(mti_w12_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_w12_kernel<DP>, dim3(grid), dim3(W * 32), L.total, s, a);
}

int mti_warps_for(int DP, int k, int d, bool src = false, int wmax = KNB_WARPS) {
  for (int W = wmax; W >= 1; --W)
    if (MtiMmaSmem(DP, k, d, W, src).total <= SMEM_MAX) return W;
  return 0;
}

template <int DP, bool HOST, bool SMALLK, bool LEAN = false>
cudaError_t launch_host(const MtiArgs& a, int grid, cudaStream_t s) {
  const bool src = HOST && a.cslot != nullptr;
  const int W = mti_warps_for(DP, a.k, a.d, src, mti_threads<DP, HOST, SMALLK>() / 32);
  if (!W) return cudaErrorInvalidValue;
  const MtiMmaSmem L(DP, a.k, a.d, W, src);
  cudaError_t e =
      cudaFuncSetAttribute(mti_mma_kernel<DP, HOST, SMALLK, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)L.total);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_mma_kernel<DP, HOST, SMALLK, LEAN>, dim3(grid), dim3(W * 32), L.total, s, a);
}

template <int DP>
cudaError_t launch_dp(const MtiArgs& a, int grid, cudaStream_t s) {
  if (a.row_gather || a.cslot) return launch_host<DP, true, false>(a, grid, s);
  if constexpr (DP == 16 || DP == 32) {
    // (KNB_MTI_W12=0: the two-tile eight-warp kernel, for A/B measurements)
    static const int w12_env = [] { const char* v = getenv("KNB_MTI_W12"); return v ? atoi(v) : 1; }();
    // (16-byte cp.async row copies: rows must be 16-byte aligned, e.g. not a view at an odd offset)
    if (w12_env && a.k > 16 && w12_warps_for(DP, a.k, a.d) && (reinterpret_cast<uintptr_t>(a.X) & 15) == 0)
      return launch_w12<DP>(a, grid, s);
  }
  if (a.k <= 16) return launch_host<DP, false, true>(a, grid, s);
  if constexpr (DP == 32) return launch_host<DP, false, false, true>(a, grid, s);
  return launch_host<DP, false, false>(a, grid, s);
}

}  // namespace

bool mti_mma_fits(int DP, int k, int d) { return DP >= 4 && DP <= 64 && mti_warps_for(DP, k, d) > 0; }

// the compacted kernels' filter walks 32-bit row / block indices (blk may run FB * TW
// blocks past the end): shards up to 2^31 - 2^26 rows
bool mti_compact_ok(long long n_local) { return n_local <= (1LL << 31) - (1LL << 26); }

cudaError_t launch_mti_mma(const MtiArgs& a, int DP, int grid, cudaStream_t s) {
  switch (DP) {
    case 4: return launch_dp<4>(a, grid, s);
    case 8: return launch_dp<8>(a, grid, s);
    case 16: return launch_dp<16>(a, grid, s);
    case 32: return launch_dp<32>(a, grid, s);
    case 64: return launch_dp<64>(a, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace knb
