// K6/K7-TC: the pruned (MTI) pass for f64 rows on the tcgen05 tensor cores, with a
// certified argmin.  Rows of 16 doubles take it automatically (BASELINE config 4: n =
// 856M, d = 16, k = 100, where clause 1 skips almost nothing and every row is re-scored
// each pass); rows of 8 and 32 (configs 3, 2) run it when forced (mti_scan="tc").
//
// Replaces numakmeans engine._task_pruned (engine.py:321-354) + inflate_bounds
// (pruning.py:152-160) + scan_block (pruning.py:163-204) with the semantics of the
// DMMA block pass (assign_mma.cu, mti_filter):
//   prologue  u += drift[a]; tight &= (drift[a] == 0)           (bound inflation)
//   clause 1  skip when u <= half_min[a]                         (pruning.py:100-102)
//   survivor  the exhaustive argmin with scan_block's tie rule; bound = the exact-recipe
//             distance to it (distance.py:28-39), tight = 1; moved rows give signed
//             deltas of sums / counts / sq (engine.py:345-353)
//
// Scores.  The tensor core has no f64 kind, and DMMA (mma.sync f64) runs the c4 pass
// at ~0.5 of the FP64 peak (latency bound, 8 warps).  Here each f64 value is split
// into two TF32 terms -- x = x_hi + x_lo (x_hi = f32(x) truncated to 10 mantissa bits,
// x_lo the f32 remainder, truncated by the tensor core) -- and one chain of kind::tf32
// UMMAs (M = 128 rows, N = k padded to 16, K = 8 each: 4 / 7 / 13 of them for rows of
// 8 / 16 / 32, Geo<XD>) accumulates, in TMEM,
//     D~_j = (x_hi + x_lo).(-2 c_hi)  +  x_hi.(-2 c_lo)  +  ||c_j||^2  +  ||x||^2
//          ~ ||x - c_j||^2
// (the x_lo.c_lo term, ~2^-20 |x||c|, is dropped; the two norms enter through a
// constant k-step: A = [1, 1, xn2_hi, xn2_lo], B = [cn2_hi, cn2_lo, 1, 1]); the operand
// layouts are listed at Geo.
//
// Certificate.  |D~_j - D_j| <= E(x) with
//     E = 2^-20 (C1 ||x|| cmax + C2 (||x||^2 + cmax^2)) + (8d + 32) 2^-53 (||x||^2 + cmax^2)
// (C1 = 12.5, C2 = 4 for rows of 8 / 16, 20 and 6 for 32: operand splitting <= 3.2 *
// 2^-20 |x_i c_i| per product, x2 for the -2 scale; the f32 accumulation <= 2^-22 per
// k-step of the partial magnitudes, bounded by ||x||^2 + cmax^2 + 2 ||x|| cmax; the
// last term is the reference's own f64 rounding of sum (x - c)^2, as in the DMMA
// certificate).  tests/test_gpu_mti_tc.py measures the worst |D~ - D| / E on
// adversarial inputs of every width and requires < 1/4.  The epilogue finds the
// smallest and second-smallest D~ of the row with integer min trees on keys = (f32 bits
// & ~127) | column (order-preserving for D~ >= 0; the column index rides in the low 7
// bits, < 2^-16 relative); a row is CERTIFIED when second - first > 2E (+ the key
// slack): its winner is the reference's argmin.  Other rows (near ties, exact ties,
// tiny negative D~) go to a queue that mti_tc_rerank_kernel re-ranks after the pass
// with the exact recipe in scan_block's order (current centroid first, strict <);
// beyond the queue's capacity the warp re-ranks them in the pass.  The outputs are the
// reference's bit for bit.
//
// Kernel shape (one CTA per SM, persistent over 128-row tiles, static schedule):
//   warp 0      TMA producer: f64 row tiles (128 rows, SWIZZLE_128B / 64B) through an
//               NX-stage ring (five stages at c4), tiles PF ahead prefetched into L2
//   warp 1      TMEM allocation (four 128-column accumulators) and the single-thread
//               UMMA issuer (tile i into accumulator i % 4)
//   warps 2-3   converters (NCONV): f64 -> (x_hi, x_lo) TF32 operand tile + the norm
//               constants + ||x||^2 per row, NA-stage ring
//   NGRP = 3 groups of four epilogue warps, tile i on group i % 3: one thread per row
//               (TMEM lane), key min trees, certificate (E(x) from ||x||^2), queue of
//               uncertified rows, exact bound of the winner from the f64 stage, MTI
//               state; then the f64 stage is released and the tile's moved rows are
//               written as a 144-byte record (row mask + old ids)
// mti_tc_rerank_kernel settles the queued rows (and adds their records' moved bits);
// mti_tc_delta_kernel turns the records into per-CTA signed deltas of sums / counts /
// sq in row order (deterministic), summed by reduce_kernel like every other pass.
// HBM traffic per row: 8d B of rows + 13 B of state read + 9-13 B written (+ records).
#include <cuda.h>
#include <math_constants.h>

#include <utility>

#include "common.cuh"
#include "kernels.h"
#include "mma_common.cuh"
#include "tc_common.cuh"

namespace knb {

namespace {

constexpr int XT = 128;                        // rows per tile (UMMA M)
constexpr uint32_t CH = XT * 128;              // one 128-byte-row SW128 operand chunk (16 KB)

// Layouts per row width XD in {8, 16, 32} (configs 3, 4, 2).  The f64 stage is the
// tile's rows as TMA wrote them: XD = 8 one 64-byte-wide box (SWIZZLE_64B), XD = 16 one
// 128-byte box (SWIZZLE_128B), XD = 32 two 128-byte boxes (columns 0-15, 16-31).  The
// TF32 operands are 128-byte K chunks (SWIZZLE_128B), one UMMA k-step = 8 tf32 = 32 B:
//   XD = 8:  A = [x_hi | x_lo | x_hi | 1 1 xn2_hi xn2_lo 0 0 0 0]
//            B = [-2c_hi | -2c_hi | -2c_lo | cn2_hi cn2_lo 1 1 0 0 0 0]      4 k-steps
//   XD = 16: A = [x_hi | x_lo], [1 1 xn2_hi xn2_lo 0..]
//            B = [-2c_hi | -2c_hi], [-2c_lo | cn2_hi cn2_lo 1 1 0..]          7 k-steps
//   XD = 32: A = [x_hi], [x_lo], [1 1 xn2_hi xn2_lo 0..]
//            B = [-2c_hi], [-2c_lo], [cn2_hi cn2_lo 1 1 0..]                  13 k-steps
template <int XD>
struct Geo {
  static_assert(XD == 8 || XD == 16 || XD == 32, "row widths 8, 16, 32");
  static constexpr uint32_t X_TILE = XT * XD * 8;         // f64 stage bytes
  static constexpr int NTMA = XD == 32 ? 2 : 1;           // TMA boxes per tile
  static constexpr int A_NCH = XD == 32 ? 3 : (XD == 16 ? 2 : 1);  // operand chunks (incl. constants)
  static constexpr uint32_t A_TILE = A_NCH * CH;
  static constexpr int B_NCH = A_NCH;
  // the certificate's product / accumulation coefficients (2^-20 units): 6.4 for the split
  // products, half a unit per f32 accumulation step
  static constexpr float C1 = XD == 32 ? 20.0f : 12.5f;
  static constexpr float C2 = XD == 32 ? 6.0f : 4.0f;
};

// byte offset of 16-byte chunk q (0 .. XD/2 - 1) of row r in the f64 stage
template <int XD>
__device__ __forceinline__ uint32_t xoff(int r, int q) {
  if constexpr (XD == 8) return (uint32_t)r * 64u + ((uint32_t)((q ^ (r >> 1)) & 3) << 4);
  else if constexpr (XD == 16) return (uint32_t)r * 128u + ((uint32_t)((q ^ r) & 7) << 4);
  else return (uint32_t)(q >> 3) * CH + (uint32_t)r * 128u + ((uint32_t)(((q & 7) ^ r) & 7) << 4);
}
// row r of a stage read element by element (exact_sq_fixed's x operand, no register copy)
template <int XD>
struct StageRow {
  const unsigned char* xs;
  int r;
  __device__ __forceinline__ double operator[](int i) const {
    return *reinterpret_cast<const double*>(xs + xoff<XD>(r, i >> 1) + (i & 1) * 8);
  }
};
#ifndef KNB_TCX_PF
#define KNB_TCX_PF 6
#endif
constexpr int PF = KNB_TCX_PF;                 // tiles pulled into L2 ahead of their TMA load
#ifndef KNB_TCX_NA
#define KNB_TCX_NA 2
#endif
constexpr int NA = KNB_TCX_NA;                 // operand stages
// ablations for timing studies only (wrong results): the converters skip the operand
// writes / the epilogue stops after the key trees
#ifndef KNB_TCX_ABL
#define KNB_TCX_ABL 0
#endif

// f64 stages at most.  Five, not the six that fit: 16 KB less shared memory moves the
// carve-out from 228 to 196 KB, i.e. 60 KB of L1 instead of 28 KB for the state loads and
// stores (measured at c4: 6 -> 45.5, 5 -> 45.0, 4 -> 46.1 ms per iteration)
#ifndef KNB_TCX_NXMAX
#define KNB_TCX_NXMAX 5
#endif
constexpr int NE = 8;                          // E(x) ring (tiles), indexed by tile & 7
constexpr int TCOLS = 128;                     // TMEM columns per accumulator buffer
#ifndef KNB_TCX_GROUPS
#define KNB_TCX_GROUPS 3
#endif
// warps: 0 TMA, 1 MMA, converters (NCONV), then NGRP epilogue groups of four; sixteen
// warps (four per scheduler) keep 128 registers per thread (measured: eighteen warps at
// 96 registers spill and run 1.97 vs 1.44 ms per 20M c4 rows)
constexpr int NGRP = KNB_TCX_GROUPS;           // epilogue groups = TMEM accumulator buffers
#ifndef KNB_TCX_CONV
#define KNB_TCX_CONV 2
#endif
constexpr int NCONV = KNB_TCX_CONV;            // converter warps (128 / (32 NCONV) rows per thread)
#ifndef KNB_TCX_REGS
#define KNB_TCX_REGS 128
#endif
// accumulator groups (16 columns each) read per TMEM batch -- load, one wait, reduce.
// Measured at c4 (seven groups; same box): 1 -> 47.0, 2 -> 46.8, 3 -> 46.1, 4 -> 47.5,
// 7 -> 46.7 ms per iteration
#ifndef KNB_TCX_GB
#define KNB_TCX_GB 3
#endif
constexpr int W_CONV = 2, W_EPI = 2 + NCONV;
constexpr int THREADS = 32 * (W_EPI + 4 * NGRP);
constexpr int TALLOC = NGRP <= 2 ? 2 * TCOLS : 4 * TCOLS;  // power-of-two TMEM allocation
// TMEM accumulator buffers: tile i uses buffer i % NACC (any group).  With three groups the
// four-buffer allocation holds a spare accumulator, so the in-order MMA issue runs one
// tile further ahead of the slowest group
#ifndef KNB_TCX_NACC
#define KNB_TCX_NACC (TALLOC / TCOLS)
#endif
constexpr int NACC = KNB_TCX_NACC;

__host__ __device__ inline uint32_t al(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

template <int XD>
struct TcxSmem {
  uint32_t x0, a0, b0, crow, hd, ebuf, bars, total;
  int NX;
  __host__ __device__ TcxSmem(int k, int N, int nx) {
    NX = nx;
    uint32_t o = 0;
    a0 = o;   o += NA * Geo<XD>::A_TILE;
    x0 = o;   o += nx * Geo<XD>::X_TILE;
    b0 = o;   o += (uint32_t)Geo<XD>::B_NCH * N * 128u;
    crow = o; o += (uint32_t)k * crow_stride<XD>() * 8u;
    hd = o;   o += (uint32_t)k * 16u;
    ebuf = o; o += (uint32_t)NE * XT * 4u;
    o = al(o, 16);
    bars = o; o += 8 * (2 * nx + 2 * NA + 2 * 4) + 16;
    total = o + 1024;  // runtime 1024-byte alignment of the dynamic window
  }
};

template <int W>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&r)[16]) {
  if constexpr (W == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
  } else {
    static_assert(W == 8, "8 or 16 columns");
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
  }
}

__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// mbarrier wait that suspends the thread in hardware (time hint) instead of spinning:
// the waiting producer / issuer / converter lanes then take no issue slots from the
// epilogue warps on the same scheduler
#ifndef KNB_TCX_SPIN
#define KNB_TCX_SPIN 0
#endif
__device__ __forceinline__ void mbar_sleep(uint64_t* bar, uint32_t parity) {
  if (KNB_TCX_SPIN) {
    mbar_wait(bar, parity);
    return;
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// key = (bits & ~127) | j in ONE lop3 (mask in a register, the column as the immediate)
template <int J>
__device__ __forceinline__ int pack_key(uint32_t bits, uint32_t mask) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(bits), "r"(mask), "n"(J));
  return (int)r;
}

// byte offset of 16-byte chunk q of row r in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + ((uint32_t)(q ^ (r & 7)) << 4); }

// Optional per-role cycle accounting (build with -DKNB_TCX_PROF=1; knb_mti_tc_prof reads
// and clears it): where the producer, issuer, converter and epilogue warps wait or work.
#ifndef KNB_TCX_PROF
#define KNB_TCX_PROF 0
#endif
__device__ unsigned long long g_tcx_prof[18];
struct ProfClock {
  long long t = 0;
  unsigned long long acc[6] = {0, 0, 0, 0, 0, 0};
  __device__ __forceinline__ void start() {
    if constexpr (KNB_TCX_PROF) t = clock64();
  }
  __device__ __forceinline__ void lap(int slot) {
    if constexpr (KNB_TCX_PROF) {
      const long long u = clock64();
      acc[slot] += (unsigned long long)(u - t);
      t = u;
    }
  }
  __device__ __forceinline__ void flush(int base, int n, bool who) {
    if constexpr (KNB_TCX_PROF) {
      if (who)
        for (int i = 0; i < n; ++i) atomicAdd(&g_tcx_prof[base + i], acc[i]);
    }
  }
};

template <class F, int... G>
__device__ __forceinline__ void for_groups_impl(F& f, std::integer_sequence<int, G...>) {
  (f(std::integral_constant<int, G>{}), ...);
}
// f(integral_constant<int, g>) for g = 0 .. NG-1, unrolled at compile time
template <int NG, class F>
__device__ __forceinline__ void for_groups(F&& f) {
  for_groups_impl(f, std::make_integer_sequence<int, NG>{});
}

// independent add-min chains of the second-smallest search (measured at c4: 2 -> 51.2,
// 4 -> 47.5, 8 -> 45.5, 16 -> 47.1 ms per iteration)
#ifndef KNB_TCX_CHAINS
#define KNB_TCX_CHAINS 8
#endif
template <int J0, int W, int E = 0>
__device__ __forceinline__ void pack_keys(const uint32_t (&v)[16], uint32_t mask, int (&key)[W]) {
  if constexpr (E < W) {
    key[E] = pack_key<J0 + E>(v[E], mask);
    pack_keys<J0, W, E + 1>(v, mask, key);
  }
}

// the smallest key of W and the second smallest (min over key - gm - 1 as unsigned:
// gm itself wraps), trees of 3-input mins and four independent chains
template <int W>
__device__ __forceinline__ void min2_keys(const int (&key)[W], int& gm, int& g2) {
  if constexpr (W == 16) {
    const int m0 = min(key[0], min(key[1], key[2])), m1 = min(key[3], min(key[4], key[5]));
    const int m2 = min(key[6], min(key[7], key[8])), m3 = min(key[9], min(key[10], key[11]));
    const int m4 = min(key[12], min(key[13], key[14]));
    gm = min(min(m0, min(m1, m2)), min(m3, min(m4, key[15])));
  } else {
    const int m0 = min(key[0], min(key[1], key[2])), m1 = min(key[3], min(key[4], key[5]));
    gm = min(min(m0, m1), min(key[6], key[7]));
  }
  const uint32_t off = (uint32_t)(-gm - 1);
  constexpr int CH = KNB_TCX_CHAINS;  // independent add-min chains
  uint32_t c[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = 0xFFFFFFFFu;
#pragma unroll
  for (int e = 0; e < W; ++e) c[e % CH] = min((uint32_t)key[e] + off, c[e % CH]);
  uint32_t cm = c[0];
#pragma unroll
  for (int i = 1; i < CH; ++i) cm = min(cm, c[i]);
  g2 = (int)((uint32_t)gm + 1u + cm);
}

template <int XD, int NG, int LAST>
__global__ void __maxnreg__(KNB_TCX_REGS)
    mti_tc_kernel(const __grid_constant__ CUtensorMap tmX, const MtiTcArgs a) {
  constexpr int N = 16 * NG;
  using G = Geo<XD>;
  pdl_enter();
  if (!a.dbg && a.ctrl->stop && !a.ctrl->ignore_stop) return;  // (the score dump ignores the stop flag)
  if (a.gate && a.ctrl->mti_choice != 1) return;  // the compacted MTI kernel runs this iteration
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int k = a.k;
  const TcxSmem<XD> L(k, N, a.nx);
  const int NX = L.NX;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + NX;
  uint64_t* a_full = bars + 2 * NX;
  uint64_t* a_empty = a_full + NA;
  uint64_t* t_full = a_empty + NA;
  uint64_t* t_empty = t_full + NACC;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(t_empty + NACC);
  double* crow = reinterpret_cast<double*>(sm + L.crow);
  double2* hd = reinterpret_cast<double2*>(sm + L.hd);
  float* ebuf = reinterpret_cast<float*>(sm + L.ebuf);  // per tile (& 7): the rows' certificate bound E
  const bool work = (int)blockIdx.x < a.gtc;  // extra CTAs (grid shared with other kernels) only write zeros

  // ---- setup: B operand image, exact-recipe centroid copy, {drift, half_min}, sums
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.bimg);
    uint4* dst = reinterpret_cast<uint4*>(sm + L.b0);
    for (int i = tid; i < G::B_NCH * N * 8; i += THREADS) dst[i] = src[i];
    for (int i = tid; i < k * XD; i += THREADS) {
      const int j = i / XD, e = i - j * XD;
      crow[j * crow_stride<XD>() + e] = a.means[i];
    }
    for (int j = tid; j < k; j += THREADS) hd[j] = make_double2(a.drift[j], a.half_min[j]);
    // (the CTA's partial sums, counts and sq are written by mti_tc_delta_kernel)
    fence_proxy_async();  // generic-proxy writes of B -> visible to the tensor core
  }
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(x_full + s, 1);
      mbar_init(x_empty + s, 4);  // the four epilogue warps of the tile's group
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(a_full + s, NCONV);
      mbar_init(a_empty + s, 1);
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(t_full + b, 1);
      mbar_init(t_empty + b, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1 && work) {
    tmem_alloc(tslot, TALLOC);
    tmem_relinquish();
  }
  if (warp == 0 && lane == 0 && work) prefetch_tmap(&tmX);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = work ? *tslot : 0u;
  const int ntiles = work ? (int)((a.n + XT - 1) / XT) : 0;
  const int t0 = blockIdx.x, tstep = a.gtc;
  const int mine = ntiles > t0 ? (ntiles - t0 + tstep - 1) / tstep : 0;  // tiles of this CTA

  // epilogue-side counters (reduced at the end)
  // (32-bit: per thread at most tiles x k; reassignments are counted by mti_tc_delta_kernel)
  unsigned skips = 0, computed = 0, flagged = 0;

  if (warp == 0) {
    if (lane == 0) {
      ProfClock pc;
      pc.start();
      // the f64 tiles, each pulled into L2 PF tiles before its TMA load
      for (int i = 0; i < PF && i < mine; ++i)
        for (int t = 0; t < G::NTMA; ++t) tma_prefetch_l2_2d(&tmX, t * 16, (t0 + i * tstep) * XT);
      int s = 0, ph = 0;
      for (int i = 0; i < mine; ++i) {
        if (i + PF < mine)
          for (int t = 0; t < G::NTMA; ++t) tma_prefetch_l2_2d(&tmX, t * 16, (t0 + (i + PF) * tstep) * XT);
        mbar_sleep(x_empty + s, ph ^ 1);
        pc.lap(0);
        mbar_arrive_expect_tx(x_full + s, G::X_TILE);
        for (int t = 0; t < G::NTMA; ++t)
          tma_load_2d(sm + L.x0 + s * G::X_TILE + t * CH, &tmX, x_full + s, t * 16, (t0 + i * tstep) * XT);
        pc.lap(1);
        if (++s == NX) { s = 0; ph ^= 1; }
      }
      pc.flush(0, 2, true);
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(XT, N);
      const uint32_t b0 = smem_u32(sm + L.b0), b1 = b0 + N * 128;
      ProfClock pc;
      pc.start();
      int b = 0, bph = 0;  // accumulator buffer of tile i (= its epilogue group) and its phase
      for (int i = 0; i < mine; ++i) {
        const int sa = i % NA;
        mbar_sleep(a_full + sa, (i / NA) & 1);
        pc.lap(0);
        mbar_sleep(t_empty + b, bph ^ 1);
        pc.lap(1);
        tc_fence_after();
        const uint32_t dt = tmem + b * TCOLS;
        const uint32_t A0 = smem_u32(sm + L.a0 + sa * G::A_TILE);
        if constexpr (XD == 8) {
          // x_hi.c_hi, x_lo.c_hi, x_hi.c_lo, [1, 1, xn2_hi, xn2_lo].[cn2_hi, cn2_lo, 1, 1]
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b0 + ks * 32), idesc, ks > 0);
        } else if constexpr (XD == 16) {
          const uint32_t AC = A0 + CH;
          // (x_hi | x_lo) . (c_hi | c_hi)
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b0 + ks * 32), idesc, ks > 0);
          // x_hi . c_lo
#pragma unroll
          for (int ks = 0; ks < 2; ++ks)
            umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b1 + ks * 32), idesc, 1);
          // [1, 1, xn2_hi, xn2_lo] . [cn2_hi, cn2_lo, 1, 1]
          umma_tf32(dt, umma_desc_sw128(AC), umma_desc_sw128(b1 + 2 * 32), idesc, 1);
        } else {
          const uint32_t A1 = A0 + CH, AC = A0 + 2 * CH, b2 = b1 + N * 128;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // x_hi . c_hi
            umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b0 + ks * 32), idesc, ks > 0);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // x_lo . c_hi
            umma_tf32(dt, umma_desc_sw128(A1 + ks * 32), umma_desc_sw128(b0 + ks * 32), idesc, 1);
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)  // x_hi . c_lo
            umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b1 + ks * 32), idesc, 1);
          umma_tf32(dt, umma_desc_sw128(AC), umma_desc_sw128(b2), idesc, 1);
        }
        umma_commit(a_empty + sa);
        umma_commit(t_full + b);
        pc.lap(2);
        if (++b == NACC) { b = 0; bph ^= 1; }
      }
      pc.flush(2, 3, true);
    }
  } else if (warp < W_EPI) {
    // ------------------------------------------------------------ converters
    const int r0 = (warp - W_CONV) * 32 + lane;
    ProfClock pc;
    pc.start();
    int s = 0, ph = 0;
    for (int i = 0; i < mine; ++i) {
      const int sa = i % NA;
      mbar_sleep(x_full + s, ph);
      pc.lap(0);
      mbar_sleep(a_empty + sa, ((i / NA) & 1) ^ 1);
      pc.lap(1);
      const unsigned char* xs = sm + L.x0 + s * G::X_TILE;
      unsigned char* A0 = sm + L.a0 + sa * G::A_TILE;
#pragma unroll
      for (int rr = 0; rr < ((KNB_TCX_ABL & 1) ? 0 : 4 / NCONV); ++rr) {
      const int r = r0 + rr * 32 * NCONV;
      float n0 = 0.0f, n1 = 0.0f;
      auto put = [&](unsigned char* base, int c, float v0, float v1, float v2, float v3) {
        *reinterpret_cast<float4*>(base + swz(r, c)) = make_float4(v0, v1, v2, v3);
      };
      if constexpr (XD <= 16) {
        // all loads and conversions first, then the operand stores (measured on c4: the
        // interleaved form below runs the pass at 52 instead of 45 ms -- the converters are
        // on the MMA's critical path); rows of 32 take the interleaved form (registers)
        float hi[XD], lo[XD];
#pragma unroll
        for (int q = 0; q < XD / 2; ++q) {
          const double2 v = *reinterpret_cast<const double2*>(xs + xoff<XD>(r, q));
          const float f0 = __double2float_rn(v.x), f1 = __double2float_rn(v.y);
          hi[2 * q] = tf32_trunc(f0);
          hi[2 * q + 1] = tf32_trunc(f1);
          lo[2 * q] = f0 - hi[2 * q];
          lo[2 * q + 1] = f1 - hi[2 * q + 1];
          n0 = fmaf(f0, f0, n0);
          n1 = fmaf(f1, f1, n1);
        }
#pragma unroll
        for (int c = 0; c < XD / 4; ++c) {
          put(A0, c, hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
          if constexpr (XD == 8) {
            put(A0, c + 2, lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
            put(A0, c + 4, hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
          } else {
            put(A0, c + 4, lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
          }
        }
      } else {
        // four dims at a time: f32, the TF32 head (truncated), the f32 remainder, the norm
#pragma unroll
        for (int c = 0; c < XD / 4; ++c) {
          const double2 v0 = *reinterpret_cast<const double2*>(xs + xoff<XD>(r, 2 * c));
          const double2 v1 = *reinterpret_cast<const double2*>(xs + xoff<XD>(r, 2 * c + 1));
          const float f0 = __double2float_rn(v0.x), f1 = __double2float_rn(v0.y);
          const float f2 = __double2float_rn(v1.x), f3 = __double2float_rn(v1.y);
          const float h0 = tf32_trunc(f0), h1 = tf32_trunc(f1), h2 = tf32_trunc(f2), h3 = tf32_trunc(f3);
          n0 = fmaf(f0, f0, n0);
          n1 = fmaf(f1, f1, n1);
          n0 = fmaf(f2, f2, n0);
          n1 = fmaf(f3, f3, n1);
          put(A0, c, h0, h1, h2, h3);
          put(A0 + CH, c, f0 - h0, f1 - h1, f2 - h2, f3 - h3);
        }
      }
      const float xn2 = n0 + n1;  // (a row constant: its rounding shifts every D~_j alike)
      const float xh = tf32_trunc(xn2), xl = xn2 - xh;
      {
        unsigned char* AC = XD == 8 ? A0 : A0 + (Geo<XD>::A_NCH - 1) * CH;
        const int q0 = XD == 8 ? 6 : 0;
        put(AC, q0, 1.0f, 1.0f, xh, xl);
        put(AC, q0 + 1, 0.0f, 0.0f, 0.0f, 0.0f);
      }
      // ||x||^2 for the epilogue's certificate bound E(x) (with a relative margin: xn2
      // carries < 2^-20 relative error)
      ebuf[(i & (NE - 1)) * XT + r] = xn2 * (1.0f + 0x1p-12f);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + sa);
      pc.lap(2);
      if (++s == NX) { s = 0; ph ^= 1; }
    }
    pc.flush(5, 3, warp == W_CONV && lane == 0);
  } else {
    // ------------------------------------------------------------ epilogue
    // two warpgroups: group g takes the CTA's tiles i with i % 2 == g (and TMEM buffer g);
    // warp q of either group owns rows [32q, 32q + 32) of its tiles; moved rows go to the
    // accumulating warp as records (the sums take them in tile order, row order)
    const int grp = (warp - W_EPI) >> 2;
    const int q = warp & 3;          // TMEM lane quarter
    const int r = q * 32 + lane;     // row within the tile
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    const float cmaxf = __double2float_ru(sqrt(a.ctrl->cmax2));
    const float cmax2f = __double2float_ru(a.ctrl->cmax2);
    auto state = [&](int i, int& av, double& uv) {
      const long long row = (long long)(t0 + i * tstep) * XT + r;
      const bool ok = i < mine && row < a.n;
      av = ok ? a.assign[row] : -1;
      uv = ok ? a.upper[row] : 0.0;
    };
    int pa;
    double pu;
    state(grp, pa, pu);
    ProfClock pc;
    pc.start();
    int s = grp % NX, ph = grp / NX;  // f64 stage of tile i and its phase
    for (int i = grp; i < mine; i += NGRP) {
      const long long row = (long long)(t0 + i * tstep) * XT + r;
      const int orig = pa;
      const double u0 = pu;
      state(i + NGRP, pa, pu);
      const bool valid = orig >= 0;
      const int oc = valid ? orig : 0;
      const double2 dh = hd[oc];                  // {drift, half_min}
      const double u = u0 + dh.x;                 // inflate (u + 0.0 == u)
      const bool skip = valid && u <= dh.y;       // clause 1
      const bool live = a.dbg ? valid : (valid && !skip);
      double x[XD];
      if (!a.dbg) {
        skips += skip ? 1 : 0;
        if (skip && dh.x != 0.0) {  // the inflated bound is the skipped row's state
          a.upper[row] = u;
          a.tight[row] = 0;
        }
      }
      pc.lap(5);
      const int tb = i % NACC;  // the tile's accumulator buffer
      const uint32_t tl = tq + (uint32_t)(tb * TCOLS);
      mbar_sleep(t_full + tb, (uint32_t)((i / NACC) & 1));
      pc.lap(0);
      tc_fence_after();
      const unsigned lmask = __ballot_sync(0xffffffffu, live);
      int k1 = 0x7fffffff, k2 = 0x7fffffff;
      if (lmask) {
        if (a.dbg) {
          uint32_t v[16];
          for (int g = 0; g < NG; ++g) {
            tmem_ld<16>(tl + 16 * g, v);
            tmem_wait_ld();
            if (valid) {
              float* o = a.dbg + row * N + 16 * g;
#pragma unroll
              for (int e = 0; e < 16; ++e) o[e] = __uint_as_float(v[e]);
            }
          }
        } else {
          // per 16-column group: keys, the group's smallest key and second smallest
          // (trees of 3-input mins; the column rides in the key's low 7 bits); the last
          // group reads only LAST columns (k <= 16 (NG - 1) + LAST)
          const uint32_t kmask = a.kmask;  // 0xFFFFFF80, opaque to ptxas: the column stays the immediate
          int gmv[NG], g2v[NG];
          constexpr int GB = NG <= KNB_TCX_GB ? NG : KNB_TCX_GB;  // groups per TMEM batch
          uint32_t v[GB][16];
          auto group = [&](auto gc, const uint32_t(&vv)[16]) {
            constexpr int g = decltype(gc)::value;
            constexpr int W = g == NG - 1 ? LAST : 16;
            int key[W];
            pack_keys<16 * g, W>(vv, kmask, key);
            int gm, g2;
            min2_keys<W>(key, gm, g2);
            gmv[g] = gm;
            g2v[g] = g2;
          };
          auto load = [&](auto gc, uint32_t(&vv)[16]) {
            constexpr int g = decltype(gc)::value;
            tmem_ld<g == NG - 1 ? LAST : 16>(tl + 16 * g, vv);
          };
          // batches of GB groups: load, one wait, reduce (bounds the registers held)
          constexpr int NB = (NG + GB - 1) / GB;
          for_groups<NB>([&](auto bc) {
            constexpr int B0 = decltype(bc)::value * GB;
            constexpr int NBG = NG - B0 < GB ? NG - B0 : GB;
            for_groups<NBG>([&](auto gc) {
              load(std::integral_constant<int, B0 + decltype(gc)::value>{}, v[decltype(gc)::value]);
            });
            tmem_wait_ld();
            for_groups<NBG>([&](auto gc) {
              group(std::integral_constant<int, B0 + decltype(gc)::value>{}, v[decltype(gc)::value]);
            });
          });
#pragma unroll
          for (int g = 0; g < NG; ++g) k1 = min(k1, gmv[g]);
#pragma unroll
          for (int g = 0; g < NG; ++g) k2 = min(k2, gmv[g] == k1 ? g2v[g] : gmv[g]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty + tb);
      pc.lap(1);

      pc.lap(2);
      unsigned mm = 0;
      int win = k1 & 127;
      if (!a.dbg && lmask && !(KNB_TCX_ABL & 2)) {
        bool cert = false;
        if (live) {
          // the certificate's bound E(x) (f32 with a relative margin)
          const float xnb = ebuf[(i & (NE - 1)) * XT + r];
          const float E = (0x1p-20f * (G::C1 * sqrtf(xnb) * cmaxf + G::C2 * (xnb + cmax2f)) +
                           (8.0f * XD + 32.0f) * 0x1p-53f * (xnb + cmax2f)) * (1.0f + 0x1p-10f);
          const float m1 = __int_as_float(k1 & ~127), m2 = __int_as_float(k2 & ~127);
          // key slack (< 2^-16 relative each) and the f32 rounding of this test
          cert = (m2 - m1) > 2.0f * E + 0x1p-15f * (fabsf(m1) + fabsf(m2)) && win < k;
          if (KNB_TCX_ABL & 16) cert = true;
        }
        {
          // the f64 rows of this tile from the stage (landed before the converters ran; the
          // wait only orders this warp's reads after the TMA)
          mbar_sleep(x_full + s, (uint32_t)ph);
          const unsigned char* xs = sm + L.x0 + s * G::X_TILE;
          if (XD != 32 && live) {  // (XD = 32 reads its row from the stage in the recipe)
#pragma unroll
            for (int c = 0; c < XD / 2; ++c) {
              const double2 vv = *reinterpret_cast<const double2*>(xs + xoff<XD>(r, c));
              x[2 * c] = vv.x;
              x[2 * c + 1] = vv.y;
            }
          }
        }
        double nd = 0.0;
        // uncertified rows go to the rerank queue (mti_tc_rerank_kernel re-ranks them after
        // the pass: a warp stalled on one row's k exact distances here would hold up the
        // tile pipeline); beyond the queue's capacity the whole warp re-ranks each one here
        // with the exact recipe, scan_block's order -- the current centroid first, then
        // ascending ids, switch on strict < of the sqrt'ed distances (pruning.py:174-203)
        unsigned fl = __ballot_sync(0xffffffffu, live && !cert);
        bool queued = false;
        if (fl) {
          if (lane == 0) flagged += __popc(fl);
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(a.rq_count, (unsigned long long)__popc(fl));
          base = __shfl_sync(0xffffffffu, base, 0);
          if ((fl >> lane) & 1u) {
            const unsigned long long slot = base + __popc(fl & ((1u << lane) - 1u));
            if (slot < (unsigned long long)a.rq_cap) {
              reinterpret_cast<longlong2*>(a.rq)[slot] = make_longlong2(row, (long long)orig);
              queued = true;
            }
          }
          fl = __ballot_sync(0xffffffffu, (live && !cert) && !queued);
        }
        while (fl) {
          const int f = __ffs(fl) - 1;
          fl &= fl - 1;
          const int fo = __shfl_sync(0xffffffffu, orig, f);
          // row f's values from the stage (a shared-memory broadcast), the centroids in place
          double xf[XD];
          {
            const unsigned char* xsf = sm + L.x0 + s * G::X_TILE;
#pragma unroll
            for (int c = 0; c < XD / 2; ++c) {
              const double2 vv = *reinterpret_cast<const double2*>(xsf + xoff<XD>(q * 32 + f, c));
              xf[2 * c] = vv.x;
              xf[2 * c + 1] = vv.y;
            }
          }
          double bd = CUDART_INF;
          int bp = 0x7fffffff, bj = 0;
          for (int j = lane; j < k; j += 32) {
            const double dj = sqrt(exact_sq_fixed<XD>(xf, crow + j * crow_stride<XD>()));
            const int pj = j == fo ? -1 : j;
            if (dj < bd || (dj == bd && pj < bp)) { bd = dj; bp = pj; bj = j; }
          }
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (od < bd || (od == bd && op < bp)) { bd = od; bp = op; bj = oj; }
          }
          if (lane == f) {
            win = bj;
            nd = bd;
          }
        }
        if (live && cert && !(KNB_TCX_ABL & 4)) {
          if constexpr (XD == 32) {  // (row and centroid straight from shared memory: registers)
            nd = sqrt(exact_sq_fixed<XD>(StageRow<XD>{sm + L.x0 + s * G::X_TILE, r}, crow + win * crow_stride<XD>()));
          } else {
            double cw[XD];
            load_crow<XD>(crow, win, cw);
            nd = sqrt(exact_sq_fixed<XD>(x, cw));
          }
        }
        const bool moved = live && !queued && win != orig;
        if (live && !queued && !(KNB_TCX_ABL & 8)) {
          a.upper[row] = nd;
          a.tight[row] = 1;
          if (moved) a.assign[row] = win;
        }
        if (lane == 0) computed += (unsigned)(__popc(lmask) * k);
        mm = __ballot_sync(0xffffffffu, moved);
      }
      // the stage goes back to the producer; the tile's moved rows go to global memory
      // for mti_tc_delta_kernel: a bit mask per row quarter and each moved row's old id
      __syncwarp();
      if (lane == 0) mbar_arrive(x_empty + s);
      if (!a.dbg) {
        unsigned char* rb = a.recs + (size_t)(t0 + i * tstep) * TC_REC;
        if ((mm >> lane) & 1u) rb[16 + r] = (unsigned char)orig;
        if (lane == 0) reinterpret_cast<unsigned*>(rb)[q] = mm;
      }
      s += NGRP;
      while (s >= NX) {
        s -= NX;
        ph ^= 1;
      }
      pc.lap(3);
    }
    pc.flush(8, 6, warp == W_EPI && lane == 0);
  }
  __syncthreads();
  if (warp == 1 && work) {
    tc_fence_after();
    tmem_dealloc(tmem, TALLOC);
  }

  // CTA partial: the scalars (mti_tc_delta_kernel writes the sums, counts and sq)
  const long long Lg = acc_len(k, XD);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  const int kk = k * (XD + 2);
  __shared__ long long red[4 * NGRP][4];
  if (warp >= W_EPI) {
    const long long c0 = 0, c1 = warp_sum_ll((long long)skips), c2 = warp_sum_ll((long long)computed),
                    c3 = warp_sum_ll((long long)flagged);
    if (lane == 0) {
      red[warp - W_EPI][0] = c0;
      red[warp - W_EPI][1] = c1;
      red[warp - W_EPI][2] = c2;
      red[warp - W_EPI][3] = c3;
    }
  }
  __syncthreads();
  if (tid == 0) {
    long long tot[4] = {0, 0, 0, 0};
    if (work)
      for (int w = 0; w < 4 * NGRP; ++w)
        for (int c = 0; c < 4; ++c) tot[c] += red[w][c];
    double* sc = out + kk;
    for (int c = 0; c < NSCAL; ++c) sc[c] = 0.0;
    sc[S_REASSIGNED] = 0.0;  // (mti_tc_delta_kernel counts the moved rows from the records)
    sc[S_SKIPS] = (double)tot[1];
    sc[S_COMPUTED] = (double)tot[2];
    if (a.counters && tot[3]) atomicAdd(a.counters, (unsigned long long)tot[3]);
  }
}

// The running-sum deltas of the rows the tcgen05 MTI pass moved (engine.py:345-353):
// +x, +1, +||x||^2 to the new cluster, the same off the old one, from the pass's per-tile
// records (a moved-row bit mask per row quarter, the old ids).  CTA b takes a contiguous
// range of tiles and walks it in chunks of dc tiles (256, or 128 when k is large): thread
// t holds tile t's four mask words -- the next chunk's are loaded while the current one
// is summed -- and an exclusive scan in shared memory makes the j-th moved row of the
// chunk a binary search away; the moved rows are cut into batches of 32 and batch m goes
// to warp m % DW.  A warp copies a batch into one of its two staging slots with cp.async
// -- eight lanes per row, four rows per instruction (whole 128-byte lines, 16-byte chunks
// swizzled by row so the per-row reads are conflict-free), plus each row's new id and the
// word holding its old id -- and issues the NEXT batch's copies before it adds the current
// one, in row order, to its private sums (lanes 0-15 the dims, lane 16 the counts, lane 17
// ||x||^2, the row's exact-recipe sum of squares).  The CTA adds its warps' sums in warp
// order into partial b: deterministic for a fixed grid.  The CTA also counts the moved
// rows (the pass's reassignments).
constexpr int DW = 8;           // warps per CTA

__host__ __device__ inline int delta_chunk(int k) { return k <= 112 ? 256 : 128; }

template <int XD>
size_t delta_smem(int k) {
  return (size_t)DW * k * (XD + 2) * sizeof(double)   // private sums
         + (size_t)DW * 2 * 32 * XD * sizeof(double)  // staging rows
         + (size_t)DW * 2 * 32 * sizeof(double)       // their ||x||^2
         + (size_t)DW * 2 * 32 * sizeof(int2)         // new / old ids
         + (size_t)8 * delta_chunk(k) * sizeof(unsigned);  // mask words + prefixes
}

// staging offset (doubles) of element e of row rr: 16-byte chunks swizzled by the row
template <int XD>
__device__ __forceinline__ int sw_off(int rr, int e) {
  return rr * XD + ((((e >> 1) ^ rr) & (XD / 2 - 1)) << 1) + (e & 1);
}

template <int XD>
__global__ void __launch_bounds__(DW * 32, 1) mti_tc_delta_kernel(const MtiTcArgs a) {
  pdl_enter();
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  if (a.gate && a.ctrl->mti_choice != 1) return;
  extern __shared__ double dsm[];
  const int k = a.k, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int dc = delta_chunk(k);
  const int per = k * (XD + 2);
  double* acc = dsm + (size_t)warp * per;
  double* cnt = acc + k * XD;
  double* sqa = cnt + k;
  double* stg = dsm + (size_t)DW * per + (size_t)warp * 2 * 32 * XD;            // [slot][row][16]
  double* sqs = dsm + (size_t)DW * per + (size_t)DW * 2 * 32 * XD + warp * 64;  // [slot][row]
  int2* ids = reinterpret_cast<int2*>(dsm + (size_t)DW * per + (size_t)DW * 2 * 32 * XD + DW * 64) + warp * 64;
  unsigned* mwd = reinterpret_cast<unsigned*>(reinterpret_cast<int2*>(dsm + (size_t)DW * per +
                                                                       (size_t)DW * 2 * 32 * XD + DW * 64) + DW * 64);
  int* wpre = reinterpret_cast<int*>(mwd + 4 * dc);  // exclusive prefix of the words' popcounts
  __shared__ int wtot[DW];
  __shared__ double dummy[DW];  // the idle lanes' target
  for (int e = lane; e < per; e += 32) acc[e] = 0.0;
  __syncwarp();
  const long long T = (a.n + XT - 1) / XT;
  const long long lo = T * blockIdx.x / gridDim.x, hi = T * (blockIdx.x + 1) / gridDim.x;
  long long moved = 0;
  const uint32_t stg_s = smem_u32(stg), ids_s = smem_u32(ids);
  auto masks = [&](long long c0) {  // tile c0 + tid's four words
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tid < dc && c0 + tid < hi) v = *reinterpret_cast<const uint4*>(a.recs + (size_t)(c0 + tid) * TC_REC);
    return v;
  };
  uint4 mk = masks(lo);

  for (long long c0 = lo; c0 < hi; c0 += dc) {
    const int run = __popc(mk.x) + __popc(mk.y) + __popc(mk.z) + __popc(mk.w);
    if (tid < dc) reinterpret_cast<uint4*>(mwd)[tid] = mk;
    int inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    int wbase = 0, M = 0;
    for (int w = 0; w < DW; ++w) {
      wbase += w < warp ? wtot[w] : 0;
      M += wtot[w];
    }
    if (tid < dc) {
      int p = wbase + inc - run;
      wpre[4 * tid] = p;
      p += __popc(mk.x);
      wpre[4 * tid + 1] = p;
      p += __popc(mk.y);
      wpre[4 * tid + 2] = p;
      p += __popc(mk.z);
      wpre[4 * tid + 3] = p;
    }
    __syncthreads();
    moved += M;
    mk = masks(c0 + dc);  // the next chunk's words, in flight during this one

    // batch m of the chunk (its moved rows [32m, 32m + 32)) into staging slot sl; returns
    // the batch's rows (0: none) and, in lane j, row j's old-id byte position.  Always
    // commits one cp.async group.
    auto fetch = [&](int m, int sl, int& sub) -> int {
      const int n = 32 * m < M ? min(32, M - 32 * m) : 0;
      long long row = 0;
      if (lane < n) {
        const int J = 32 * m + lane;
        int w = 0;  // the last word whose prefix <= J
        for (int step = 2 * dc; step; step >>= 1)
          if (w + step < 4 * dc && wpre[w + step] <= J) w += step;
        const int bit = __fns(mwd[w], 0, J - wpre[w] + 1);
        const long long t = c0 + (w >> 2);
        const int r = (w & 3) * 32 + bit;
        row = t * XT + r;
        sub = r & 3;
        const uint32_t id = ids_s + (uint32_t)((sl * 32 + lane) * sizeof(int2));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(id), "l"(a.assign + row) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(id + 4),
                     "l"(a.recs + (size_t)t * TC_REC + 16 + (r & ~3)) : "memory");
      }
      // XD / 2 lanes per row: lane l copies 16-byte chunk l % (XD / 2) of row
      // (64 / XD) i + l / (XD / 2): whole rows per instruction
      constexpr int CPR = XD / 2, RPI = 32 / CPR;
#pragma unroll
      for (int i = 0; i < 32 / RPI; ++i) {
        const int rr = RPI * i + lane / CPR;
        const long long rw = __shfl_sync(0xffffffffu, row, rr);
        if (rr < n)
          cp_async16_s(stg_s + (uint32_t)((sl * 32 * XD + sw_off<XD>(rr, 2 * (lane % CPR))) * sizeof(double)),
                       a.X + rw * XD + 2 * (lane % CPR));
      }
      cp_async_commit();
      return n;
    };
    int m = warp, sl = 0, sub = 0, nsub = 0;
    int n = fetch(m, 0, sub);
    while (n > 0) {
      const int nn = fetch(m + DW, sl ^ 1, nsub);  // the next batch's copies are in flight during the additions
      cp_async_wait_1();
      __syncwarp();
      const double* sg = stg + sl * 32 * XD;
      double* sq = sqs + sl * 32;
      int2* id = ids + sl * 32;
      if (lane < n) {
        double x[XD];
#pragma unroll
        for (int e = 0; e < XD; e += 2) {
          const double2 v = *reinterpret_cast<const double2*>(sg + sw_off<XD>(lane, e));
          x[e] = v.x;
          x[e + 1] = v.y;
        }
        sq[lane] = exact_sq_fixed<XD>(x, Zero{});
        const int2 v = id[lane];
        id[lane].y = (v.y >> (8 * sub)) & 0xFF;  // the old id's byte
      }
      __syncwarp();
      // per lane and pass: the sum it owns is base[cluster * stride] (value vi = 32 pass +
      // lane: the dims acc[c][vi], then cnt[c], sqa[c]; idle lanes a dummy slot) and the
      // value it adds (the count's is 1).  No branches: every lane runs the same
      // read-modify-writes.  Two consecutive rows whose four clusters are distinct (the
      // usual case) are read, added and written together; otherwise one after the other --
      // the same order of additions per sum either way.
      const int to_l = id[lane].x, fr_l = id[lane].y;
#pragma unroll
      for (int pass = 0; pass < (XD + 2 + 31) / 32; ++pass) {
        const int vi = 32 * pass + lane;
        double* base = vi < XD ? acc + vi : (vi == XD ? cnt : (vi == XD + 1 ? sqa : dummy + warp));
        const int stride = vi < XD ? XD : (vi <= XD + 1 ? 1 : 0);
        auto val = [&](int j) { return vi < XD ? sg[sw_off<XD>(j, vi)] : (vi == XD + 1 ? sq[j] : 1.0); };
        int j = 0;
        while (j < n) {
          const int t0 = __shfl_sync(0xffffffffu, to_l, j), f0 = __shfl_sync(0xffffffffu, fr_l, j);
          const int j1 = j + 1 < n ? j + 1 : j;
          const int t1 = __shfl_sync(0xffffffffu, to_l, j1), f1 = __shfl_sync(0xffffffffu, fr_l, j1);
          if (j + 1 < n && t1 != t0 && t1 != f0 && f1 != t0 && f1 != f0) {
            const double v0 = val(j), w0 = val(j + 1);
            double* a0 = base + t0 * stride;
            double* b0 = base + f0 * stride;
            double* a1 = base + t1 * stride;
            double* b1 = base + f1 * stride;
            const double ra0 = *a0, rb0 = *b0, ra1 = *a1, rb1 = *b1;
            *a0 = ra0 + v0;
            *b0 = rb0 - v0;
            *a1 = ra1 + w0;
            *b1 = rb1 - w0;
            j += 2;
          } else {
            const double v0 = val(j);
            double* a0 = base + t0 * stride;
            double* b0 = base + f0 * stride;
            const double ra0 = *a0, rb0 = *b0;
            *a0 = ra0 + v0;
            *b0 = rb0 - v0;
            j += 1;
          }
        }
      }
      __syncwarp();
      n = nn;
      sub = nsub;
      m += DW;
      sl ^= 1;
    }
    cp_async_wait_all();
    __syncthreads();  // (the next chunk overwrites the words and prefixes)
  }
  double* out = a.partials + (long long)blockIdx.x * acc_len(k, XD);
  for (int e = tid; e < per; e += DW * 32) {
    double v = 0.0;
    for (int w = 0; w < DW; ++w) v += dsm[(size_t)w * per + e];
    out[e] = v;
  }
  if (tid == 0) out[per + S_REASSIGNED] = (double)moved;
}

// The uncertified rows of the pass (the queue the epilogue filled), one row per lane: f64
// norm-form scores ||x||^2 + ||c_j||^2 - 2 x.c_j over all k centroids (the centroid read is
// a shared-memory broadcast), keeping the three smallest; then the exact recipe only for
// those within twice the certificate tolerance (8d + 32) 2^-53 (||x||^2 + max ||c||^2) of
// the smallest score -- every other centroid is strictly farther for the reference too --
// (a row with a third centroid inside the window re-scores the whole window), ranked by
// (sqrt'ed distance, id with the current centroid first): scan_block's choice, which keeps
// the current centroid on an exact tie and otherwise the lowest id (pruning.py:174-203).
// Then the row's MTI state, and for a moved row its bit and old id in the tile's record
// (the epilogue left both out), so mti_tc_delta_kernel sums it like any other moved row.
template <int XD>
__global__ void __launch_bounds__(256) mti_tc_rerank_kernel(const MtiTcArgs a) {
  pdl_enter();
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  if (a.gate && a.ctrl->mti_choice != 1) return;
  extern __shared__ double crs[];  // k rows of crow_stride: the centroid, then ||c||^2
  const int k = a.k;
  for (int i = threadIdx.x; i < k * XD; i += blockDim.x) {
    const int j = i / XD, e = i - j * XD;
    crs[j * crow_stride<XD>() + e] = a.means[i];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double c2 = 0.0;
#pragma unroll
    for (int e = 0; e < XD; ++e) c2 = fma(crs[j * crow_stride<XD>() + e], crs[j * crow_stride<XD>() + e], c2);
    crs[j * crow_stride<XD>() + XD] = c2;
  }
  __syncthreads();
  const unsigned long long cnt = *a.rq_count;
  const long long m = cnt < (unsigned long long)a.rq_cap ? (long long)cnt : a.rq_cap;
  const double cmax2 = a.ctrl->cmax2;
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  for (long long e0 = (long long)blockIdx.x * blockDim.x; e0 < m; e0 += nthreads) {
    const long long e = e0 + threadIdx.x;
    if (e >= m) break;  // (nothing below synchronises)
    const longlong2 q = reinterpret_cast<const longlong2*>(a.rq)[e];
    const long long row = q.x;
    const int fo = (int)q.y;
    double x[XD];
    const double2* xr = reinterpret_cast<const double2*>(a.X + row * XD);
#pragma unroll
    for (int c = 0; c < XD / 2; ++c) {
      const double2 v = __ldg(xr + c);
      x[2 * c] = v.x;
      x[2 * c + 1] = v.y;
    }
    double xn2 = 0.0;
#pragma unroll
    for (int c = 0; c < XD; ++c) xn2 = fma(x[c], x[c], xn2);
    auto score = [&](int j) {
      const double2* cj = reinterpret_cast<const double2*>(crs + j * crow_stride<XD>());
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
      for (int c = 0; c < XD / 2; c += 2) {
        const double2 u = cj[c], w = cj[c + 1];
        d0 = fma(x[2 * c], u.x, d0);
        d1 = fma(x[2 * c + 1], u.y, d1);
        d2 = fma(x[2 * c + 2], w.x, d2);
        d3 = fma(x[2 * c + 3], w.y, d3);
      }
      return fma(-2.0, (d0 + d1) + (d2 + d3), crs[j * crow_stride<XD>() + XD]) + xn2;
    };
    double s1 = CUDART_INF, s2 = CUDART_INF, s3 = CUDART_INF;
    int j1 = 0, j2 = 0;
    for (int j = 0; j < k; ++j) {
      const double sj = score(j);
      if (sj < s3) {
        if (sj < s2) {
          s3 = s2;
          if (sj < s1) {
            s2 = s1;
            j2 = j1;
            s1 = sj;
            j1 = j;
          } else {
            s2 = sj;
            j2 = j;
          }
        } else {
          s3 = sj;
        }
      }
    }
    const double hi_s = s1 + 2.0 * (8.0 * XD + 32.0) * 0x1p-53 * (xn2 + cmax2);
    double bd = CUDART_INF;
    int bp = 0x7fffffff, bj = 0;
    auto take = [&](int j) {
      double cj[XD];
      load_crow<XD>(crs, j, cj);
      const double dj = sqrt(exact_sq_fixed<XD>(x, cj));
      const int pj = j == fo ? -1 : j;
      if (dj < bd || (dj == bd && pj < bp)) { bd = dj; bp = pj; bj = j; }
    };
    if (s3 <= hi_s) {  // three or more in the window: all of them
      for (int j = 0; j < k; ++j)
        if (score(j) <= hi_s) take(j);
    } else {
      take(j1);
      if (s2 <= hi_s) take(j2);
    }
    a.upper[row] = bd;
    a.tight[row] = 1;
    if (bj != fo) {
      a.assign[row] = bj;
      const long long t = row / XT;
      const int r = (int)(row - t * XT);
      unsigned char* rb = a.recs + (size_t)t * TC_REC;
      rb[16 + r] = (unsigned char)fo;
      atomicOr(reinterpret_cast<unsigned*>(rb) + (r >> 5), 1u << (r & 31));
    }
  }
}

// B operand image in global memory, exactly as the kernel's shared memory holds it (Geo's
// layout for XD; the cn2 entries carry ||c_j||^2 as hi + lo, the A side's [1, 1] picks
// them up); padded rows j >= k score 2^100 (never a winner, never in a window)
template <int XD>
__global__ void mti_tc_prep_kernel(const double* __restrict__ means, int k, int N, uint4* __restrict__ bimg,
                                   unsigned long long* __restrict__ rq_count) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && rq_count) *rq_count = 0;
  constexpr int NCH = Geo<XD>::B_NCH;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < NCH * N * 8; i += gridDim.x * blockDim.x) {
    const int chunk = i / (N * 8), rem = i - chunk * N * 8, j = rem >> 3, qq = rem & 7;
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const bool real = j < k;
    // what 16-byte chunk (chunk, qq) of row j holds: -2 c_hi / -2 c_lo at dims e0.., or the
    // norm constants, or zeros
    int kind = 0, e0 = 0;  // 1: c_hi, 2: c_lo, 3: constants
    if constexpr (XD == 8) {
      if (qq < 4) { kind = 1; e0 = (qq & 1) * 4; }
      else if (qq < 6) { kind = 2; e0 = (qq - 4) * 4; }
      else if (qq == 6) kind = 3;
    } else if constexpr (XD == 16) {
      if (chunk == 0) { kind = 1; e0 = (qq & 3) * 4; }
      else if (qq < 4) { kind = 2; e0 = qq * 4; }
      else if (qq == 4) kind = 3;
    } else {
      if (chunk < 2) { kind = chunk + 1; e0 = qq * 4; }
      else if (qq == 0) kind = 3;
    }
    if (kind == 1 || kind == 2) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double c = real ? means[(long long)j * XD + e0 + m] : 0.0;
        const float ch = tf32_trunc(__double2float_rn(c));
        const float cl = tf32_rna(__double2float_rn(c - (double)ch));
        v[m] = -2.0f * (kind == 1 ? ch : cl);
      }
    } else if (kind == 3) {
      double cn2 = 0.0;
      if (real)
        for (int e = 0; e < XD; ++e) {
          const double c = means[(long long)j * XD + e];
          cn2 = fma(c, c, cn2);
        }
      const float h = real ? tf32_trunc(__double2float_rn(cn2)) : 0x1p100f;
      const float l = real ? tf32_rna(__double2float_rn(cn2 - (double)h)) : 0.0f;
      v[0] = h;
      v[1] = l;
      v[2] = 1.0f;
      v[3] = 1.0f;
    }
    const uint32_t off = (uint32_t)chunk * N * 128u + (uint32_t)j * 128u + ((uint32_t)(qq ^ (j & 7)) << 4);
    bimg[off >> 4] = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                                __float_as_uint(v[3]));
  }
}

template <int XD, int NG, int LAST>
cudaError_t launch_ng(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  const TcxSmem<XD> L(a.k, 16 * NG, a.nx);
  cudaError_t e =
      cudaFuncSetAttribute(mti_tc_kernel<XD, NG, LAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_tc_kernel<XD, NG, LAST>, dim3(grid), dim3(THREADS), L.total, s, *tm, a);
}

template <int XD, int NG>
cudaError_t launch_last(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  // the score dump reads every column; otherwise the last group reads 8 when that covers k
  if (!a.dbg && a.k <= 16 * (NG - 1) + 8) return launch_ng<XD, NG, 8>(tm, a, grid, s);
  return launch_ng<XD, NG, 16>(tm, a, grid, s);
}

template <int XD>
cudaError_t launch_xd(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  switch ((a.k + 15) / 16) {
    case 1: return launch_last<XD, 1>(tm, a, grid, s);
    case 2: return launch_last<XD, 2>(tm, a, grid, s);
    case 3: return launch_last<XD, 3>(tm, a, grid, s);
    default: break;
  }
  if constexpr (XD != 32) {  // (row width 32: k <= 32, see mti_tc_stages)
    switch ((a.k + 15) / 16) {
      case 4: return launch_last<XD, 4>(tm, a, grid, s);
      case 5: return launch_last<XD, 5>(tm, a, grid, s);
      case 6: return launch_last<XD, 6>(tm, a, grid, s);
      case 7: return launch_last<XD, 7>(tm, a, grid, s);
      case 8: return launch_last<XD, 8>(tm, a, grid, s);
      default: break;
    }
  }
  return cudaErrorInvalidValue;
}

constexpr size_t SMEM_MAX = 227 * 1024;

template <int XD>
int stages_xd(int k) {
  const int N = (k + 15) / 16 * 16;
  if (delta_smem<XD>(k) > SMEM_MAX) return 0;
  for (int nx = KNB_TCX_NXMAX; nx >= 3; --nx)
    if (TcxSmem<XD>(k, N, nx).total <= SMEM_MAX) return nx;
  return 0;
}

}  // namespace

// stages of the f64 ring that fit (0: the kernel does not apply): rows of 8, 16 or 32
// doubles, k <= 128 (row width 32: k <= 32, the delta kernel's staging and sums)
int mti_tc_stages(int d, int k) {
  if (k < 1 || k > 128) return 0;
  if (d == 8) return stages_xd<8>(k);
  if (d == 16) return stages_xd<16>(k);
  if (d == 32) return k <= 32 ? stages_xd<32>(k) : 0;
  return 0;
}

size_t mti_tc_bimg_bytes(int d, int k) {
  const int nch = d == 32 ? 3 : (d == 16 ? 2 : 1);
  return (size_t)nch * ((k + 15) / 16 * 16) * 128;
}

int mti_tc_prof(unsigned long long* out) {
  unsigned long long all[18];
  if (cudaMemcpyFromSymbol(all, g_tcx_prof, sizeof(all)) != cudaSuccess) return -1;
  for (int i = 0; i < 16; ++i) out[i] = all[i];
  out[12] = all[16];  // (profiling builds: slot 12 reports the rows the accumulating warp summed)
  static const unsigned long long z[18] = {};
  if (cudaMemcpyToSymbol(g_tcx_prof, z, sizeof(z)) != cudaSuccess) return -1;
  return KNB_TCX_PROF;
}

cudaError_t launch_mti_tc_prep(const double* means, int d, int k, void* bimg, unsigned long long* rq_count,
                               cudaStream_t s) {
  const int N = (k + 15) / 16 * 16;
  const int blocks = (3 * N * 8 + 255) / 256;
  uint4* b = reinterpret_cast<uint4*>(bimg);
  if (d == 8) mti_tc_prep_kernel<8><<<blocks, 256, 0, s>>>(means, k, N, b, rq_count);
  else if (d == 16) mti_tc_prep_kernel<16><<<blocks, 256, 0, s>>>(means, k, N, b, rq_count);
  else mti_tc_prep_kernel<32><<<blocks, 256, 0, s>>>(means, k, N, b, rq_count);
  return cudaGetLastError();
}

template <int XD>
cudaError_t rerank_xd(const MtiTcArgs& a, int grid, cudaStream_t s) {
  const size_t smem = (size_t)a.k * crow_stride<XD>() * sizeof(double);
  cudaError_t e = cudaFuncSetAttribute(mti_tc_rerank_kernel<XD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_tc_rerank_kernel<XD>, dim3(grid), dim3(256), smem, s, a);
}

cudaError_t launch_mti_tc_rerank(const MtiTcArgs& a, int grid, cudaStream_t s) {
  if (a.d == 8) return rerank_xd<8>(a, grid, s);
  if (a.d == 16) return rerank_xd<16>(a, grid, s);
  return rerank_xd<32>(a, grid, s);
}

template <int XD>
cudaError_t delta_xd(const MtiTcArgs& a, int grid, cudaStream_t s) {
  const size_t smem = delta_smem<XD>(a.k);
  cudaError_t e = cudaFuncSetAttribute(mti_tc_delta_kernel<XD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_tc_delta_kernel<XD>, dim3(grid), dim3(DW * 32), smem, s, a);
}

cudaError_t launch_mti_tc_delta(const MtiTcArgs& a, int grid, cudaStream_t s) {
  if (a.d == 8) return delta_xd<8>(a, grid, s);
  if (a.d == 16) return delta_xd<16>(a, grid, s);
  return delta_xd<32>(a, grid, s);
}

cudaError_t launch_mti_tc(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  if (a.d == 8) return launch_xd<8>(tm, a, grid, s);
  if (a.d == 16) return launch_xd<16>(tm, a, grid, s);
  if (a.d == 32) return launch_xd<32>(tm, a, grid, s);
  return cudaErrorInvalidValue;
}

}  // namespace knb
