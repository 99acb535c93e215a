// K6/K7-TC: the pruned (MTI) pass for f64 rows with d = 16 on the tcgen05 tensor
// cores, with a certified argmin (BASELINE config 4: n = 856M, d = 16, k = 100,
// where clause 1 skips almost nothing and every row is re-scored each pass).
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
// x_lo the f32 remainder, truncated by the tensor core) -- and one chain of seven
// kind::tf32 UMMAs (M = 128 rows, N = k padded to 16, K = 8 each) accumulates, in
// TMEM,
//     D~_j = (x_hi + x_lo).(-2 c_hi)  +  x_hi.(-2 c_lo)  +  ||c_j||^2  +  ||x||^2
//          ~ ||x - c_j||^2
// (the x_lo.c_lo term, ~2^-20 |x||c|, is dropped; the two norms enter through a
// constant k-step: A = [1, 1, xn2_hi, xn2_lo], B = [cn2_hi, cn2_lo, 1, 1]).
// Operand layout, K-major with the 128-byte swizzle (tc_common.cuh descriptors):
//     A chunk 0 = [x_hi(16) | x_lo(16)]      B chunk 0 = [-2c_hi(16) | -2c_hi(16)]
//     A chunk 1 = [x_hi(16) | consts(8)]     B chunk 1 = [-2c_lo(16) | consts(8)]
// k-steps 0-3 on chunk 0, 0-2 on chunk 1.
//
// Certificate.  |D~_j - D_j| <= E(x) with
//     E = 2^-20 (12 ||x|| cmax + 4 (||x||^2 + cmax^2)) + (8d + 32) 2^-53 (||x||^2 + cmax^2)
// (operand splitting: <= 3.2 * 2^-20 |x_i c_i| per product, x2 for the -2 scale; the
// f32 accumulation over seven k-steps: <= 2^-22 per step of the partial magnitudes,
// bounded by ||x||^2 + cmax^2 + 2 ||x|| cmax; the last term is the reference's own f64
// rounding of sum (x - c)^2, as in the DMMA certificate).  tests/test_gpu_mti_tc.py
// measures the worst |D~ - D| / E on adversarial inputs and requires < 1/4.
// The epilogue finds the smallest and second-smallest D~ of the row with integer
// min trees on keys = (f32 bits & ~127) | column (order-preserving for D~ >= 0; the
// column index rides in the low 7 bits, < 2^-16 relative); a row is CERTIFIED when
// second - first > 2E (+ the key slack): its winner is the reference's argmin.  Other
// rows (near ties, exact ties, tiny negative D~) are re-ranked by the whole warp with
// the exact recipe over all k centroids in scan_block's order (current centroid
// first, strict <), so the outputs are the reference's bit for bit.
//
// Kernel shape (one CTA per SM, persistent over 128-row tiles, static schedule):
//   warp 0      TMA producer: f64 row tiles (128 rows x 128 B, SWIZZLE_128B) through an
//               NX-stage ring
//   warp 1      TMEM allocation (2 x 128 columns: double-buffered accumulator) and the
//               single-thread UMMA issuer
//   warps 2-5   converters: one thread per row, f64 -> (x_hi, x_lo) TF32 operand tile
//               (two 128-byte chunks) + the norm constants, NA-stage ring
//   warps 6-9   epilogue: one thread per row (TMEM lane), key min trees, certificate,
//               warp-wide exact rerank of uncertified rows, exact bound of the winner
//               from the f64 tile, MTI state, moved rows accumulated in row order into
//               warp-private sums (deterministic), then the f64 stage is released
// HBM traffic per row: 128 B of rows + 12 B of state read + 9 B written (+4 if moved).
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"
#include "mma_common.cuh"
#include "tc_common.cuh"

namespace knb {

namespace {

constexpr int XT = 128;                        // rows per tile (UMMA M)
constexpr int XD = 16;                         // dims
constexpr uint32_t X_TILE = XT * XD * 8;       // f64 tile, 16 KB
constexpr uint32_t A_CHUNK = XT * 128;         // one 128-byte K chunk of the operand tile
constexpr uint32_t A_TILE = 2 * A_CHUNK;
constexpr int NA = 2;                          // operand stages
constexpr int TCOLS = 128;                     // TMEM columns per accumulator buffer
constexpr int THREADS = 320;
constexpr int W_CONV = 2, W_EPI = 6;

__host__ __device__ inline uint32_t al(uint32_t v, uint32_t a) { return (v + a - 1) / a * a; }

struct TcxSmem {
  uint32_t x0, a0, b0, crow, hd, acc0, per_warp, bars, total;
  int NX;
  __host__ __device__ TcxSmem(int k, int N, int nx) {
    NX = nx;
    uint32_t o = 0;
    a0 = o;   o += NA * A_TILE;
    x0 = o;   o += nx * X_TILE;
    b0 = o;   o += 2u * N * 128u;
    crow = o; o += (uint32_t)k * crow_stride<XD>() * 8u;
    hd = o;   o += (uint32_t)k * 16u;
    o = al(o, 16);
    acc0 = o;
    per_warp = al((uint32_t)k * (XD + 2) * 8u, 16);
    o += 4 * per_warp;
    bars = o; o += 8 * (2 * nx + 2 * NA + 4) + 16;
    total = o + 1024;  // runtime 1024-byte alignment of the dynamic window
  }
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }

__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// byte offset of 16-byte chunk q of row r in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t swz(int r, int q) { return (uint32_t)r * 128u + ((uint32_t)(q ^ (r & 7)) << 4); }

template <int NG>
__global__ void __launch_bounds__(THREADS, 1)
    mti_tc_kernel(const __grid_constant__ CUtensorMap tmX, const MtiTcArgs a) {
  constexpr int N = 16 * NG;
  pdl_enter();
  if (!a.dbg && a.ctrl->stop && !a.ctrl->ignore_stop) return;  // (the score dump ignores the stop flag)
  if (a.gate && a.ctrl->mti_choice != 1) return;  // the compacted MTI kernel runs this iteration
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int k = a.k;
  const TcxSmem L(k, N, a.nx);
  const int NX = L.NX;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + NX;
  uint64_t* a_full = bars + 2 * NX;
  uint64_t* a_empty = a_full + NA;
  uint64_t* t_full = a_empty + NA;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(t_empty + 2);
  double* crow = reinterpret_cast<double*>(sm + L.crow);
  double2* hd = reinterpret_cast<double2*>(sm + L.hd);
  const bool work = (int)blockIdx.x < a.gtc;  // extra CTAs (grid shared with other kernels) only write zeros

  // ---- setup: B operand image, exact-recipe centroid copy, {drift, half_min}
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.bimg);
    uint4* dst = reinterpret_cast<uint4*>(sm + L.b0);
    for (int i = tid; i < 2 * N * 8; i += THREADS) dst[i] = src[i];
    for (int i = tid; i < k * XD; i += THREADS) {
      const int j = i / XD, e = i - j * XD;
      crow[j * crow_stride<XD>() + e] = a.means[i];
    }
    for (int j = tid; j < k; j += THREADS) hd[j] = make_double2(a.drift[j], a.half_min[j]);
    fence_proxy_async();  // generic-proxy writes of B -> visible to the tensor core
  }
  if (tid == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(x_full + s, 1);
      mbar_init(x_empty + s, 4);
    }
    for (int s = 0; s < NA; ++s) {
      mbar_init(a_full + s, 4);
      mbar_init(a_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(t_full + b, 1);
      mbar_init(t_empty + b, 4);
    }
    fence_barrier_init();
  }
  if (warp == 1 && work) {
    tmem_alloc(tslot, 2 * TCOLS);
    tmem_relinquish();
  }
  if (warp == 0 && lane == 0 && work) prefetch_tmap(&tmX);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = work ? *tslot : 0u;
  const long long ntiles = work ? (a.n + XT - 1) / XT : 0;
  const long long t0 = blockIdx.x, tstep = a.gtc;

  // epilogue-side counters (reduced at the end)
  long long reassigned = 0, skips = 0, computed = 0, flagged = 0;

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (long long t = t0; t < ntiles; t += tstep, ++i) {
        const int s = i % NX;
        mbar_wait(x_empty + s, ((i / NX) & 1) ^ 1);
        mbar_arrive_expect_tx(x_full + s, X_TILE);
        tma_load_2d(sm + L.x0 + s * X_TILE, &tmX, x_full + s, 0, (int)(t * XT));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(XT, N);
      const uint32_t b0 = smem_u32(sm + L.b0), b1 = b0 + N * 128;
      int i = 0;
      for (long long t = t0; t < ntiles; t += tstep, ++i) {
        const int sa = i % NA, b = i & 1;
        mbar_wait(a_full + sa, (i / NA) & 1);
        mbar_wait(t_empty + b, ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dt = tmem + b * TCOLS;
        const uint32_t A0 = smem_u32(sm + L.a0 + sa * A_TILE), A1 = A0 + A_CHUNK;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_tf32(dt, umma_desc_sw128(A0 + ks * 32), umma_desc_sw128(b0 + ks * 32), idesc, ks > 0);
#pragma unroll
        for (int ks = 0; ks < 3; ++ks)
          umma_tf32(dt, umma_desc_sw128(A1 + ks * 32), umma_desc_sw128(b1 + ks * 32), idesc, 1);
        umma_commit(a_empty + sa);
        umma_commit(t_full + b);
      }
    }
  } else if (warp < W_EPI) {
    // ------------------------------------------------------------ converters
    const int r = (warp - W_CONV) * 32 + lane;
    int i = 0;
    for (long long t = t0; t < ntiles; t += tstep, ++i) {
      const int s = i % NX, sa = i % NA;
      mbar_wait(x_full + s, (i / NX) & 1);
      mbar_wait(a_empty + sa, ((i / NA) & 1) ^ 1);
      const unsigned char* xs = sm + L.x0 + s * X_TILE;
      unsigned char* A0 = sm + L.a0 + sa * A_TILE;
      unsigned char* A1 = A0 + A_CHUNK;
      float hi[XD], lo[XD];
      float xn2 = 0.0f;
#pragma unroll
      for (int q = 0; q < XD / 2; ++q) {
        const double2 v = *reinterpret_cast<const double2*>(xs + swz(r, q));
        const float f0 = __double2float_rn(v.x), f1 = __double2float_rn(v.y);
        hi[2 * q] = tf32_trunc(f0);
        hi[2 * q + 1] = tf32_trunc(f1);
        lo[2 * q] = f0 - hi[2 * q];
        lo[2 * q + 1] = f1 - hi[2 * q + 1];
        xn2 = fmaf(f0, f0, xn2);
        xn2 = fmaf(f1, f1, xn2);
      }
      const float xh = tf32_trunc(xn2), xl = xn2 - xh;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const float4 h = make_float4(hi[4 * c], hi[4 * c + 1], hi[4 * c + 2], hi[4 * c + 3]);
        *reinterpret_cast<float4*>(A0 + swz(r, c)) = h;
        *reinterpret_cast<float4*>(A0 + swz(r, c + 4)) =
            make_float4(lo[4 * c], lo[4 * c + 1], lo[4 * c + 2], lo[4 * c + 3]);
        *reinterpret_cast<float4*>(A1 + swz(r, c)) = h;
      }
      *reinterpret_cast<float4*>(A1 + swz(r, 4)) = make_float4(1.0f, 1.0f, xh, xl);
      *reinterpret_cast<float4*>(A1 + swz(r, 5)) = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(a_full + sa);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;          // TMEM lane quarter
    const int r = q * 32 + lane;     // row within the tile
    double* acc = reinterpret_cast<double*>(sm + L.acc0 + (warp - W_EPI) * L.per_warp);
    double* cnt = acc + k * XD;
    double* sqa = cnt + k;
    for (int e = lane; e < k * (XD + 2); e += 32) acc[e] = 0.0;
    __syncwarp();
    const double cmax2 = a.ctrl->cmax2, cmax = sqrt(cmax2);
    const double slop = (8.0 * XD + 32.0) * 0x1p-53;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    auto state = [&](long long t, int& av, double& uv) {
      const long long row = t * XT + r;
      const bool ok = t < ntiles && row < a.n;
      av = ok ? a.assign[row] : -1;
      uv = ok ? a.upper[row] : 0.0;
    };
    int pa;
    double pu;
    state(t0, pa, pu);
    int i = 0;
    for (long long t = t0; t < ntiles; t += tstep, ++i) {
      const int s = i % NX, b = i & 1;
      const int orig = pa;
      const double u0 = pu;
      state(t + tstep, pa, pu);
      const long long row = t * XT + r;
      const bool valid = orig >= 0;
      const int oc = valid ? orig : 0;
      const double2 dh = hd[oc];                  // {drift, half_min}
      const double u = u0 + dh.x;                 // inflate (u + 0.0 == u)
      const bool skip = valid && u <= dh.y;       // clause 1
      const bool live = a.dbg ? valid : (valid && !skip);
      if (!a.dbg) {
        skips += skip ? 1 : 0;
        if (skip && dh.x != 0.0) {  // the inflated bound is the skipped row's state
          a.upper[row] = u;
          a.tight[row] = 0;
        }
      }
      mbar_wait(t_full + b, (i >> 1) & 1);
      tc_fence_after();
      const unsigned lmask = __ballot_sync(0xffffffffu, live);
      int k1 = 0x7fffffff, k2 = 0x7fffffff;
      if (lmask) {
        uint32_t v[NG][16];
#pragma unroll
        for (int g = 0; g < NG; ++g) tmem_ld16(tl + b * TCOLS + 16 * g, v[g]);
        tmem_wait_ld();
        if (a.dbg) {
          if (valid) {
            float* o = a.dbg + row * N;
#pragma unroll
            for (int g = 0; g < NG; ++g)
#pragma unroll
              for (int e = 0; e < 16; ++e) o[16 * g + e] = __uint_as_float(v[g][e]);
          }
        } else {
#pragma unroll
          for (int g = 0; g < NG; ++g) {
            int key[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) key[e] = (int)((v[g][e] & 0xFFFFFF80u) | (uint32_t)(16 * g + e));
            int gm = key[0];
#pragma unroll
            for (int e = 1; e < 15; e += 2) gm = min(gm, min(key[e], key[e + 1]));
            gm = min(gm, key[15]);
            // second smallest of the group: min over key - gm - 1 as unsigned (gm itself wraps)
            const uint32_t off = (uint32_t)(-gm - 1);
            uint32_t g2 = 0xFFFFFFFFu;
#pragma unroll
            for (int e = 0; e < 16; ++e) g2 = min(g2, (uint32_t)key[e] + off);
            const int g2k = (int)((uint32_t)gm + 1u + g2);
            const int nk1 = min(k1, gm);
            k2 = min(max(k1, gm), min(k2, g2k));
            k1 = nk1;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(t_empty + b);

      // the f64 rows of this tile (landed before the converters ran; the wait only
      // orders this warp's reads after the TMA)
      mbar_wait(x_full + s, (i / NX) & 1);
      const unsigned char* xs = sm + L.x0 + s * X_TILE;
      if (!a.dbg && lmask) {
        double x[XD];
#pragma unroll
        for (int c = 0; c < XD / 2; ++c) {
          const double2 vv = *reinterpret_cast<const double2*>(xs + swz(r, c));
          x[2 * c] = vv.x;
          x[2 * c + 1] = vv.y;
        }
        bool cert = false;
        int win = k1 & 127;
        if (live) {
          double xn2 = 0.0;
#pragma unroll
          for (int e = 0; e < XD; ++e) xn2 = fma(x[e], x[e], xn2);
          const double E = 0x1p-20 * (12.0 * sqrt(xn2) * cmax + 4.0 * (xn2 + cmax2)) + slop * (xn2 + cmax2);
          const double m1 = (double)__int_as_float(k1 & ~127), m2 = (double)__int_as_float(k2 & ~127);
          const double lo2 = m2 - 0x1p-16 * fabs(m2), hi1 = m1 + 0x1p-16 * fabs(m1);
          cert = lo2 - hi1 > 2.0 * E && win < k;
        }
        double nd = 0.0;
        // uncertified rows: the whole warp re-ranks each one with the exact recipe,
        // scan_block's order -- the current centroid first, then ascending ids, switch
        // on strict < of the sqrt'ed distances (pruning.py:174-203)
        unsigned fl = __ballot_sync(0xffffffffu, live && !cert);
        if (lane == 0) flagged += __popc(fl);
        while (fl) {
          const int f = __ffs(fl) - 1;
          fl &= fl - 1;
          const int fo = __shfl_sync(0xffffffffu, orig, f);
          double xf[XD];
#pragma unroll
          for (int c = 0; c < XD / 2; ++c) {
            const double2 vv = *reinterpret_cast<const double2*>(xs + swz(q * 32 + f, c));
            xf[2 * c] = vv.x;
            xf[2 * c + 1] = vv.y;
          }
          double bd = CUDART_INF;
          int bp = 0x7fffffff, bj = 0;
          for (int j = lane; j < k; j += 32) {
            double cj[XD];
            load_crow<XD>(crow, j, cj);
            const double dj = sqrt(exact_sq_fixed<XD>(xf, cj));
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
        if (live && cert) {
          double cw[XD];
          load_crow<XD>(crow, win, cw);
          nd = sqrt(exact_sq_fixed<XD>(x, cw));
        }
        const bool moved = live && win != orig;
        double sq = 0.0;
        if (live) {
          a.upper[row] = nd;
          a.tight[row] = 1;
          if (moved) {
            a.assign[row] = win;
            ++reassigned;
            sq = exact_sq_fixed<XD>(x, Zero{});
          }
        }
        if (lane == 0) computed += (long long)__popc(lmask) * k;
        const unsigned mm = __ballot_sync(0xffffffffu, moved);
        if (mm)
          accumulate_in_row_order<XD, TileLayout<XD>, true>(mm, win, orig, sq, xs + q * 32 * 128, acc, cnt, sqa, XD,
                                                            lane);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(x_empty + s);
    }
  }
  __syncthreads();
  if (warp == 1 && work) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * TCOLS);
  }

  // CTA partial: the four epilogue warps' sums in warp order, then the scalars
  const long long Lg = acc_len(k, XD);
  double* out = a.partials + (long long)blockIdx.x * Lg;
  const int kk = k * (XD + 2);
  for (int e = tid; e < kk; e += THREADS) {
    double v = 0.0;
    if (work)
      for (int w = 0; w < 4; ++w) v += reinterpret_cast<const double*>(sm + L.acc0 + w * L.per_warp)[e];
    out[e] = v;
  }
  __shared__ long long red[4][4];
  if (warp >= W_EPI) {
    const long long c0 = warp_sum_ll(reassigned), c1 = warp_sum_ll(skips), c2 = warp_sum_ll(computed),
                    c3 = warp_sum_ll(flagged);
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
      for (int w = 0; w < 4; ++w)
        for (int c = 0; c < 4; ++c) tot[c] += red[w][c];
    double* sc = out + kk;
    for (int c = 0; c < NSCAL; ++c) sc[c] = 0.0;
    sc[S_REASSIGNED] = (double)tot[0];
    sc[S_SKIPS] = (double)tot[1];
    sc[S_COMPUTED] = (double)tot[2];
    if (a.counters && tot[3]) atomicAdd(a.counters, (unsigned long long)tot[3]);
  }
}

// B operand image in global memory, exactly as the kernel's shared memory holds it:
// chunk 0 row j = [-2 c_hi | -2 c_hi], chunk 1 row j = [-2 c_lo | cn2_hi, cn2_lo, 1, 1,
// 0, 0, 0, 0 | 0 ...]; padded rows j >= k score 2^100 (never a winner, never in a window)
__global__ void mti_tc_prep_kernel(const double* __restrict__ means, int k, int N, uint4* __restrict__ bimg) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * N * 8; i += gridDim.x * blockDim.x) {
    const int chunk = i / (N * 8), rem = i - chunk * N * 8, j = rem >> 3, qq = rem & 7;
    float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    const bool real = j < k;
    if (chunk == 0 || qq < 4) {
      const int e0 = (chunk == 0 ? (qq & 3) : qq) * 4;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const double c = real ? means[(long long)j * XD + e0 + m] : 0.0;
        const float ch = tf32_trunc(__double2float_rn(c));
        const float cl = tf32_rna(__double2float_rn(c - (double)ch));
        v[m] = -2.0f * (chunk == 0 ? ch : cl);
      }
    } else if (qq == 4) {
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

template <int NG>
cudaError_t launch_ng(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  const TcxSmem L(a.k, 16 * NG, a.nx);
  cudaError_t e = cudaFuncSetAttribute(mti_tc_kernel<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  return launch_pdl(mti_tc_kernel<NG>, dim3(grid), dim3(THREADS), L.total, s, *tm, a);
}

constexpr size_t SMEM_MAX = 227 * 1024;

}  // namespace

// stages of the f64 ring that fit (0: the kernel does not apply)
int mti_tc_stages(int d, int k) {
  if (d != XD || k < 1 || k > 128) return 0;
  const int N = (k + 15) / 16 * 16;
  for (int nx = 4; nx >= 2; --nx)
    if (TcxSmem(k, N, nx).total <= SMEM_MAX) return nx;
  return 0;
}

size_t mti_tc_bimg_bytes(int k) { return (size_t)2 * ((k + 15) / 16 * 16) * 128; }

cudaError_t launch_mti_tc_prep(const double* means, int k, void* bimg, cudaStream_t s) {
  const int N = (k + 15) / 16 * 16;
  mti_tc_prep_kernel<<<(2 * N * 8 + 255) / 256, 256, 0, s>>>(means, k, N, reinterpret_cast<uint4*>(bimg));
  return cudaGetLastError();
}

cudaError_t launch_mti_tc(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s) {
  switch ((a.k + 15) / 16) {
    case 1: return launch_ng<1>(tm, a, grid, s);
    case 2: return launch_ng<2>(tm, a, grid, s);
    case 3: return launch_ng<3>(tm, a, grid, s);
    case 4: return launch_ng<4>(tm, a, grid, s);
    case 5: return launch_ng<5>(tm, a, grid, s);
    case 6: return launch_ng<6>(tm, a, grid, s);
    case 7: return launch_ng<7>(tm, a, grid, s);
    case 8: return launch_ng<8>(tm, a, grid, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace knb
