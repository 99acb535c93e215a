// Warp-level building blocks shared by the tensor-core kernels (assign_mma.cu,
// mti_mma.cu): DMMA scoring of a 32-row block against all centroids with the
// near-tie certificate, and the deterministic warp-local segmented accumulation.
#pragma once

#include <math_constants.h>

#include "common.cuh"

#ifndef KNB_EXPERIMENT
#define KNB_EXPERIMENT 0
#endif


namespace knb {

constexpr int BR = 32;  // rows per warp block

// Row stride (doubles) of the exact-recipe centroid copy in shared memory: DP + 2, so
// rows stay 16-byte aligned (16-byte loads) and the lanes of a warp reading DIFFERENT
// centroids' chunk e spread over all eight 16-byte bank groups (a DP stride put every
// lane in the same bank).
template <int DP>
__host__ __device__ constexpr int crow_stride() { return DP + 2; }

template <int DP>
__device__ __forceinline__ void load_crow(const double* __restrict__ crow, int j, double (&c)[DP]) {
  const double2* p = reinterpret_cast<const double2*>(crow + j * crow_stride<DP>());
#pragma unroll
  for (int q = 0; q < DP / 2; ++q) {
    const double2 v = p[q];
    c[2 * q] = v.x;
    c[2 * q + 1] = v.y;
  }
}

// not volatile: the mma has no side effects, so ptxas may interleave it with the epilogue
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
#if KNB_EXPERIMENT == 2  // experiment: no tensor work
  c[0] += a; c[1] += b; return;
#endif
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// running argmax with the near-tie flag; integer ops on the high word of s - best
__device__ __forceinline__ void score_update(double& best, int& bid, bool& flag, double s, int j, int tolhi) {
#if KNB_EXPERIMENT == 1  // experiment: no epilogue (keep the value live)
  best = fmax(best, s); return;
#endif
  const double diff = __dsub_rn(s, best);
  const int h = __double2hiint(diff);
  const bool better = h > 0;
  const bool near = (h & 0x7fffffff) <= tolhi;
  flag = near | (flag & !better);
  best = better ? s : best;
  bid = better ? j : bid;
}

// merge a partial state whose ids all come after the running one's (ties keep the
// running, earlier id)
__device__ __forceinline__ void merge_later(double& best, int& bid, bool& flag, double ob, int oi, bool of,
                                            int tolhi) {
  const double diff = __dsub_rn(ob, best);
  const int h = __double2hiint(diff);
  const bool near = (h & 0x7fffffff) <= tolhi;
  const bool other = h > 0;
  flag = near | (other ? of : flag);
  best = other ? ob : best;
  bid = other ? oi : bid;
}

// merge the disjoint partial (best, id, flag) held by lane ^ lanemask
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

// Lane that finishes row r of a block after the quad combine (row = t4*8 + g).
__device__ __forceinline__ int owner_lane(int r) { return ((r & 7) << 2) | (r >> 3); }

// Upper bound of ||x||^2 for a survivor of the MTI filter: u >= d(x, c_a) (the inflated
// bound, exact recipe up to rounding) and ||c_a||^2 = -2 chn[a], so
// ||x||^2 <= (||c_a|| + u)^2 <= 2 ||c_a||^2 + 2 u^2; the factor covers the rounding of
// both terms (relative 1e-13 at most) with a wide margin.
__device__ __forceinline__ double xnorm2_bound(double u, double chn_a) {
  return (2.0 * u * u - 4.0 * chn_a) * (1.0 + 0x1p-30);
}

struct Scored {
  int id;       // certified argmax (or 0 when uncertified)
  bool flag;    // near tie: caller re-ranks with the exact recipe
  double best;  // s of the winner (x.c - ||c||^2/2)
  double xn2;   // ||x||^2 of the lane's row
};

// Score the 32 rows of a block (TileLayout<DP>, BR rows at tb) against every centroid.
// bf: centroids in B-fragment order, chn: -||c||^2/2 (dummy columns -inf).
// Each lane returns the result for its row owner_lane^-1(lane) = t4*8 + g.
// SMALLK: at most two 8-centroid tiles (k <= 16) -- one step, no software pipeline, so
// the second set of accumulators never needs registers
// LEAN: fewest registers (A fragments re-read from shared memory, one accumulator set,
// tiles scored one step at a time) for kernels that trade them for more warps
// BCROW: `bf` is the row-major centroid copy with stride crow_stride<DP>() instead of
// the fragment-ordered array (saves kp x DP x 8 bytes of shared memory; the 8 rows x 32
// bytes of one fragment load still take the minimum two wavefronts at that stride)
// XB: the caller knows an upper bound of ||x||^2 for every row (lane r holds row r's in
// xb); the certificate only needs an upper bound, so the d-term sums are skipped.
// TL: the staging tile's layout (TileLayout<DP> or its cp.async-only variant)
// ONE: k <= 8 (a single centroid tile; the dense pass instantiates it for such k)
template <int DP, bool SMALLK = false, bool LEAN = false, bool BCROW = false, bool XB = false,
          class TL = TileLayout<DP>, bool ONE = false>
__device__ __forceinline__ Scored score_block(const unsigned char* tb, const double* bf, const double* chn,
                                              int ntile8, double tolk, double cmax2, int lane, double xb = 0.0) {
  constexpr int KS = DP / 4;
  constexpr bool ACACHE = DP <= 32 && !LEAN;
  const int g = lane >> 2, t4 = lane & 3;
  double afr[4][ACACHE ? KS : 1];
  double xn2[4];
#pragma unroll
  for (int pg = 0; pg < 4; ++pg) {
    if constexpr (XB) {
      xn2[pg] = __shfl_sync(0xffffffffu, xb, pg * 8 + g);
      if constexpr (ACACHE) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
          afr[pg][ks] = *reinterpret_cast<const double*>(tb + TL::elem_off(pg * 8 + g, ks * 4 + t4, BR));
      }
      continue;
    }
    double s2 = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const double v = *reinterpret_cast<const double*>(tb + TL::elem_off(pg * 8 + g, ks * 4 + t4, BR));
      if constexpr (ACACHE) afr[pg][ks] = v;
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
  // Centroid-tile-major: for each 8-centroid tile, 4 independent accumulator chains
  // (one per 8-row group) run d/4 k-steps; that tile's epilogue only depends on its own
  // chains, so ptxas overlaps it with the next tile's DMMAs.
  // Two tiles per step (8 independent chains), software-pipelined: the DMMAs of step
  // q+2 are issued before the epilogue of step q, so the tensor pipe works while the
  // epilogue's dependent integer chain runs.  An odd tile count pads with a dummy
  // tile whose chn is -inf (never wins, never near).
  auto mma_step = [&](int q, double (&c0)[4][2], double (&c1)[4][2]) {
    const bool two = q + 1 < ntile8;
    const double2 h0 = *reinterpret_cast<const double2*>(chn + q * 8 + 2 * t4);
    const double2 h1 = two ? *reinterpret_cast<const double2*>(chn + (q + 1) * 8 + 2 * t4)
                           : make_double2(-CUDART_INF, -CUDART_INF);
#pragma unroll
    for (int pg = 0; pg < 4; ++pg) {
      c0[pg][0] = h0.x; c0[pg][1] = h0.y;
      c1[pg][0] = h1.x; c1[pg][1] = h1.y;
    }
    const int q1 = two ? q + 1 : q;  // a valid fragment address for the dummy tile
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double bv0, bv1;
      if constexpr (BCROW) {
        bv0 = bf[(q * 8 + g) * crow_stride<DP>() + ks * 4 + t4];
        bv1 = bf[(q1 * 8 + g) * crow_stride<DP>() + ks * 4 + t4];
      } else {
        bv0 = bf[((q * KS + ks) << 5) + lane];
        bv1 = bf[((q1 * KS + ks) << 5) + lane];
      }
#pragma unroll
      for (int pg = 0; pg < 4; ++pg) {
        double av;
        if constexpr (ACACHE) av = afr[pg][ks];
        else av = *reinterpret_cast<const double*>(tb + TL::elem_off(pg * 8 + g, ks * 4 + t4, BR));
        dmma(c0[pg], av, bv0);
        dmma(c1[pg], av, bv1);
      }
    }
  };
  // The step's four scores per row group are first reduced among themselves (two
  // independent pairs, then a merge), and only the result is merged into the
  // running state: the loop-carried chain is one merge per step instead of four
  // updates.  Same result: the argmax (lowest id on ties) and "some other score
  // within tol of it" do not depend on the order of the merges.
  auto epilogue = [&](int q, const double (&c0)[4][2], const double (&c1)[4][2]) {
    const int j0 = q * 8 + 2 * t4;
#pragma unroll
    for (int pg = 0; pg < 4; ++pg) {
      double pb = c0[pg][0], qb = c1[pg][0];
      int pi = j0, qi = j0 + 8;
      bool pf = false, qf = false;
      score_update(pb, pi, pf, c0[pg][1], j0 + 1, tolhi[pg]);
      score_update(qb, qi, qf, c1[pg][1], j0 + 9, tolhi[pg]);
      merge_later(pb, pi, pf, qb, qi, qf, tolhi[pg]);
      merge_later(best[pg], bid[pg], flag[pg], pb, pi, pf, tolhi[pg]);
    }
  };
  // k <= 8 (one tile): only the real tile's DMMAs; the second set stays at -inf
  auto mma_one = [&](double (&c0)[4][2], double (&c1)[4][2]) {
    const double2 h0 = *reinterpret_cast<const double2*>(chn + 2 * t4);
#pragma unroll
    for (int pg = 0; pg < 4; ++pg) {
      c0[pg][0] = h0.x; c0[pg][1] = h0.y;
      c1[pg][0] = -CUDART_INF; c1[pg][1] = -CUDART_INF;
    }
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      double bv0;
      if constexpr (BCROW) bv0 = bf[g * crow_stride<DP>() + ks * 4 + t4];
      else bv0 = bf[(ks << 5) + lane];
#pragma unroll
      for (int pg = 0; pg < 4; ++pg) {
        double av;
        if constexpr (ACACHE) av = afr[pg][ks];
        else av = *reinterpret_cast<const double*>(tb + TL::elem_off(pg * 8 + g, ks * 4 + t4, BR));
        dmma(c0[pg], av, bv0);
      }
    }
  };
  double ca0[4][2], ca1[4][2];
  if constexpr (ONE) mma_one(ca0, ca1);
  else mma_step(0, ca0, ca1);
  if constexpr (SMALLK || ONE) {
    epilogue(0, ca0, ca1);
  } else if constexpr (LEAN) {
    epilogue(0, ca0, ca1);
#pragma unroll 1
    for (int q = 2; q < ntile8; q += 2) {
      mma_step(q, ca0, ca1);
      epilogue(q, ca0, ca1);
    }
  } else {
    double cb0[4][2], cb1[4][2];
    int q = 0;
#pragma unroll 1
    for (; q + 2 < ntile8; q += 4) {
      mma_step(q + 2, cb0, cb1);
      epilogue(q, ca0, ca1);
      if (q + 4 < ntile8) mma_step(q + 4, ca0, ca1);
      epilogue(q + 2, cb0, cb1);
    }
    if (q < ntile8) epilogue(q, ca0, ca1);
  }
#pragma unroll
  for (int pg = 0; pg < 4; ++pg) {
    combine(best[pg], bid[pg], flag[pg], tolhi[pg], 1);
    combine(best[pg], bid[pg], flag[pg], tolhi[pg], 2);
  }
  Scored r{bid[0], flag[0], best[0], xn2[0]};
#pragma unroll
  for (int pg = 1; pg < 4; ++pg)
    if (t4 == pg) { r.id = bid[pg]; r.flag = flag[pg]; r.best = best[pg]; r.xn2 = xn2[pg]; }
  return r;
}

// Scorer results of row `lane` (score_block leaves row r's in lane owner_lane(r)); after
// this, lane r handles row r: 8 consecutive rows per quarter-warp, so the exact tree's
// 16-byte row loads hit 8 distinct bank groups under either tile swizzle
__device__ __forceinline__ Scored rows_to_lanes(const Scored& sc, int lane) {
  const int src = owner_lane(lane);
  Scored o;
  o.id = __shfl_sync(0xffffffffu, sc.id, src);
  o.flag = __shfl_sync(0xffffffffu, (int)sc.flag, src) != 0;
  o.best = __shfl_sync(0xffffffffu, sc.best, src);
  o.xn2 = __shfl_sync(0xffffffffu, sc.xn2, src);
  return o;
}

// Exact recipe on the lane's row: re-rank over every centroid (ascending, strict <,
// sqrt domain, distance.py:106-116) when flagged, else the distance to `id`.
// orig >= 0 (pruned passes): the scan starts from the point's current centroid and its
// exact distance and skips it, as scan_block does (pruning.py:174-203: cur = orig,
// switch only on dx < u), so an exact tie keeps the current centroid; orig < 0 (full
// passes, nearest_block_into): the lowest id wins a tie.
template <int DP, class TL = TileLayout<DP>>
__device__ __forceinline__ double exact_winner(const unsigned char* tb, int r, const double* crow, int k, int d,
                                               bool flag, int& id, double* sq_out, int orig = -1) {
  double x[DP];
#pragma unroll
  for (int q2 = 0; q2 < DP / 2; ++q2) {
    const double2 v = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, q2, BR));
    x[2 * q2] = v.x;
    x[2 * q2 + 1] = v.y;
  }
  double nd;
  if (flag) {
    auto dist = [&](int j) {
      if constexpr (DP <= 32) {
        double cj[DP];
        load_crow<DP>(crow, j, cj);
        return sqrt(exact_sq<DP>(x, cj, d));
      } else {
        return sqrt(exact_sq<DP>(x, crow + j * crow_stride<DP>(), d));
      }
    };
    double bd = orig >= 0 ? dist(orig) : CUDART_INF;
    int bi = orig >= 0 ? orig : 0;
    for (int j = 0; j < k; ++j) {
      if (j == orig) continue;
      const double dj = dist(j);
      if (dj < bd) { bd = dj; bi = j; }
    }
    id = bi;
    nd = bd;
  } else {
    if constexpr (DP <= 32) {  // 16-byte loads into registers
      double ci[DP];
      load_crow<DP>(crow, id, ci);
      nd = sqrt(exact_sq<DP>(x, ci, d));
    } else {  // (DP = 64 is register-bound)
      nd = sqrt(exact_sq<DP>(x, crow + id * crow_stride<DP>(), d));
    }
  }
  if (sq_out) *sq_out = exact_sq<DP>(x, Zero{}, d);
  return nd;
}

// scan_block's choice for the lane's row by the exact recipe alone, no tensor-core scores
// (narrow rows and few centroids -- config 3, d = 8, k = 10 -- where k exact distances
// are ~16 k FP64 instructions and the DMMA scorer's fixed epilogue / combine / certificate
// cost more): start from the current centroid `orig`, then ascending ids, switch on strict
// < (pruning.py:174-203).  The scan runs on the SQUARED distances and takes one square
// root, of the winner: sqrt is monotone, so no switch where sq_j >= best is the
// reference's decision too, and a switch with sq_j < best (1 - 2^-50) is strict after the
// roots' roundings (2^-53 relative each); a switch inside that margin -- the roots may
// collide -- sends the row through the sqrt-domain scan.  Every lane reads the same
// centroid (shared-memory broadcast).  Returns the winner's distance; id = the winner.
// FULL: d == DP, the tree's shape is known at compile time (decided once, outside the scan)
// HAS_ORIG: pruned passes (scan_block's rule above); false: full passes
// (nearest_block_into, distance.py:106-116: ascending ids, strict <, the lowest id wins a tie)
template <int DP, bool FULL, bool HAS_ORIG>
__device__ __forceinline__ double direct_scan(const double (&x)[DP], const double* crow, int k, int d, int orig,
                                              int& id) {
  auto sqd = [&](int j) {
    double cj[DP];
    load_crow<DP>(crow, j, cj);
    if constexpr (FULL) return exact_sq_fixed<DP>(x, cj);
    else return exact_sq<DP>(x, cj, d);
  };
  double bs = CUDART_INF;
  int bi = 0;
  if constexpr (HAS_ORIG) {
    bs = sqd(orig);
    bi = orig;
  }
  bool close = false;
  // branch-free (selects), two centroids' distance chains in flight
  auto step = [&](double sj, int j) {  // (j == orig repeats bs bit for bit: no switch)
    const bool lt = sj < bs;
    close |= lt && !(sj < bs * (1.0 - 0x1p-50));
    bs = lt ? sj : bs;
    bi = lt ? j : bi;
  };
  int j = 0;
  for (; j + 2 <= k; j += 2) {
    const double s0 = sqd(j), s1 = sqd(j + 1);
    step(s0, j);
    step(s1, j + 1);
  }
  if (j < k) step(sqd(j), j);
  double nd = sqrt(bs);
  if (close) {
    nd = HAS_ORIG ? sqrt(sqd(orig)) : CUDART_INF;
    bi = HAS_ORIG ? orig : 0;
    for (int jj = 0; jj < k; ++jj) {
      if (HAS_ORIG && jj == orig) continue;
      const double dj = sqrt(sqd(jj));
      if (dj < nd) { nd = dj; bi = jj; }
    }
  }
  id = bi;
  return nd;
}

// sq_out: also ||x||^2 by the exact recipe (row_sqnorms, the pruned run's first pass)
template <int DP, class TL = TileLayout<DP>, bool HAS_ORIG = true>
__device__ __forceinline__ double direct_winner(const unsigned char* tb, int r, const double* crow, int k, int d,
                                                int orig, int& id, double* sq_out = nullptr) {
  double x[DP];
#pragma unroll
  for (int q2 = 0; q2 < DP / 2; ++q2) {
    const double2 v = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, q2, BR));
    x[2 * q2] = v.x;
    x[2 * q2 + 1] = v.y;
  }
  if (sq_out) *sq_out = exact_sq<DP>(x, Zero{}, d);
  if (d == DP) return direct_scan<DP, true, HAS_ORIG>(x, crow, k, d, orig, id);
  return direct_scan<DP, false, HAS_ORIG>(x, crow, k, d, orig, id);
}

// exact_sq_fixed<DP> (d == DP, DP in {16, 32, 64}) streamed: x from tile row r, c from a
// crow row, eight elements at a time in the tree's own grouping (group a of every
// 32-element block feeds z[a][*], then acc[a][l] = z[a][l] + z[a][l + 4] joins s[l] in
// the order ((acc0 + acc1) + acc2) + acc3) -- the same roundings in the same order,
// with about 20 doubles live instead of the whole row and centroid
// SELF: c = 0 (row_sqnorms' vecdot(x, x): x - 0.0 == x, the same tree)
template <int DP, bool SELF = false, class TL = TileLayout<DP>>
__device__ __forceinline__ double exact_sq_stream(const unsigned char* tb, int r, const double* __restrict__ c) {
  static_assert(DP == 16 || DP == 32 || DP == 64, "streamed tree for d == DP in {16, 32, 64}");
  constexpr int n32 = DP & ~31;
  double s[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    double acc[4];
    if constexpr (n32 > 0) {
      double z[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) z[l] = 0.0;
#pragma unroll
      for (int i = 0; i < n32; i += 32) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int e = i + 8 * a + 2 * h;
          const double2 xv = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, e >> 1, BR));
          const double2 cv = SELF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(c + e);
          const double v0 = __dsub_rn(xv.x, cv.x), v1 = __dsub_rn(xv.y, cv.y);
          z[2 * h] = __fma_rn(v0, v0, z[2 * h]);
          z[2 * h + 1] = __fma_rn(v1, v1, z[2 * h + 1]);
        }
      }
#pragma unroll
      for (int l = 0; l < 4; ++l) acc[l] = __dadd_rn(z[l], z[l + 4]);
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = 4 * a + 2 * h;
        const double2 xv = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, e >> 1, BR));
        const double2 cv = SELF ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(c + e);
        const double v0 = __dsub_rn(xv.x, cv.x), v1 = __dsub_rn(xv.y, cv.y);
        acc[2 * h] = __fma_rn(v0, v0, 0.0);
        acc[2 * h + 1] = __fma_rn(v1, v1, 0.0);
      }
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) s[l] = a == 0 ? acc[l] : __dadd_rn(s[l], acc[l]);
  }
  return __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
}

// exact_winner for d == DP with the streamed tree (fewest registers); same orig rule
template <int DP, class TL = TileLayout<DP>>
__device__ __forceinline__ double exact_winner_stream(const unsigned char* tb, int r, const double* crow, int k,
                                                      bool flag, int& id, int orig = -1) {
  if (flag) {
    double bd = orig >= 0 ? sqrt(exact_sq_stream<DP, false, TL>(tb, r, crow + orig * crow_stride<DP>()))
                          : CUDART_INF;
    int bi = orig >= 0 ? orig : 0;
    for (int j = 0; j < k; ++j) {
      if (j == orig) continue;
      const double dj = sqrt(exact_sq_stream<DP, false, TL>(tb, r, crow + j * crow_stride<DP>()));
      if (dj < bd) { bd = dj; bi = j; }
    }
    id = bi;
    return bd;
  }
  return sqrt(exact_sq_stream<DP, false, TL>(tb, r, crow + id * crow_stride<DP>()));
}

// vecdot(x, x) of tile row r by the exact recipe (row_sqnorms, distance.py:66-72)
template <int DP, class TL = TileLayout<DP>>
__device__ __forceinline__ double row_self_sq(const unsigned char* tb, int r, int d) {
  double x[DP];
#pragma unroll
  for (int q2 = 0; q2 < DP / 2; ++q2) {
    const double2 v = *reinterpret_cast<const double2*>(tb + TL::chunk_off(r, q2, BR));
    x[2 * q2] = v.x;
    x[2 * q2 + 1] = v.y;
  }
  return exact_sq<DP>(x, Zero{}, d);
}

// Deterministic warp-local accumulation in row order, lanes = dims.  For every row r
// set in `rowmask` (ascending; the row's values live in lane owner_lane(r)):
//   acc[to][e] += x[r][e], cnt[to] += 1, sqa[to] += sq, and when from >= 0 the same
//   amounts are subtracted from cluster `from` (a moved row's signed delta,
//   engine.py:345-353).  Full passes pass every valid row with from = -1.
// IDENT: row r's values live in lane r (instead of owner_lane(r))
template <int DP, class TL = TileLayout<DP>, bool IDENT = false>
__device__ __forceinline__ void accumulate_in_row_order(unsigned rowmask, int to, int from, double sq,
                                                        const unsigned char* tb, double* acc, double* cnt,
                                                        double* sqa, int d, int lane) {
  const int e0 = lane < d ? lane : 0;
  const int e1 = lane + 32 < d ? lane + 32 : 0;
  while (rowmask) {
    const int r = __ffs(rowmask) - 1;
    rowmask &= rowmask - 1;
    const int src = IDENT ? r : owner_lane(r);
    const int t = __shfl_sync(0xffffffffu, to, src);
    const int f = __shfl_sync(0xffffffffu, from, src);
    const double q = __shfl_sync(0xffffffffu, sq, src);
    const double x0 = *reinterpret_cast<const double*>(tb + TL::elem_off(r, e0, BR));
    if (lane < d) {
      acc[t * d + lane] += x0;
      if (f >= 0) acc[f * d + lane] -= x0;
    }
    if constexpr (DP > 32) {
      const double x1 = *reinterpret_cast<const double*>(tb + TL::elem_off(r, e1, BR));
      if (lane + 32 < d) {
        acc[t * d + lane + 32] += x1;
        if (f >= 0) acc[f * d + lane + 32] -= x1;
      }
    }
    if (lane == 0) {
      cnt[t] += 1.0;
      sqa[t] += q;
      if (f >= 0) {
        cnt[f] -= 1.0;
        sqa[f] -= q;
      }
    }
  }
}

// accumulate_in_row_order for a FULL pass (every row of the mask joins cluster `to`, nothing
// is subtracted) over rows of 16 doubles, two rows per step: lanes 0-15 add row 2i, lanes
// 16-31 row 2i + 1 (values, count and ||x||^2) to their rows' clusters; when the two rows
// share a cluster the halves add one after the other.  Every sum still receives its rows in
// ascending row order -- the same additions in the same order as the one-row walk (bit-
// identical sums) in half the steps.  Config 4's first pass: the one-row walk, 58
// instructions per row, was half of its 323 ms; 236 ms with this.  (Narrower rows, four
// or eight per step, measured slower than the one-row walk at small k -- config 3: 1.92-1.98
// vs 1.82 ms -- where rows of one step share a cluster half of the time.)
template <int DP, class TL = TileLayout<DP>, bool IDENT = false>
__device__ __forceinline__ void accumulate_full_rows(unsigned rowmask, int to, double sq, const unsigned char* tb,
                                                     double* acc, double* cnt, double* sqa, int d, int lane) {
  if constexpr (DP != 16) {
    accumulate_in_row_order<DP, TL, IDENT>(rowmask, to, -1, sq, tb, acc, cnt, sqa, d, lane);
  } else {
    const int half = lane >> 4, e = lane & 15;
    const int ee = e < d ? e : 0;
    // step i's cluster ids, ||x||^2 and row values are fetched while step i - 1 adds (the
    // tile and the lanes' results are read-only here; only the sums carry a dependence)
    struct Step {
      int t, t_other;
      double q, x0;
    };
    auto fetch = [&](int r0) {
      const int r = (r0 < BR ? r0 : 0) + half;
      const int src = IDENT ? r : owner_lane(r);
      Step s;
      s.t = __shfl_sync(0xffffffffu, to, src);
      s.q = __shfl_sync(0xffffffffu, sq, src);
      s.x0 = *reinterpret_cast<const double*>(tb + TL::elem_off(r, ee, BR));
      s.t_other = __shfl_xor_sync(0xffffffffu, s.t, 16);
      return s;
    };
    Step nx = fetch(0);
#pragma unroll 1
    for (int r0 = 0; r0 < BR; r0 += 2) {
      const Step c = nx;
      nx = fetch(r0 + 2);
      const unsigned two = (rowmask >> r0) & 3u;
      if (two == 0u) continue;  // warp-uniform
      const bool ok = (two >> half) & 1u;
      const int t = c.t;
      const bool clash = two == 3u && t == c.t_other;  // warp-uniform
      auto add = [&]() {
        if (ok && e < d) acc[t * d + e] += c.x0;
        if (ok && e == 0) {
          cnt[t] += 1.0;
          sqa[t] += c.q;
        }
      };
      if (!clash) {
        add();
      } else {
        if (half == 0) add();
        __syncwarp();
        if (half == 1) add();
      }
      __syncwarp();  // the next step's halves may touch the same sums from other lanes
    }
  }
}

// Bit r set when the lane owning row r (owner_lane(r)) passes `pred`.
__device__ __forceinline__ unsigned row_mask(bool pred, int my_row) {
  return __reduce_or_sync(0xffffffffu, pred ? (1u << my_row) : 0u);
}

}  // namespace knb
