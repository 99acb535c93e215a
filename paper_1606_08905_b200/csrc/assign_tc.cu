// K1-TC: the dense assignment pass for f32 rows on the tcgen05 tensor cores
// (BASELINE config 5: d = 256, k = 1000, pruning off), with a certified argmin.
//
// The reference computes every distance in f64 as sqrt(vecdot(x - c, x - c))
// and keeps the lowest-id strict-less minimum (distance.py:94-116) on the f64
// upcast of the f32 matrix (matrix.py:40).  Here:
//
//   score    s_j = x . c_j - ||c_j||^2 / 2 from one kind::tf32 UMMA per 128 rows x
//            256 centroids x 8 dims, accumulated in TMEM (argmax s == argmin d)
//   bound    |s~_j - s_j| <= T(x) = e ||x|| cmax + (f32 rounding) + (reference
//            rounding slop), e = 1.25 * 2^-9: the tensor core TRUNCATES each f32
//            operand to 10 mantissa bits (< 2^-10 relative each, measured by
//            tools/tf32_probe.py), products are exact in f32, and the f32 sums add
//            < 2^-15 of sum |x_i c_i|; the tests check measured errors stay under
//            e / 2 on adversarial inputs
//   certify  s~_1 - s~_2 > 2 T(x): the tensor-core argmax IS the reference's
//            argmin -- written directly
//   rerank   otherwise every centroid with s~_j >= s~_1 - 2 T(x) (up to seven, else
//            all k) is re-scored with the exact f64 recipe (tc_rerank_kernel, one
//            warp-wide ddot tree per candidate): the reference's answer, ties to the
//            lowest id
//   window   the epilogue keeps only scores >= a per-row floor known before the
//            scan, so the per-score work is one add, one compare and a branch that
//            is almost never taken:
//              first pass     a TC_MAX pass finds max_j s~_j, the TC_COLLECT pass
//                             then keeps s~_j >= max - 2T (the GEMM runs twice)
//              later passes   u >= d(x, c_old) from the previous pass and the
//                             centroid drift give max_j s~_j >= (|x|^2 - (u +
//                             drift)^2) / 2 - T, so the floor is that minus 2T
//
// Kernel shape (one CTA per SM, persistent over 128-row tiles, 8 warps):
//   warp 0      TMA producer of the row tile (d/32 chunks of 128 rows x 128 B,
//               SWIZZLE_128B), one mbarrier per chunk so the next tile's chunk c
//               loads as soon as the last MMA reading chunk c retires
//   warp 1      TMA producer of centroid chunks (256 centroids x 32 dims) through
//               a 3-stage ring
//   warp 2      TMEM allocation (512 columns = two 128 x 256 f32 accumulators)
//               and the single-thread MMA issuer
//   warps 4-7   epilogue: tcgen05.ld 64 columns at a time, s = acc + chn, window
//               test, certificate, assignment / distance bound / rerank queue
// HBM traffic: the rows once per pass (d * 4 B per row); the centroid matrix
// (k_pad * d_pad * 4 B) is re-read from L2 once per 128-row tile.
#include <cuda.h>
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace knb {

namespace {

constexpr int TC_M = 128;
constexpr int TC_N = 256;
constexpr int TC_KC = 32;
constexpr int TC_BST = 6;
constexpr int TC_THREADS = 384;  // 4 control warps + 8 epilogue warps
constexpr uint32_t A_CHUNK = TC_M * 128;
constexpr uint32_t B_CHUNK = (TC_N / 2) * 128;  // this CTA's half of a centroid chunk

constexpr int LIST = 7;  // candidates a queue entry carries (row + 7 ids); more -> all k
constexpr int TOPK = 8;  // window scores kept per row (and per epilogue half)

__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// the TOPK largest window scores of a row, descending; equal scores keep the
// earlier (lower) id first.  push() returns the score that fell off the end.
struct Top {
  float s[TOPK];
  int i[TOPK];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int m = 0; m < TOPK; ++m) { s[m] = -CUDART_INF_F; i[m] = -1; }
  }
  __device__ __forceinline__ float push(float v, int j) {
#pragma unroll
    for (int m = 0; m < TOPK; ++m) {
      if (v > s[m]) {
        const float ts = s[m];
        const int ti = i[m];
        s[m] = v;
        i[m] = j;
        v = ts;
        j = ti;
      }
    }
    return v;
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_assign_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmC,
                     const TcArgs a) {
  if (a.ctrl->stop && !a.ctrl->ignore_stop) return;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  unsigned char* A = sm;
  unsigned char* Bs = sm + a.nkc * A_CHUNK;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Bs + TC_BST * B_CHUNK);
  uint64_t* a_full = bars;
  uint64_t* a_empty = bars + 8;
  uint64_t* b_full = bars + 16;
  uint64_t* b_empty = b_full + TC_BST;
  uint64_t* t_full = b_empty + TC_BST;
  uint64_t* t_empty = t_full + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();  // CTA pair: rank 0 issues the M = 256 MMAs
  const bool leader = rank == 0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.nkc; ++i) {
      mbar_init(a_full + i, 1);
      mbar_init(a_empty + i, 1);
    }
    for (int s = 0; s < TC_BST; ++s) {
      mbar_init(b_full + s, 1);
      mbar_init(b_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(t_full + b, 1);
      mbar_init(t_empty + b, 16);  // one arrival per epilogue warp of both CTAs
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    tmem_alloc2(tslot, 2 * TC_N);
    tmem_relinquish2();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmC);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // pair tiles of 256 rows: this CTA owns rows [256 pt + 128 rank, + 128)
  const long long ntp = (a.n + 2 * TC_M - 1) / (2 * TC_M);
  const long long pt0 = blockIdx.x >> 1, ptstep = gridDim.x >> 1;

  if (warp == 0) {
    if (lane == 0) {  // row tiles (both CTAs; completion counted at the leader)
      int it = 0;
      for (long long pt = pt0; pt < ntp; pt += ptstep, ++it) {
        for (int kc = 0; kc < a.nkc; ++kc) {
          mbar_wait(a_empty + kc, (it & 1) ^ 1);
          if (leader) mbar_arrive_expect_tx(a_full + kc, 2 * A_CHUNK);
          tma_load_2d_pair(A + kc * A_CHUNK, &tmX, a_full + kc, kc * TC_KC, (int)(pt * 2 * TC_M + rank * TC_M));
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // centroid chunks: this CTA loads centroids [256 nt + 128 rank, + 128)
      int s = 0;
      uint32_t ph = 0;
      for (long long pt = pt0; pt < ntp; pt += ptstep)
        for (int nt = 0; nt < a.nnt; ++nt)
          for (int kc = 0; kc < a.nkc; ++kc) {
            mbar_wait(b_empty + s, ph ^ 1);
            if (leader) mbar_arrive_expect_tx(b_full + s, 2 * B_CHUNK);
            tma_load_2d_pair(Bs + s * B_CHUNK, &tmC, b_full + s, kc * TC_KC, nt * TC_N + (int)rank * (TC_N / 2));
            if (++s == TC_BST) { s = 0; ph ^= 1; }
          }
    }
  } else if (warp == 2) {
    if (lane == 0 && leader) {  // MMA issuer (M = 256 across the pair, N = 256)
      const uint32_t idesc = umma_idesc_tf32(2 * TC_M, TC_N);
      int s = 0, it = 0;
      uint32_t ph = 0, u = 0;
      for (long long pt = pt0; pt < ntp; pt += ptstep, ++it) {
        for (int nt = 0; nt < a.nnt; ++nt, ++u) {
          const uint32_t ab = u & 1;
          mbar_wait(t_empty + ab, ((u >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t dt = tmem + ab * TC_N;
          for (int kc = 0; kc < a.nkc; ++kc) {
            if (nt == 0) mbar_wait(a_full + kc, it & 1);
            mbar_wait(b_full + s, ph);
            tc_fence_after();
            const uint32_t abase = smem_u32(A + kc * A_CHUNK), bbase = smem_u32(Bs + s * B_CHUNK);
#pragma unroll
            for (int k4 = 0; k4 < TC_KC / 8; ++k4)
              umma_tf32_pair(dt, umma_desc_sw128(abase + k4 * 32), umma_desc_sw128(bbase + k4 * 32), idesc,
                             (kc | k4) != 0);
            umma_commit_pair(b_empty + s);
            if (nt == a.nnt - 1) umma_commit_pair(a_empty + kc);
            if (++s == TC_BST) { s = 0; ph ^= 1; }
          }
          umma_commit_pair(t_full + ab);
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    // two warps per TMEM lane quarter: half h scans columns [128h, 128h + 128) of
    // every N-tile; half 1 hands its per-row result to half 0 through a small global
    // scratch (named barrier per quarter), half 0 certifies and writes the outputs
    const int q = warp & 3;
    const int h = (warp - 4) >> 2;
    const int r = q * 32 + lane;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    const double cmax2 = a.ctrl->cmax2;
    const double cmax = sqrt(cmax2);
    const double slop = (8.0 * a.d + 32.0) * 0x1p-53;
    const unsigned lt = (1u << lane) - 1u;
    int4* myq = a.queue + 2 * (long long)(blockIdx.x * 4 + q) * a.qcap;
    long long qn = 0;
    unsigned long long moved = 0, flagged = 0, fulls = 0;
    uint32_t u = 0;
    int par = 0;
    for (long long pt = pt0; pt < ntp; pt += ptstep, par ^= 1) {
      const long long row = pt * 2 * TC_M + rank * TC_M + r;
      const bool valid = row < a.n;
      int old = 0;
      double xn2 = 0.0, T = 0.0;
      float lim = -CUDART_INF_F;
      if (valid) {
        old = a.assign[row];
        xn2 = a.xn2[row];
        const double xn = sqrt(xn2);
        T = a.err_rel * xn * cmax + 0x1p-20 * (xn * cmax + cmax2) + slop * (xn2 + cmax2);
        if (a.mode == TC_COLLECT_SMAX) {
          // the same scores' maximum from the TC_MAX pass: the window is exact
          lim = __double2float_rd((double)a.bound[row] - 2.0 * T - 0x1p-30 * (fabs((double)a.bound[row]) + T));
        } else if (a.mode == TC_COLLECT_BOUND) {
          // u >= d(x, c_old) under the previous centroids, so d(x, c_old') <= u + drift:
          // max_j s~_j >= s~_old >= (||x||^2 - (u + drift)^2) / 2 - T; window 2T below it
          const double ub = (double)a.bound[row] + a.drift[old];
          const double sl = 0.5 * (xn2 - ub * ub) - 3.0 * T;
          lim = __double2float_rd(sl - 0x1p-30 * (fabs(sl) + xn2 + ub * ub));
        }
      }
      const float w2 = __double2float_ru(2.0 * T);
      // window state (registers only): the TOPK largest scores >= lim, sorted; lim
      // only rises (to the running best - 2T); the largest score pushed out of the
      // list is remembered so an incomplete list is detected
      Top top;
      top.reset();
      float best = -CUDART_INF_F, dropped = -CUDART_INF_F;
      for (int nt = 0; nt < a.nnt; ++nt, ++u) {
        const uint32_t ab = u & 1;
        mbar_wait(t_full + ab, (u >> 1) & 1);
        tc_fence_after();
#pragma unroll 1
        for (int cc = h * (TC_N / 2); cc < (h + 1) * (TC_N / 2); cc += 64) {
          float v0[32], v1[32];
          tmem_ld32(tl + ab * TC_N + cc, v0);
          tmem_ld32(tl + ab * TC_N + cc + 32, v1);
          const int j0 = nt * TC_N + cc;
          const float4* ch = reinterpret_cast<const float4*>(a.chn32 + j0);
          float4 c4[16];
#pragma unroll
          for (int g = 0; g < 16; ++g) c4[g] = __ldg(ch + g);
          tmem_wait_ld();
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            v0[4 * g + 0] += c4[g].x;
            v0[4 * g + 1] += c4[g].y;
            v0[4 * g + 2] += c4[g].z;
            v0[4 * g + 3] += c4[g].w;
            v1[4 * g + 0] += c4[8 + g].x;
            v1[4 * g + 1] += c4[8 + g].y;
            v1[4 * g + 2] += c4[8 + g].z;
            v1[4 * g + 3] += c4[8 + g].w;
          }
          if (a.dbg) {  // score dump (tests of the error bound)
            if (valid) {
              float* o = a.dbg + row * a.kp + j0;
#pragma unroll
              for (int m = 0; m < 32; ++m) { o[m] = v0[m]; o[32 + m] = v1[m]; }
            }
            continue;
          }
          // chunk maximum as a tree (independent 3-input max ops)
          float t8[8];
#pragma unroll
          for (int g = 0; g < 8; ++g)
            t8[g] = fmaxf(fmaxf(fmaxf(v0[4 * g], v0[4 * g + 1]), fmaxf(v0[4 * g + 2], v0[4 * g + 3])),
                          fmaxf(fmaxf(v1[4 * g], v1[4 * g + 1]), fmaxf(v1[4 * g + 2], v1[4 * g + 3])));
          const float cm = fmaxf(fmaxf(fmaxf(t8[0], t8[1]), fmaxf(t8[2], t8[3])),
                                 fmaxf(fmaxf(t8[4], t8[5]), fmaxf(t8[6], t8[7])));
          if (a.mode == TC_MAX) {
            best = fmaxf(best, cm);
          } else if (__any_sync(0xffffffffu, cm >= lim)) {
            // rare path: some row of the warp has scores inside its window here.
            // Columns hit by any lane are re-read from TMEM one at a time (a
            // warp-uniform column index), so no score array goes to local memory.
            uint32_t h0 = 0u, h1 = 0u;
            if (cm >= lim) {
#pragma unroll
              for (int m = 0; m < 32; ++m) {
                h0 |= (v0[m] >= lim ? 1u : 0u) << m;
                h1 |= (v1[m] >= lim ? 1u : 0u) << m;
              }
            }
#pragma unroll
            for (int half2 = 0; half2 < 2; ++half2) {
              const uint32_t mine = half2 ? h1 : h0;
              uint32_t un = __reduce_or_sync(0xffffffffu, mine);
#pragma unroll 1
              while (un) {
                const int m = __ffs(un) - 1;
                un &= un - 1;
                const int col = cc + 32 * half2 + m;
                float x = tmem_ld1(tl + ab * TC_N + col);
                x += __ldg(a.chn32 + nt * TC_N + col);  // the same add as the chunk's
                if (((mine >> m) & 1u) && x >= lim) {
                  const int j = nt * TC_N + col;
                  lim = fmaxf(lim, __fsub_rd(x, w2));
                  dropped = fmaxf(dropped, top.push(x, j));
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(t_empty + ab);
      }
      if (a.dbg) continue;
      // ---- merge the two halves of the row (half 1 -> scratch -> half 0)
      TcHalf* hs = a.scratch + ((long long)(blockIdx.x * 2 + par) * TC_M + r);
      if (a.mode != TC_MAX) best = top.s[0];
      if (h == 1) {
        hs->best = best;
        hs->dropped = dropped;
#pragma unroll
        for (int m = 0; m < TOPK; ++m) { hs->v[m] = top.s[m]; hs->j[m] = top.i[m]; }
      }
      named_barrier_sync(1 + q, 64);
      if (h == 1) continue;
      {
        int besti = top.i[0];
        const float b1 = hs->best;
        if (b1 > best) {  // equal maxima: the lower id (half 0) stays first
          best = b1;
          besti = hs->j[0];
        }
        dropped = fmaxf(dropped, hs->dropped);
        if (a.mode == TC_MAX) {
          if (valid) a.bound[row] = best;
          continue;
        }
        // certificate: the candidates are the scores within 2T of the maximum
        bool flag = false;
        int4 e0 = make_int4((int)row, -1, -1, -1), e1 = make_int4(-1, -1, -1, -1);
        if (valid) {
          const double thr = (double)best - 2.0 * T;
          int c[LIST];
#pragma unroll
          for (int m = 0; m < LIST; ++m) c[m] = -1;
          int nc = 0;
          auto add = [&](float v, int id) {
            if ((double)v >= thr) {
#pragma unroll
              for (int p = 0; p < LIST; ++p)
                if (p == nc) c[p] = id;
              ++nc;
            }
          };
#pragma unroll
          for (int m = 0; m < TOPK; ++m) add(top.s[m], top.i[m]);
#pragma unroll
          for (int m = 0; m < TOPK; ++m) add(hs->v[m], hs->j[m]);
          if (besti < 0 || nc > LIST || (double)dropped >= thr) {
            // candidate list incomplete: all k, by a whole CTA (tc_rerank_full_kernel)
            const unsigned long long pos = atomicAdd(a.counters + 3, 1ull);
            a.fullq[pos] = (int)row;
            ++fulls;
            ++flagged;
          } else if (nc == 1) {
            a.assign[row] = besti;
            moved += (besti != old);
            // upper bound of d(x, c_best) for the next pass: S >= s~ - T
            const double d2 = xn2 - 2.0 * ((double)best - T);
            a.bound[row] = __double2float_ru(sqrt(d2 > 0.0 ? d2 : 0.0) * (1.0 + 0x1p-40));
          } else {
            flag = true;
            e0.y = c[0]; e0.z = c[1]; e0.w = c[2];
            e1.x = c[3]; e1.y = c[4]; e1.z = c[5]; e1.w = c[6];
          }
          a.old_assign[row] = old;
        }
        const unsigned fm = __ballot_sync(0xffffffffu, flag);
        if (flag) {
          int4* slot = myq + 2 * (qn + __popc(fm & lt));
          slot[0] = e0;
          slot[1] = e1;
        }
        qn += __popc(fm);
        flagged += flag;
      }
    }
    if (h == 0 && a.mode != TC_MAX && !a.dbg) {
      if (lane == 0) a.qcount[blockIdx.x * 4 + q] = (int)qn;
      moved = (unsigned long long)warp_sum_ll((long long)moved);
      flagged = (unsigned long long)warp_sum_ll((long long)flagged);
      fulls = (unsigned long long)warp_sum_ll((long long)fulls);
      if (lane == 0) {
        atomicAdd(a.counters + 0, moved);
        atomicAdd(a.counters + 1, flagged);
        atomicAdd(a.counters + 2, fulls);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // the peer's MMAs and TMEM reads are done
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2(tmem, 2 * TC_N);
  }
}

// Exact f64 re-scoring of the rows the certificate could not settle: one warp per
// queued row, one warp-wide exact distance per candidate; the lexicographic
// (distance, id) minimum is the reference's strict-less ascending scan
// (distance.py:114-116).  Overflowed windows go to tc_rerank_full_kernel.
__global__ void __launch_bounds__(128) tc_rerank_kernel(const float* __restrict__ X, int d, int k,
                                                        const double* __restrict__ means, int32_t* assign,
                                                        const int32_t* __restrict__ old_assign,
                                                        const int4* __restrict__ queue, const int* qcount,
                                                        long long qcap, unsigned long long* counters,
                                                        float* __restrict__ bound, const Ctrl* ctrl) {
  if (ctrl->stop && !ctrl->ignore_stop) return;
  const int lane = threadIdx.x & 31;
  const int wstep = gridDim.y * (blockDim.x >> 5);
  const int w0 = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int cnt = qcount[blockIdx.x];
  const int4* base = queue + 2 * (long long)blockIdx.x * qcap;
  unsigned long long moved = 0;
  for (int i = w0; i < cnt; i += wstep) {
    const int4 e0 = base[2 * i], e1 = base[2 * i + 1];
    const long long row = e0.x;
    const float* x = X + row * d;
    double bd = CUDART_INF;
    int bi = 0x7fffffff;
    const int c[7] = {e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
    if ((d & 31) == 0) {
      // d a multiple of 32 (<= 256): the row stays in registers and every candidate's
      // loads are independent, so all of them are in flight together
      const int nq = d >> 5;
      double xv[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) xv[q] = q < nq ? (double)x[32 * q + lane] : 0.0;
      // candidates two at a time (the list is filled from the front); a missing second
      // one re-reads the first centroid (L1) and is discarded
#pragma unroll
      for (int m = 0; m < 7; m += 2) {
        if (c[m] < 0) break;  // warp-uniform
        const bool two = m + 1 < 7 && c[m + 1] >= 0;
        const double* ca = means + (long long)c[m] * d;
        const double* cb = means + (long long)(two ? c[m + 1] : c[m]) * d;
        double za = 0.0, zb = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (q < nq) {
            const double va = __dsub_rn(xv[q], ca[32 * q + lane]);
            const double vb = __dsub_rn(xv[q], cb[32 * q + lane]);
            za = __fma_rn(va, va, za);
            zb = __fma_rn(vb, vb, zb);
          }
        }
        const double da = sqrt(warp_tree_finish(za, lane));
        if (da < bd || (da == bd && c[m] < bi)) { bd = da; bi = c[m]; }
        if (two) {
          const double db = sqrt(warp_tree_finish(zb, lane));
          if (db < bd || (db == bd && c[m + 1] < bi)) { bd = db; bi = c[m + 1]; }
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < 7; ++m) {
        if (c[m] >= 0) {
          const double dist = sqrt(warp_exact_sq(x, means + (long long)c[m] * d, d, lane));
          if (dist < bd || (dist == bd && c[m] < bi)) { bd = dist; bi = c[m]; }
        }
      }
    }
    if (lane == 0) {
      assign[row] = bi;
      moved += (bi != old_assign[row]);
      bound[row] = __double2float_ru(bd * (1.0 + 0x1p-40));  // next pass's window (TC_COLLECT_BOUND)
    }
  }
  if (lane == 0 && moved) atomicAdd(counters + 0, moved);
}

// Rows whose candidate window overflowed: every centroid, exact recipe, one CTA per row
// (32 warps split the centroids, ascending and strict-less within a warp, then the
// lexicographic (distance, id) minimum across warps -- the reference's scan).
__global__ void __launch_bounds__(1024) tc_rerank_full_kernel(const float* __restrict__ X, int d, int k,
                                                              const double* __restrict__ means, int32_t* assign,
                                                              const int32_t* __restrict__ old_assign,
                                                              const int* __restrict__ fullq,
                                                              unsigned long long* counters, float* __restrict__ bound,
                                                              const Ctrl* ctrl) {
  if (ctrl->stop && !ctrl->ignore_stop) return;
  __shared__ double sd[32];
  __shared__ int si[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const long long cnt = (long long)counters[3];
  for (long long e = blockIdx.x; e < cnt; e += gridDim.x) {
    const long long row = fullq[e];
    const float* x = X + row * d;
    double bd = CUDART_INF;
    int bi = 0x7fffffff;
    for (int j = warp; j < k; j += nw) {
      const double dist = sqrt(warp_exact_sq(x, means + (long long)j * d, d, lane));
      if (dist < bd) { bd = dist; bi = j; }
    }
    if (lane == 0) { sd[warp] = bd; si[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w)
        if (sd[w] < bd || (sd[w] == bd && si[w] < bi)) { bd = sd[w]; bi = si[w]; }
      assign[row] = bi;
      if (bi != old_assign[row]) atomicAdd(counters + 0, 1ull);
      bound[row] = __double2float_ru(bd * (1.0 + 0x1p-40));
    }
    __syncthreads();
  }
}

// f32 tensor-core operand of the centroids: k_pad x d_pad, zero padded; the score
// offset -||c||^2 / 2 per centroid, -inf for the padding so it never wins.
__global__ void tc_prep_kernel(const double* __restrict__ means, const double* __restrict__ cn2, int k, int d,
                               int kp, int dp, float* __restrict__ c32, float* __restrict__ chn32) {
  const long long tot = (long long)kp * dp;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / dp), e = (int)(i - (long long)j * dp);
    // the B operand pre-rounded to TF32 (nearest): the tensor core's truncation of it is
    // then exact, and only the row operand's truncation remains in the certificate
    float v = (j < k && e < d) ? (float)means[(long long)j * d + e] : 0.0f;
    uint32_t t;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(v));
    c32[i] = __uint_as_float(t);
    if (e == 0) chn32[j] = j < k ? (float)(-0.5 * cn2[j]) : -CUDART_INF_F;
  }
}

// ||x||^2 per row in f64 (products of f32 values are exact in f64): one warp per row.
__global__ void row_sqnorm_f32_kernel(const float* __restrict__ X, long long n, int d, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < n; r += nw) {
    const float* x = X + r * d;
    double s = 0.0;
    for (int e = lane; e < d; e += 32) {
      const double v = x[e];
      s = __fma_rn(v, v, s);
    }
    s = warp_sum(s);
    if (lane == 0) out[r] = s;
  }
}

__global__ void tc_scalars_kernel(const unsigned long long* counters, long long n_local, int k, int d,
                                  double* exch, const Ctrl* ctrl) {
  if (ctrl->stop && !ctrl->ignore_stop) return;
  double* sc = exch + (long long)k * d + 2LL * k;
  for (int i = 0; i < NSCAL; ++i) sc[i] = 0.0;
  sc[S_REASSIGNED] = (double)counters[0];
  sc[S_COMPUTED] = (double)n_local * (double)k;
  sc[S_ROWS] = (double)n_local;
}

}  // namespace

size_t tc_smem_bytes(int nkc) {
  return (size_t)nkc * A_CHUNK + (size_t)TC_BST * B_CHUNK + 8 * (2 * 8 + 2 * TC_BST + 4) + 16 + 1024;
}

int tc_rows_per_tile() { return TC_M; }

cudaError_t launch_tc_assign(const CUtensorMap* tmX, const CUtensorMap* tmC, const TcArgs& a, int grid,
                             cudaStream_t s) {
  const size_t sm = tc_smem_bytes(a.nkc);
  cudaError_t e = cudaFuncSetAttribute(tc_assign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return e;
  tc_assign_kernel<<<grid, TC_THREADS, sm, s>>>(*tmX, *tmC, a);  // grid even: CTA pairs
  return cudaGetLastError();
}

cudaError_t launch_tc_rerank_full(const TcArgs& a, const double* means, int grid, cudaStream_t s) {
  tc_rerank_full_kernel<<<grid, 1024, 0, s>>>(a.X, a.d, a.k, means, a.assign, a.old_assign, a.fullq, a.counters,
                                              a.bound, a.ctrl);
  return cudaGetLastError();
}

cudaError_t launch_tc_rerank(const TcArgs& a, const double* means, int regions, cudaStream_t s) {
  tc_rerank_kernel<<<dim3(regions, 16), 128, 0, s>>>(a.X, a.d, a.k, means, a.assign, a.old_assign, a.queue, a.qcount,
                                           a.qcap, a.counters, a.bound, a.ctrl);
  return cudaGetLastError();
}

cudaError_t launch_tc_prep(const double* means, const double* cn2, int k, int d, int kp, int dp, float* c32,
                           float* chn32, cudaStream_t s) {
  long long tot = (long long)kp * dp;
  int blocks = (int)((tot + 255) / 256);
  if (blocks > 2048) blocks = 2048;
  tc_prep_kernel<<<blocks, 256, 0, s>>>(means, cn2, k, d, kp, dp, c32, chn32);
  return cudaGetLastError();
}

cudaError_t launch_row_sqnorm_f32(const float* X, long long n, int d, double* out, cudaStream_t s) {
  row_sqnorm_f32_kernel<<<1184, 256, 0, s>>>(X, n, d, out);
  return cudaGetLastError();
}

cudaError_t launch_tc_scalars(const unsigned long long* counters, long long n_local, int k, int d, double* exch,
                              const Ctrl* ctrl, cudaStream_t s) {
  tc_scalars_kernel<<<1, 1, 0, s>>>(counters, n_local, k, d, exch, ctrl);
  return cudaGetLastError();
}

}  // namespace knb
