// Shared device helpers for the B200 Lloyd / MTI k-means path.
//
// The exact distance recipe: the reference computes every point-centroid
// distance as sqrt(vecdot(x - c, x - c)) in f64 (numakmeans distance.py:28-39);
// for f64 rows np.vecdot is OpenBLAS ddot, whose SkylakeX kernel sums in a fixed
// tree (restated in oracle/exact_tree.c).  exact_sq()
// below evaluates the same tree with explicitly rounded intrinsics so no FMA
// contraction can change a bit; where the host BLAS uses that kernel the GPU's
// MTI bounds, drifts and tightened distances are bit-identical to the oracle's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "state.cuh"

namespace knb {

// ---------------------------------------------------------------- exact recipe
// x: the point, either in registers (natural order) or any addressable array;
// c: the centroid row.  d <= DP.  Mirrors oracle/exact_tree.c::tree_sq.
// exact_sq for d == DP: the tree's shape is known at compile time (no per-element
// bound tests -- for d = 32 those were a fifth of the MTI kernel's instructions)
template <int DP, typename XS, typename CS>
__device__ __forceinline__ double exact_sq_fixed(const XS& x, const CS& c) {
  constexpr int n1 = DP & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if constexpr (n1 > 0) {
    double acc[4][4];
    if constexpr (n32 > 0) {
      double z[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 8; ++l) z[a][l] = 0.0;
#pragma unroll
      for (int i = 0; i < n32; i += 32)
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int l = 0; l < 8; ++l) {
            const double v = __dsub_rn(x[i + 8 * a + l], c[i + 8 * a + l]);
            z[a][l] = __fma_rn(v, v, z[a][l]);
          }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[a][l] = __dadd_rn(z[a][l], z[a][l + 4]);
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[a][l] = 0.0;
    }
#pragma unroll
    for (int i = n32; i < n1; i += 16)
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          const double v = __dsub_rn(x[i + 4 * a + l], c[i + 4 * a + l]);
          acc[a][l] = __fma_rn(v, v, acc[a][l]);
        }
    double s[4];
#pragma unroll
    for (int l = 0; l < 4; ++l)
      s[l] = __dadd_rn(__dadd_rn(__dadd_rn(acc[0][l], acc[1][l]), acc[2][l]), acc[3][l]);
    dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
  }
#pragma unroll
  for (int i = n1; i < DP; ++i) {
    const double v = __dsub_rn(x[i], c[i]);
    dot = __fma_rn(v, v, dot);
  }
  return dot;
}

template <int DP, typename XS, typename CS>
__device__ __forceinline__ double exact_sq(const XS& x, const CS& c, int d) {
  if (d == DP) return exact_sq_fixed<DP>(x, c);
  const int n1 = d & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if (n1) {
    double acc[4][4];
    if constexpr (DP >= 32) {
      double z[4][8];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 8; ++l) z[a][l] = 0.0;
#pragma unroll
      for (int i = 0; i + 32 <= DP; i += 32) {
        if (i < n32) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int l = 0; l < 8; ++l) {
              double v = __dsub_rn(x[i + 8 * a + l], c[i + 8 * a + l]);
              z[a][l] = __fma_rn(v, v, z[a][l]);
            }
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[a][l] = __dadd_rn(z[a][l], z[a][l + 4]);
    } else {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[a][l] = 0.0;  // z + z of zeros
    }
    if constexpr (DP >= 16) {
#pragma unroll
      for (int i = 0; i + 16 <= DP; i += 16) {
        if (i >= n32 && i < n1) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int l = 0; l < 4; ++l) {
              double v = __dsub_rn(x[i + 4 * a + l], c[i + 4 * a + l]);
              acc[a][l] = __fma_rn(v, v, acc[a][l]);
            }
        }
      }
    }
    double s[4];
#pragma unroll
    for (int l = 0; l < 4; ++l)
      s[l] = __dadd_rn(__dadd_rn(__dadd_rn(acc[0][l], acc[1][l]), acc[2][l]), acc[3][l]);
    dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
  }
#pragma unroll
  for (int i = 0; i < DP; ++i) {
    if (i >= n1 && i < d) {
      double v = __dsub_rn(x[i], c[i]);
      dot = __fma_rn(v, v, dot);
    }
  }
  return dot;
}

// Runtime-d variant for arbitrary d (no register array): same tree.
// TX = double, or float for f32 rows (the reference's f64 upcast is exact).
template <typename TX>
__device__ __forceinline__ double exact_sq_rt(const TX* __restrict__ x, const double* __restrict__ c, int d) {
  const int n1 = d & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if (n1) {
    double z[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int l = 0; l < 8; ++l) z[a][l] = 0.0;
    for (int i = 0; i < n32; i += 32) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          double v = __dsub_rn((double)x[i + 8 * a + l], c[i + 8 * a + l]);
          z[a][l] = __fma_rn(v, v, z[a][l]);
        }
    }
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int l = 0; l < 4; ++l) acc[a][l] = __dadd_rn(z[a][l], z[a][l + 4]);
    for (int i = n32; i < n1; i += 16) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) {
          double v = __dsub_rn((double)x[i + 4 * a + l], c[i + 4 * a + l]);
          acc[a][l] = __fma_rn(v, v, acc[a][l]);
        }
    }
    double s[4];
#pragma unroll
    for (int l = 0; l < 4; ++l)
      s[l] = __dadd_rn(__dadd_rn(__dadd_rn(acc[0][l], acc[1][l]), acc[2][l]), acc[3][l]);
    dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
  }
  for (int i = n1; i < d; ++i) {
    double v = __dsub_rn((double)x[i], c[i]);
    dot = __fma_rn(v, v, dot);
  }
  return dot;
}

// vecdot(x, x) for runtime d (row_sqnorms, distance.py:66-72): the same tree on
// x itself (x - 0 == x exactly, so this equals exact_sq_rt against a zero row).
__device__ __forceinline__ double exact_self_rt(const double* __restrict__ x, int d) {
  const int n1 = d & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if (n1) {
    double z[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int l = 0; l < 8; ++l) z[a][l] = 0.0;
    for (int i = 0; i < n32; i += 32) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 8; ++l) z[a][l] = __fma_rn(x[i + 8 * a + l], x[i + 8 * a + l], z[a][l]);
    }
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int l = 0; l < 4; ++l) acc[a][l] = __dadd_rn(z[a][l], z[a][l + 4]);
    for (int i = n32; i < n1; i += 16) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int l = 0; l < 4; ++l) acc[a][l] = __fma_rn(x[i + 4 * a + l], x[i + 4 * a + l], acc[a][l]);
    }
    double s[4];
#pragma unroll
    for (int l = 0; l < 4; ++l)
      s[l] = __dadd_rn(__dadd_rn(__dadd_rn(acc[0][l], acc[1][l]), acc[2][l]), acc[3][l]);
    dot = __dadd_rn(__dadd_rn(s[0], s[2]), __dadd_rn(s[1], s[3]));
  }
  for (int i = n1; i < d; ++i) dot = __fma_rn(x[i], x[i], dot);
  return dot;
}

// Exact distance of one row to one centroid by a whole warp, bit-identical to
// exact_sq_rt (the OpenBLAS ddot tree of oracle/exact_tree.c): lane 8a + l owns
// accumulator z[a][l] of the 32-wide blocks, lanes l < 4 then own acc[a][l] of the
// 16-wide blocks, and the final adds run in the tree's order through shuffles.
// The result is valid in every lane.
template <typename TX>
__device__ __forceinline__ double warp_exact_sq(const TX* __restrict__ x, const double* __restrict__ c, int d,
                                                int lane) {
  const int n1 = d & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if (n1) {
    double z = 0.0;
#pragma unroll 8  // independent loads: one memory latency for the whole row
    for (int i = 0; i < n32; i += 32) {
      const double v = __dsub_rn((double)x[i + lane], c[i + lane]);
      z = __fma_rn(v, v, z);
    }
    const int a = lane >> 3, l = lane & 7;
    // acc[a][l] = z[a][l] + z[a][l + 4]   (lanes with l < 4)
    double acc = __dadd_rn(z, __shfl_down_sync(0xffffffffu, z, 4));
    for (int i = n32; i < n1; i += 16) {
      if (l < 4) {
        const double v = __dsub_rn((double)x[i + 4 * a + l], c[i + 4 * a + l]);
        acc = __fma_rn(v, v, acc);
      }
    }
    // s[l] = ((acc[0][l] + acc[1][l]) + acc[2][l]) + acc[3][l]   (on lane l < 4)
    const double a1 = __shfl_down_sync(0xffffffffu, acc, 8);
    const double a2 = __shfl_down_sync(0xffffffffu, acc, 16);
    const double a3 = __shfl_down_sync(0xffffffffu, acc, 24);
    const double sl = __dadd_rn(__dadd_rn(__dadd_rn(acc, a1), a2), a3);
    const double s0 = __shfl_sync(0xffffffffu, sl, 0), s1 = __shfl_sync(0xffffffffu, sl, 1);
    const double s2 = __shfl_sync(0xffffffffu, sl, 2), s3 = __shfl_sync(0xffffffffu, sl, 3);
    dot = __dadd_rn(__dadd_rn(s0, s2), __dadd_rn(s1, s3));
  }
  for (int i = n1; i < d; ++i) {
    const double v = __dsub_rn((double)x[i], c[i]);
    dot = __fma_rn(v, v, dot);
  }
  return dot;
}

// vecdot(x, x) by a whole warp, bit-identical to exact_self_rt (warp_exact_sq's tree
// with x - 0 == x)
__device__ __forceinline__ double warp_exact_self(const double* __restrict__ x, int d, int lane) {
  const int n1 = d & ~15, n32 = n1 & ~31;
  double dot = 0.0;
  if (n1) {
    double z = 0.0;
#pragma unroll 8
    for (int i = 0; i < n32; i += 32) {
      const double v = x[i + lane];
      z = __fma_rn(v, v, z);
    }
    const int a = lane >> 3, l = lane & 7;
    double acc = __dadd_rn(z, __shfl_down_sync(0xffffffffu, z, 4));
    for (int i = n32; i < n1; i += 16) {
      if (l < 4) {
        const double v = x[i + 4 * a + l];
        acc = __fma_rn(v, v, acc);
      }
    }
    const double a1 = __shfl_down_sync(0xffffffffu, acc, 8);
    const double a2 = __shfl_down_sync(0xffffffffu, acc, 16);
    const double a3 = __shfl_down_sync(0xffffffffu, acc, 24);
    const double sl = __dadd_rn(__dadd_rn(__dadd_rn(acc, a1), a2), a3);
    const double s0 = __shfl_sync(0xffffffffu, sl, 0), s1 = __shfl_sync(0xffffffffu, sl, 1);
    const double s2 = __shfl_sync(0xffffffffu, sl, 2), s3 = __shfl_sync(0xffffffffu, sl, 3);
    dot = __dadd_rn(__dadd_rn(s0, s2), __dadd_rn(s1, s3));
  }
  for (int i = n1; i < d; ++i) dot = __fma_rn(x[i], x[i], dot);
  return dot;
}

// The tail of warp_exact_sq for d a multiple of 32 (no 16-wide or scalar blocks):
// lane 8a + l holds z[a][l]; returns the tree's dot in every lane.
__device__ __forceinline__ double warp_tree_finish(double z, int lane) {
  const double acc = __dadd_rn(z, __shfl_down_sync(0xffffffffu, z, 4));
  const double a1 = __shfl_down_sync(0xffffffffu, acc, 8);
  const double a2 = __shfl_down_sync(0xffffffffu, acc, 16);
  const double a3 = __shfl_down_sync(0xffffffffu, acc, 24);
  const double sl = __dadd_rn(__dadd_rn(__dadd_rn(acc, a1), a2), a3);
  const double s0 = __shfl_sync(0xffffffffu, sl, 0), s1 = __shfl_sync(0xffffffffu, sl, 1);
  const double s2 = __shfl_sync(0xffffffffu, sl, 2), s3 = __shfl_sync(0xffffffffu, sl, 3);
  (void)lane;
  return __dadd_rn(__dadd_rn(s0, s2), __dadd_rn(s1, s3));
}

// A zero array stand-in so exact_sq(x, Zero{}, d) computes vecdot(x, x)
// (row_sqnorms, distance.py:66-72: no subtract; x - 0 == x exactly).
struct Zero {
  __device__ __forceinline__ double operator[](int) const { return 0.0; }
};

// --------------------------------------------------------------- smem layout
// Point tiles are stored the way a 2-D TMA box with hardware swizzle lands
// them: panels of up to 16 doubles (128 B) per row; inside a panel the 16-byte
// chunk index of row r is XOR-ed with bits of r so that 8 consecutive rows
// reading the same logical chunk hit 8 distinct bank groups.
//   row bytes 128 -> SWIZZLE_128B: chunk ^= r & 7
//   row bytes  64 -> SWIZZLE_64B : chunk ^= (r >> 1) & 3
//   row bytes  32 -> SWIZZLE_32B : chunk ^= (r >> 2) & 1
//   row bytes  16 -> no swizzle
// SW = 1 (tiles written by cp.async, never by TMA): 128-byte rows use the chunk
// permutation s(r) = 2 (r & 3) + ((r >> 2) & 1) instead of r & 7.  Both spread 8
// consecutive rows over the 8 bank groups; s also spreads the DMMA A-fragment load
// (a half-warp reads 4 rows x 2 adjacent chunks: {c ^ s(r)} hits 8 distinct groups,
// where r & 7 hits 4 twice -- a 2-way conflict on every fragment load).  64-byte rows
// likewise: s(r) = 2 ((r >> 1) & 1) + ((r >> 2) & 1) instead of (r >> 1) & 3.
template <int DP, int SW = 0>
struct TileLayout {
  static constexpr int PW = DP < 16 ? DP : 16;      // doubles per panel row
  static constexpr int RB = PW * 8;                 // bytes per panel row
  static constexpr int NPANEL = DP / PW;
  static constexpr int CH = PW / 2;                 // 16-byte chunks per panel row
  __device__ static __forceinline__ int swz(int r) {
    if constexpr (RB == 128 && SW == 1) return ((r & 3) << 1) | ((r >> 2) & 1);
    else if constexpr (RB == 128) return r & 7;
    else if constexpr (RB == 64 && SW == 1) return (((r >> 1) & 1) << 1) | ((r >> 2) & 1);
    else if constexpr (RB == 64) return (r >> 1) & 3;
    else if constexpr (RB == 32) return (r >> 2) & 1;
    else return 0;
  }
  // byte offset of logical 16-byte chunk q (0 <= q < DP/2) of row r, tile of R rows
  __device__ static __forceinline__ int chunk_off(int r, int q, int R) {
    const int p = q / CH, c = q % CH;
    return p * R * RB + r * RB + ((c ^ swz(r)) << 4);
  }
  // byte offset of element e of row r
  __device__ static __forceinline__ int elem_off(int r, int e, int R) {
    return chunk_off(r, e >> 1, R) + ((e & 1) << 3);
  }
  __host__ __device__ static constexpr int tile_bytes(int R) { return R * DP * 8; }
};

// ------------------------------------------------------------------ PTX bits
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// 2-D tensor TMA load: box at (col, row) of the tensor map into smem, completion on bar.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int col,
                                            int row) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(smem_u32(bar)), "r"(col), "r"(row)
      : "memory");
}

// 2-D tensor TMA prefetch of a box into L2 (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_l2_2d(const void* tmap, int col, int row) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tmap), "r"(col), "r"(row)
               : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// 16-byte async copy global -> shared (LDGSTS), bypassing L1.
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// Programmatic dependent launch: the iteration's kernels are launched with
// programmatic stream serialization, each lets its dependents launch as soon as it
// starts and waits (griddepcontrol.wait: full completion and visibility of the
// previous kernel) before touching any state, so launch latency overlaps the previous
// kernel's tail.  Both are no-ops for a kernel launched without the attribute.
#ifndef KNB_PDL
#define KNB_PDL 1
#endif
__device__ __forceinline__ void pdl_enter() {
#if KNB_PDL
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// shared-window address forms (no generic -> shared conversion per copy)
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8_s(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ int hi_word(double v) { return __double2hiint(v); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace knb
