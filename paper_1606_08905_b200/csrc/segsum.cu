// K3-wide: deterministic per-cluster accumulation when the k x d sums do not fit a
// CTA's shared memory (config 5: k x d = 256k doubles = 2 MB).
//
// The reference merges per-task accumulators in task order (centroids.py:88-107)
// and, in its running-sum mode, adds +x to the new and -x to the old cluster of
// every moved row (engine.py:345-353, :371-375).  Here the contributions of one
// pass are first ORDERED by cluster with a stable counting sort, then summed per
// cluster in that fixed order -- no floating-point atomics, bit-reproducible:
//
//   local    one warp per block of R rows: per-cluster counts and each entry's
//            rank inside its (block, cluster) bucket, 32 rows at a time with
//            __match_any_sync (entries of a chunk: all "+new" then all "-old")
//   scan     per cluster over blocks (exclusive), then over clusters: cluster
//            starts and work-item starts (chunks of CH entries)
//   place    entry -> its slot of the cluster-sorted array (row << 1 | negative)
//   items    one CTA per chunk of <= CH entries of one cluster: thread e sums
//            dimension e over the chunk in order (f32 or f64 rows, f64 sums),
//            plus the signed count and sum of ||x||^2
//   combine  one CTA per cluster: its chunk records in order -> exchange vector
// Work: full passes read every row once (d * elem bytes); dense passes after the
// first read only the moved rows (twice: + and -).
#include <math_constants.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

constexpr int SEG_R = 4096;   // rows per local block
constexpr int SEG_CH = 256;   // entries per work item

__device__ __forceinline__ bool seg_stopped(const Ctrl* c) { return c->stop && !c->ignore_stop; }

__global__ void seg_local_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  extern __shared__ int cnt[];
  const int lane = threadIdx.x;
  const long long b = blockIdx.x;
  for (int c = lane; c < a.k; c += 32) cnt[c] = 0;
  __syncwarp();
  const long long lo = b * SEG_R;
  const long long hi = lo + SEG_R < a.n ? lo + SEG_R : a.n;
  const unsigned lt = (1u << lane) - 1u;
  for (long long base = lo; base < hi; base += 32) {
    const long long r = base + lane;
    const bool valid = r < hi;
    const int nw = valid ? a.assign[r] : -1;
    const int od = (valid && a.mode == 1) ? a.old_assign[r] : -1;
    const int kp = (valid && (a.mode != 1 || od != nw)) ? nw : -1;
    const int km = (valid && a.mode == 1 && od != nw) ? od : -1;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {
      const int key = pass ? km : kp;
      const unsigned peers = __match_any_sync(0xffffffffu, key);
      const int cbase = key >= 0 ? cnt[key] : 0;
      __syncwarp();
      if (key >= 0) {
        a.lrank[2 * r + pass] = cbase + __popc(peers & lt);
        if (lane == __ffs(peers) - 1) cnt[key] = cbase + __popc(peers);
      }
      __syncwarp();
    }
  }
  for (int c = lane; c < a.k; c += 32) a.counts[(long long)c * a.B + b] = cnt[c];
}

// one CTA per cluster: exclusive scan of its per-block counts, total out
__global__ void seg_scan_blocks_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  __shared__ int wsum[32];
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int* row = a.counts + (long long)c * a.B;
  int carry = 0;
  for (int base = 0; base < a.B; base += blockDim.x) {
    const int i = base + tid;
    const int v = i < a.B ? row[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int s = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      wsum[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const int before = (w ? wsum[w - 1] : 0) + x - v;
    if (i < a.B) row[i] = carry + before;
    const int chunk_total = wsum[(blockDim.x >> 5) - 1];
    __syncthreads();
    carry += chunk_total;
  }
  if (tid == 0) a.ctot[c] = carry;
}

// single CTA: cluster starts and work-item starts (exclusive scans over k)
__global__ void seg_scan_clusters_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  __shared__ int ws[2][32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, nw = blockDim.x >> 5;
  int carry_s = 0, carry_i = 0;
  for (int base = 0; base < a.k; base += blockDim.x) {
    const int c = base + tid;
    const int t = c < a.k ? a.ctot[c] : 0;
    const int it = (t + SEG_CH - 1) / SEG_CH;
    int xs = t, xi = it;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ys = __shfl_up_sync(0xffffffffu, xs, o), yi = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) { xs += ys; xi += yi; }
    }
    if (lane == 31) { ws[0][w] = xs; ws[1][w] = xi; }
    __syncthreads();
    if (w == 0) {
      int ss = lane < nw ? ws[0][lane] : 0, si = lane < nw ? ws[1][lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ys = __shfl_up_sync(0xffffffffu, ss, o), yi = __shfl_up_sync(0xffffffffu, si, o);
        if (lane >= o) { ss += ys; si += yi; }
      }
      ws[0][lane] = ss;
      ws[1][lane] = si;
    }
    __syncthreads();
    const int bs = (w ? ws[0][w - 1] : 0) + xs - t, bi = (w ? ws[1][w - 1] : 0) + xi - it;
    if (c < a.k) {
      a.cstart[c] = carry_s + bs;
      a.istart[c] = carry_i + bi;
    }
    const int ts = ws[0][nw - 1], ti = ws[1][nw - 1];
    __syncthreads();
    carry_s += ts;
    carry_i += ti;
  }
  if (tid == 0) {
    a.cstart[a.k] = carry_s;
    a.istart[a.k] = carry_i;
  }
}

__global__ void seg_place_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < a.n;
       r += (long long)gridDim.x * blockDim.x) {
    const int nw = a.assign[r];
    const int od = a.mode == 1 ? a.old_assign[r] : -1;
    const long long b = r / SEG_R;
    if (a.mode != 1 || od != nw) {
      const long long pos = (long long)a.cstart[nw] + a.counts[(long long)nw * a.B + b] + a.lrank[2 * r];
      a.sorted[pos] = r << 1;
    }
    if (a.mode == 1 && od != nw) {
      const long long pos = (long long)a.cstart[od] + a.counts[(long long)od * a.B + b] + a.lrank[2 * r + 1];
      a.sorted[pos] = (r << 1) | 1;
    }
  }
}

template <typename T>
__global__ void seg_items_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  const int item = blockIdx.x;
  if (item >= a.istart[a.k]) return;
  // the cluster owning this item: last c with istart[c] <= item (empty clusters
  // share their successor's start and are skipped by taking the last)
  int lo = 0, hi = a.k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.istart[mid] <= item) lo = mid;
    else hi = mid - 1;
  }
  const int c = lo;
  const long long e0 = (long long)a.cstart[c] + (long long)(item - a.istart[c]) * SEG_CH;
  long long e1 = e0 + SEG_CH;
  if (e1 > a.cstart[c + 1]) e1 = a.cstart[c + 1];
  const T* X = static_cast<const T*>(a.X);
  const int d = a.d;
  double* rec = a.records + (long long)item * (d + 2);
  for (int e = threadIdx.x; e < d; e += blockDim.x) {
    double s = 0.0;
    long long i = e0;
    for (; i + 8 <= e1; i += 8) {  // eight row loads in flight, summed in entry order
      long long q[8];
      double v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) q[t] = a.sorted[i + t];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = (double)X[(q[t] >> 1) * d + e];
#pragma unroll
      for (int t = 0; t < 8; ++t) s += (q[t] & 1) ? -v[t] : v[t];
    }
    for (; i < e1; ++i) {
      const long long q = a.sorted[i];
      const double v = (double)X[(q >> 1) * d + e];
      s += (q & 1) ? -v : v;
    }
    rec[e] = s;
  }
  if (threadIdx.x == 0) {
    double cn = 0.0, sq = 0.0;
    for (long long i = e0; i < e1; ++i) {
      const long long q = a.sorted[i];
      const double w = a.xn2 ? a.xn2[q >> 1] : 0.0;
      if (q & 1) { cn -= 1.0; sq -= w; }
      else { cn += 1.0; sq += w; }
    }
    rec[d] = cn;
    rec[d + 1] = sq;
  }
}

__global__ void seg_combine_kernel(SegArgs a) {
  if (seg_stopped(a.ctrl)) return;
  const int c = blockIdx.x, d = a.d;
  const int i0 = a.istart[c], i1 = a.istart[c + 1];
  const long long kd = (long long)a.k * d;
  for (int e = threadIdx.x; e < d + 2; e += blockDim.x) {
    double s = 0.0;
    for (int i = i0; i < i1; ++i) s += a.records[(long long)i * (d + 2) + e];
    if (e < d) a.exch[(long long)c * d + e] = s;
    else if (e == d) a.exch[kd + c] = s;
    else a.exch[kd + a.k + c] = s;
  }
}

}  // namespace

int seg_blocks(long long n) { return (int)((n + SEG_R - 1) / SEG_R); }
long long seg_max_items(long long n, int k) { return (2 * n + SEG_CH - 1) / SEG_CH + k; }

cudaError_t launch_segsum(const SegArgs& a, int elem, cudaStream_t s) {
  if (a.n <= 0) {
    cudaError_t e = cudaMemsetAsync(a.exch, 0, sizeof(double) * ((size_t)a.k * a.d + 2 * (size_t)a.k), s);
    return e;
  }
  const size_t lsm = (size_t)a.k * sizeof(int);
  cudaError_t e = cudaSuccess;
  if (lsm > 48 * 1024) {
    e = cudaFuncSetAttribute(seg_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
    if (e != cudaSuccess) return e;
  }
  seg_local_kernel<<<a.B, 32, lsm, s>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  seg_scan_blocks_kernel<<<a.k, 256, 0, s>>>(a);
  seg_scan_clusters_kernel<<<1, 1024, 0, s>>>(a);
  {
    long long blocks = (a.n + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    seg_place_kernel<<<(int)blocks, 256, 0, s>>>(a);
  }
  const long long items = seg_max_items(a.n, a.k);
  int tpb = ((a.d + 31) / 32) * 32;
  if (tpb > 256) tpb = 256;
  if (elem == 4) seg_items_kernel<float><<<(unsigned)items, tpb, 0, s>>>(a);
  else seg_items_kernel<double><<<(unsigned)items, tpb, 0, s>>>(a);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  seg_combine_kernel<<<a.k, 128, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace knb
