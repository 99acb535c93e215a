// Semi-external (rows beyond HBM) I/O accounting and the HBM row cache.
//
// The rows live in host memory (read once from the matrix file, page-locked and
// mapped); HBM holds the O(n) state plus a row cache.  Per iteration this file
//   * marks the rows the iteration fetches (numakmeans outofcore.py:_DiskSource):
//     a full pass fetches every row (task_rows, engine.py:285-290), a pruned pass
//     the survivors of clause 1 (rows_by_ids, engine.py:321-334);
//   * reproduces the reference's I/O counters exactly (fetch_rows,
//     outofcore.py:163-225): bytes_requested = row_bytes per fetched row, cache
//     hits / misses against the published cache, bytes_read = page_size x the
//     distinct pages touched by the uncached fetched rows of each fetch call (one
//     call per task: page_runs, outofcore.py:118-145, is the union of the rows' page
//     intervals);
//   * at refresh iterations t = start, 3 start, 7 start, ... (should_refresh,
//     outofcore.py:282-290) rebuilds the cache exactly like RowCache.rebuild
//     (outofcore.py:250-270): flush, then each worker partition keeps its smallest
//     rows_per_partition fetched row ids; the rows are copied into HBM and later
//     passes gather them from there instead of over the host link.
// Every kernel reads the iteration index from the device control block, so the
// work is graph-capturable and skipped once the run has stopped.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "kernels.h"

namespace knb {

namespace {

constexpr int SEM_B = 1024;  // rows per block of the rebuild scan
__host__ __device__ __forceinline__ int rebuild_blocks(long long n) { return (int)((n + SEM_B - 1) / SEM_B); }

__device__ __forceinline__ bool halted(const Ctrl* c) { return c->stop && !c->ignore_stop; }

__device__ __forceinline__ bool refresh_at(long long t, int start) {
  if (start < 1 || t < start || t % start != 0) return false;
  const long long q = t / start + 1;
  return (q & (q - 1)) == 0;
}

// worker partition of a row: partition_rows (matrix.py:196-213), sizes base+1 then base
__device__ __forceinline__ int part_of(long long r, long long base, long long rem) {
  const long long big = rem * (base + 1);
  if (r < big) return (int)(r / (base + 1));
  return (int)(rem + (r - big) / base);
}
__device__ __forceinline__ long long part_lo(int w, long long base, long long rem) {
  return (long long)w * base + (w < rem ? w : rem);
}

__device__ __forceinline__ bool io_slot(const SemArgs& s, long long* t_out) {
  const long long t = s.ctrl->t;
  *t_out = t;
  return t >= 0 && t < s.max_iters;
}

template <typename T>
__device__ __forceinline__ void block_add(T v, T* red, T* dst) {
  v = (T)warp_sum_ll((long long)v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T s = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    if (s) atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)s);
  }
}

// first / last page of a row (page arithmetic relative to the payload)
struct PageMath {
  long long rb, ps;
  int shift;  // log2(ps) when ps is a power of two, else -1
  __device__ __forceinline__ long long page(long long byte) const {
    return shift >= 0 ? byte >> shift : byte / ps;
  }
};

// start row of the task holding row r (partition ranges split by task_size)
__device__ __forceinline__ long long task_start(const SemArgs& s, long long r) {
  const int w = part_of(r, s.pbase, s.prem);
  const long long lo = part_lo(w, s.pbase, s.prem);
  return lo + (r - lo) / s.task_size * s.task_size;
}

// One fused pass over the pre-pass state: marks the rows this iteration fetches and
// counts rows requested, cache hits / misses and pages read.  A warp walks a
// contiguous range of rows 32 at a time; a miss row adds the pages of its byte
// interval not already covered by the previous miss row of the same task (page_runs'
// union, outofcore.py:118-145); the previous miss row comes from the ballot, or for
// a range's first rows from a short look-back over the rows sharing its first page.

constexpr int SEM_Q = 4;  // 32-row chunks per step of the account walk

__device__ __forceinline__ bool fetch_of(const SemArgs& s, bool full, long long r) {
  if (full) return true;
  const int a = s.assign[r];
  return !(s.upper[r] + s.drift[a] <= s.half_min[a]);  // the filter's inflate + clause 1
}

__global__ void __launch_bounds__(KNB_NT) sem_account_kernel(const SemArgs s, const int ps_shift,
                                                             const long long range) {
  __shared__ long long red[4][KNB_NT / 32];
  if (halted(s.ctrl)) return;
  long long t;
  if (!io_slot(s, &t)) return;
  const bool full = !s.pruning || s.ctrl->full_pass;
  const PageMath pm{s.row_bytes, s.page_size, ps_shift};
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long tw = ((long long)gridDim.x * blockDim.x) >> 5;
  long long req = 0, hit = 0, miss = 0, pages = 0;
  auto is_miss = [&](long long r, bool f) { return f && !(s.cache_enabled && s.cslot[r] >= 0); };
  for (long long lo = gw * range; lo < s.n; lo += tw * range) {
    const long long hi = lo + range < s.n ? lo + range : s.n;
    // previous miss row before the range that can share a page with its first row
    long long carry = -1;
    if (lo > 0) {
      const long long r0 = pm.page(lo * pm.rb) * pm.ps / pm.rb;  // first row touching that page
      for (long long top = lo - 1; top >= r0 && carry < 0; top -= 32) {
        const long long j = top - lane;
        const bool m = j >= r0 && is_miss(j, fetch_of(s, full, j));
        const unsigned b = __ballot_sync(0xffffffffu, m);
        if (b) carry = top - (__ffs(b) - 1);
      }
    }
    for (long long c0 = lo; c0 < hi; c0 += 32 * SEM_Q) {
      // issue SEM_Q rows' loads per lane before the first use (memory-level parallelism)
      int av[SEM_Q];
      double uv[SEM_Q];
#pragma unroll
      for (int q = 0; q < SEM_Q; ++q) {
        const long long i = c0 + 32 * q + lane;
        av[q] = (!full && i < hi) ? __ldg(s.assign + i) : 0;
        uv[q] = (!full && i < hi) ? __ldg(s.upper + i) : 0.0;
      }
      bool fv[SEM_Q];
      int sv[SEM_Q];
#pragma unroll
      for (int q = 0; q < SEM_Q; ++q) {
        const long long i = c0 + 32 * q + lane;
        fv[q] = i < hi && (full || !(uv[q] + __ldg(s.drift + av[q]) <= __ldg(s.half_min + av[q])));
        sv[q] = (fv[q] && s.cache_enabled) ? s.cslot[i] : -1;
      }
#pragma unroll
      for (int q = 0; q < SEM_Q; ++q) {
        const long long c = c0 + 32 * q, i = c + lane;
        const bool f = fv[q], m = f && sv[q] < 0;
        if (i < hi) s.fetched[i] = f ? 1 : 0;
        if (f) {
          ++req;
          if (s.cache_enabled) { if (m) ++miss; else ++hit; }
        }
        const unsigned b = __ballot_sync(0xffffffffu, m);
        if (m) {
          const unsigned below = b & ((1u << lane) - 1u);
          const long long j = below ? c + (31 - __clz(below)) : carry;
          const long long first = pm.page(i * pm.rb), last = pm.page(i * pm.rb + pm.rb - 1);
          long long from = first;
          if (j >= 0 && task_start(s, j) == task_start(s, i)) {
            const long long lj = pm.page(j * pm.rb + pm.rb - 1);
            if (lj + 1 > from) from = lj + 1;
          }
          pages += last - from + 1;
        }
        if (b) carry = c + (31 - __clz(b));
      }
    }
  }
  long long* io = s.io + t * 4;
  block_add(req, red[0], io + 0);
  block_add(pages, red[1], io + 1);
  block_add(hit, red[2], io + 2);
  block_add(miss, red[3], io + 3);
}

__device__ __forceinline__ bool rebuilding(const SemArgs& s, long long* t) {
  if (!s.cache_enabled || s.rows_per_part <= 0 || halted(s.ctrl)) return false;
  *t = s.ctrl->t;
  return refresh_at(*t, s.refresh_start);
}

// flush + per-block fetched counts
__global__ void sem_count_kernel(const SemArgs s) {
  long long t;
  if (!rebuilding(s, &t)) return;
  const long long slots = (long long)s.T * s.rows_per_part;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < slots; j += (long long)gridDim.x * blockDim.x)
    s.crow[j] = -1;
  __shared__ long long red[KNB_NT / 32];
  const int nb = rebuild_blocks(s.n);
  for (int blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const long long lo = (long long)blk * SEM_B;
    int c = 0;
    for (long long i = lo + threadIdx.x; i < lo + SEM_B && i < s.n; i += blockDim.x) {
      s.cslot[i] = -1;
      c += s.fetched[i];
    }
    const long long v = warp_sum_ll(c);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      long long sum = 0;
      for (int w = 0; w < KNB_NT / 32; ++w) sum += red[w];
      s.bcount[blk] = sum;
    }
    __syncthreads();
  }
}

// exclusive scan of the block counts (one CTA) and each partition's first prefix
__global__ void sem_scan_kernel(const SemArgs s, int nb) {
  long long t;
  if (!rebuilding(s, &t)) return;
  __shared__ long long carry;
  __shared__ long long wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    const int b = b0 + threadIdx.x;
    const long long v = b < nb ? s.bcount[b] : 0;
    long long x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      long long z = lane < nw ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      if (lane < nw) wsum[lane] = z;
    }
    __syncthreads();
    const long long incl = x + (w ? wsum[w - 1] : 0) + carry;
    if (b < nb) s.bpre[b] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  // fetched rows before each partition's first row
  for (int p = threadIdx.x; p < s.T; p += blockDim.x) {
    const long long lo = part_lo(p, s.pbase, s.prem);
    if (lo >= s.n) { s.plo[p] = 0; continue; }
    const long long b = lo / SEM_B;
    long long v = s.bpre[b];
    for (long long i = b * SEM_B; i < lo; ++i) v += s.fetched[i];
    s.plo[p] = v;
  }
}

// each partition's first rows_per_part fetched rows (ascending id) get cache slots
__global__ void sem_mark_kernel(const SemArgs s) {
  long long t;
  if (!rebuilding(s, &t)) return;
  __shared__ int wcnt[SEM_B / 32];
  const int lane = threadIdx.x & 31;
  const int nb = rebuild_blocks(s.n);
  // blockDim.x == SEM_B: one row per thread
  for (int blk = blockIdx.x; blk < nb; blk += gridDim.x) {
    const long long i = (long long)blk * SEM_B + threadIdx.x;
    const bool f = i < s.n && s.fetched[i];
    const unsigned b = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[threadIdx.x >> 5] = __popc(b);
    __syncthreads();
    if (f) {
      long long pos = s.bpre[blk] + __popc(b & ((1u << lane) - 1u));
      for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) pos += wcnt[w];
      const int p = part_of(i, s.pbase, s.prem);
      const long long rank = pos - s.plo[p];
      if (rank < s.rows_per_part) {
        const long long slot = (long long)p * s.rows_per_part + rank;
        s.cslot[i] = (int32_t)slot;
        s.crow[slot] = i;
      }
    }
    __syncthreads();
  }
}

// copy the selected rows into the HBM cache (one warp per slot)
__global__ void sem_fill_kernel(const SemArgs s) {
  long long t;
  if (!rebuilding(s, &t)) return;
  const long long slots = (long long)s.T * s.rows_per_part;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long tw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long j = gw; j < slots; j += tw) {
    const long long r = s.crow[j];
    if (r < 0) continue;
    const double* src = s.X + r * s.d;
    double* dst = s.cache + j * s.d;
    for (int e = lane; e < s.d; e += 32) dst[e] = src[e];
  }
}

}  // namespace

int sem_rebuild_blocks(long long n) { return rebuild_blocks(n); }

cudaError_t launch_sem_account(const SemArgs& s, int sms, cudaStream_t st) {
  // enough warps to fill every SM (the walk is latency-bound), ranges of 128..4096 rows
  long long range = s.n / (64LL * sms) / 128 * 128;
  range = range < 128 ? 128 : (range > 4096 ? 4096 : range);
  const long long ranges = (s.n + range - 1) / range;
  const long long want = (ranges + KNB_WARPS - 1) / KNB_WARPS;
  const int g = (int)(want < 8LL * sms ? (want > 0 ? want : 1) : 8LL * sms);
  int shift = -1;
  if ((s.page_size & (s.page_size - 1)) == 0)
    for (shift = 0; (1LL << shift) < s.page_size; ++shift) {}
  sem_account_kernel<<<g, KNB_NT, 0, st>>>(s, shift, range);
  return cudaGetLastError();
}

cudaError_t launch_sem_rebuild(const SemArgs& s, int sms, cudaStream_t st) {
  if (!s.cache_enabled || s.rows_per_part <= 0) return cudaSuccess;
  const int nb = sem_rebuild_blocks(s.n);
  const int g1 = nb < 4 * sms ? nb : 4 * sms;  // grid-stride: cheap to launch when not refreshing
  sem_count_kernel<<<g1, KNB_NT, 0, st>>>(s);
  sem_scan_kernel<<<1, 1024, 0, st>>>(s, nb);
  sem_mark_kernel<<<nb < 2 * sms ? nb : 2 * sms, SEM_B, 0, st>>>(s);
  const long long slots = (long long)s.T * s.rows_per_part;
  const long long want = (slots * 32 + KNB_NT - 1) / KNB_NT;
  const int g = (int)(want < 8LL * sms ? want : 8LL * sms);
  sem_fill_kernel<<<g > 0 ? g : 1, KNB_NT, 0, st>>>(s);
  return cudaGetLastError();
}

}  // namespace knb
