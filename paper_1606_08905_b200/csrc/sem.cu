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

// fetched mask + requested / hit / miss counts
__global__ void sem_mask_kernel(const SemArgs s) {
  __shared__ long long red[3][KNB_NT / 32];
  if (halted(s.ctrl)) return;
  long long t;
  if (!io_slot(s, &t)) return;
  const bool full = !s.pruning || s.ctrl->full_pass;
  long long req = 0, hit = 0, miss = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < s.n; i += (long long)gridDim.x * blockDim.x) {
    bool f = true;
    if (!full) {
      const int a = s.assign[i];
      f = !(s.upper[i] + s.drift[a] <= s.half_min[a]);  // the filter's inflate + clause 1
    }
    s.fetched[i] = f ? 1 : 0;
    if (f) {
      ++req;
      if (s.cache_enabled) {
        if (s.cslot[i] >= 0) ++hit;
        else ++miss;
      }
    }
  }
  long long* io = s.io + t * 4;
  block_add(req, red[0], io + 0);
  block_add(hit, red[1], io + 2);
  block_add(miss, red[2], io + 3);
}

// pages read: per page, the number of distinct tasks with an uncached fetched row on it
__global__ void sem_pages_kernel(const SemArgs s) {
  __shared__ long long red[KNB_NT / 32];
  if (halted(s.ctrl)) return;
  long long t;
  if (!io_slot(s, &t)) return;
  const long long rb = s.row_bytes, ps = s.page_size;
  const long long npages = (s.n * rb + ps - 1) / ps;
  long long pages = 0;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < npages; p += (long long)gridDim.x * blockDim.x) {
    const long long r0 = p * ps / rb;
    long long r1 = ((p + 1) * ps - 1) / rb;
    if (r1 > s.n - 1) r1 = s.n - 1;
    long long task_end = -1, last_task = -1;
    for (long long r = r0; r <= r1; ++r) {
      if (!s.fetched[r]) continue;
      if (s.cache_enabled && s.cslot[r] >= 0) continue;
      if (r >= task_end) {  // locate the task holding r: tasks split each partition by task_size
        const int w = part_of(r, s.pbase, s.prem);
        const long long lo = part_lo(w, s.pbase, s.prem);
        const long long hi = part_lo(w + 1, s.pbase, s.prem);
        const long long ts = lo + (r - lo) / s.task_size * s.task_size;
        task_end = ts + s.task_size < hi ? ts + s.task_size : hi;
        if (ts != last_task) { ++pages; last_task = ts; }
      }
    }
  }
  block_add(pages, red, s.io + t * 4 + 1);
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
  const long long lo = (long long)blockIdx.x * SEM_B;
  int c = 0;
  for (long long i = lo + threadIdx.x; i < lo + SEM_B && i < s.n; i += blockDim.x) {
    s.cslot[i] = -1;
    c += s.fetched[i];
  }
  __shared__ long long red[KNB_NT / 32];
  long long v = warp_sum_ll(c);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long sum = 0;
    for (int w = 0; w < KNB_NT / 32; ++w) sum += red[w];
    s.bcount[blockIdx.x] = sum;
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
  const long long lo = (long long)blockIdx.x * SEM_B;
  const int lane = threadIdx.x & 31;
  // blockDim.x == SEM_B: one row per thread
  const long long i = lo + threadIdx.x;
  const bool f = i < s.n && s.fetched[i];
  const unsigned b = __ballot_sync(0xffffffffu, f);
  if (lane == 0) wcnt[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (!f) return;
  long long pos = s.bpre[blockIdx.x] + __popc(b & ((1u << lane) - 1u));
  for (int w = 0; w < (int)(threadIdx.x >> 5); ++w) pos += wcnt[w];
  const int p = part_of(i, s.pbase, s.prem);
  const long long rank = pos - s.plo[p];
  if (rank < s.rows_per_part) {
    const long long slot = (long long)p * s.rows_per_part + rank;
    s.cslot[i] = (int32_t)slot;
    s.crow[slot] = i;
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

int sem_rebuild_blocks(long long n) { return (int)((n + SEM_B - 1) / SEM_B); }

cudaError_t launch_sem_account(const SemArgs& s, int sms, cudaStream_t st) {
  const long long want = (s.n + KNB_NT - 1) / KNB_NT;
  const int g = (int)(want < 8LL * sms ? (want > 0 ? want : 1) : 8LL * sms);
  sem_mask_kernel<<<g, KNB_NT, 0, st>>>(s);
  const long long npages = (s.n * s.row_bytes + s.page_size - 1) / s.page_size;
  const long long wp = (npages + KNB_NT - 1) / KNB_NT;
  const int gp = (int)(wp < 8LL * sms ? (wp > 0 ? wp : 1) : 8LL * sms);
  sem_pages_kernel<<<gp, KNB_NT, 0, st>>>(s);
  return cudaGetLastError();
}

cudaError_t launch_sem_rebuild(const SemArgs& s, int sms, cudaStream_t st) {
  if (!s.cache_enabled || s.rows_per_part <= 0) return cudaSuccess;
  const int nb = sem_rebuild_blocks(s.n);
  sem_count_kernel<<<nb, KNB_NT, 0, st>>>(s);
  sem_scan_kernel<<<1, 1024, 0, st>>>(s, nb);
  sem_mark_kernel<<<nb, SEM_B, 0, st>>>(s);
  const long long slots = (long long)s.T * s.rows_per_part;
  const long long want = (slots * 32 + KNB_NT - 1) / KNB_NT;
  const int g = (int)(want < 8LL * sms ? want : 8LL * sms);
  sem_fill_kernel<<<g > 0 ? g : 1, KNB_NT, 0, st>>>(s);
  return cudaGetLastError();
}

}  // namespace knb
