// Staged copies between a caller's ordinary (pageable) host memory and HBM.
//
// A cudaMemcpy from pageable memory is staged by the driver through a pinned bounce
// buffer one chunk at a time, on one CPU thread: ~6 GB/s measured for config 4's 110 GB
// of rows.  Here W worker threads each own two pinned chunks and their own stream: a
// worker copies its next chunk of the caller's array into a free pinned chunk (CPU
// memcpy, in parallel across workers) while the copy engine moves its previous chunk,
// so CPU copying and DMA overlap and the copy is bound by the host link instead.  The
// pinned pool (W x 2 chunks) is allocated once per device and reused by every later
// copy (pinning memory is slow: ~1.4 GB/s).  Used by knb_upload_rows(_f32) and
// knb_get_assignments for transfers of STAGE_MIN (16 MB) bytes or more, in 8 MB chunks.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <cstdlib>
#include <unordered_map>
#include <vector>

#include "kernels.h"

namespace knb {

namespace {

// chunk size and worker count: KNB_STAGE_CHUNK_MB / KNB_STAGE_WORKERS override the
// defaults (read once, when the pool is built)
size_t g_chunk = 8ull << 20;  // bytes per pinned chunk
int g_workers = 8;
void read_stage_env() {
  static bool done = false;
  if (done) return;
  done = true;
  if (const char* v = std::getenv("KNB_STAGE_CHUNK_MB")) {
    const long mb = std::atol(v);
    if (mb >= 1 && mb <= 256) g_chunk = (size_t)mb << 20;
  }
  if (const char* v = std::getenv("KNB_STAGE_WORKERS")) {
    const int w = std::atoi(v);
    if (w >= 1 && w <= 64) g_workers = w;
  }
}

struct Pool {
  std::vector<char*> buf;           // 2 per worker
  std::vector<cudaStream_t> stream; // 1 per worker
  std::vector<cudaEvent_t> done;    // 2 per worker: the last copy out of / into that chunk
  std::mutex use;                   // one staged copy at a time per device
};

std::mutex g_mu;
std::unordered_map<int, Pool*> g_pools;

cudaError_t pool_for(int device, Pool** out) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto it = g_pools.find(device);
  if (it != g_pools.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  read_stage_env();
  Pool* p = new Pool();
  cudaError_t e = cudaSuccess;
  for (int w = 0; w < g_workers && e == cudaSuccess; ++w) {
    cudaStream_t s = nullptr;
    e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) break;
    p->stream.push_back(s);
    for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
      char* h = nullptr;
      e = cudaHostAlloc(reinterpret_cast<void**>(&h), g_chunk, cudaHostAllocPortable);
      if (e != cudaSuccess) break;
      p->buf.push_back(h);
      cudaEvent_t ev = nullptr;
      e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventRecord(ev, s);  // starts completed
      p->done.push_back(ev);
    }
  }
  if (e != cudaSuccess) {  // leave nothing half-built behind; the caller falls back to cudaMemcpy
    for (char* h : p->buf) cudaFreeHost(h);
    for (cudaEvent_t ev : p->done) if (ev) cudaEventDestroy(ev);
    for (cudaStream_t s : p->stream) cudaStreamDestroy(s);
    delete p;
    cudaGetLastError();
    return e;
  }
  g_pools[device] = p;
  *out = p;
  return cudaSuccess;
}

}  // namespace

cudaError_t staging_reserve(int device) {
  Pool* p = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  return pool_for(device, &p);
}

// dst / src: device pointer on one side, pageable host pointer on the other (h2d says
// which).  Synchronous: returns once every byte has landed.
cudaError_t staged_copy(int device, void* dst, const void* src, size_t bytes, bool h2d) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  // page-locked host memory (cudaHostAlloc / registered, e.g. a pinned torch tensor):
  // the copy engine reads it directly
  cudaPointerAttributes at;
  const void* host = h2d ? src : dst;
  const bool pinned = cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost;
  cudaGetLastError();
  Pool* p = nullptr;
  if (pinned || bytes < STAGE_MIN || pool_for(device, &p) != cudaSuccess) {
    e = cudaMemcpy(dst, src, bytes, h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost);
    // From pageable memory an H2D cudaMemcpy returns once the source is staged, possibly
    // before its DMA has landed, and only the legacy stream is ordered after that DMA; the
    // caller's kernels run on a non-blocking stream, so wait for it here (a check of the
    // rows right after an upload read the tail of a previous allocation otherwise).
    if (e == cudaSuccess && h2d && !pinned) e = cudaStreamSynchronize(cudaStreamLegacy);
    return e;
  }
  std::lock_guard<std::mutex> lock(p->use);
  const size_t CHUNK = g_chunk;
  const size_t nchunks = (bytes + CHUNK - 1) / CHUNK;
  const int W = (int)std::min<size_t>((size_t)p->stream.size(), nchunks);
  std::atomic<int> err{(int)cudaSuccess};
  auto worker = [&](int w) {
    cudaError_t le = cudaSetDevice(device);
    int b = 0;
    for (size_t i = w; i < nchunks && le == cudaSuccess && err.load() == (int)cudaSuccess; i += W, b ^= 1) {
      const size_t off = i * CHUNK, len = std::min(CHUNK, bytes - off);
      char* buf = p->buf[2 * w + b];
      cudaEvent_t ev = p->done[2 * w + b];
      le = cudaEventSynchronize(ev);  // the chunk's previous copy has finished
      if (le != cudaSuccess) break;
      if (h2d) {
        std::memcpy(buf, static_cast<const char*>(src) + off, len);
        le = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, p->stream[w]);
        if (le == cudaSuccess) le = cudaEventRecord(ev, p->stream[w]);
      } else {
        le = cudaMemcpyAsync(buf, static_cast<const char*>(src) + off, len, cudaMemcpyDeviceToHost, p->stream[w]);
        if (le == cudaSuccess) le = cudaStreamSynchronize(p->stream[w]);
        if (le == cudaSuccess) std::memcpy(static_cast<char*>(dst) + off, buf, len);
      }
    }
    if (le == cudaSuccess) le = cudaStreamSynchronize(p->stream[w]);
    if (le != cudaSuccess) {
      int ok = (int)cudaSuccess;
      err.compare_exchange_strong(ok, (int)le);
    }
  };
  std::vector<std::thread> th;
  for (int w = 1; w < W; ++w) th.emplace_back(worker, w);
  worker(0);
  for (auto& t : th) t.join();
  return (cudaError_t)err.load();
}

}  // namespace knb
