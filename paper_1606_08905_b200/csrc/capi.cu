// C ABI of libknorb200.so (declared in include/knor_b200.h).
//
// One knb_ctx = one GPU's row shard and all of its device state.  Everything is
// enqueued on the context stream; only calls that hand data back to the host
// synchronise.  No CPU fallback exists: every failure is reported.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <mutex>
#include <unordered_map>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/knor_b200.h"
#include "kernels.h"

using namespace knb;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define KNB_CUDA(call)                                                                      \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      return fail(e_ == cudaErrorMemoryAllocation ? KNB_E_NOMEM : KNB_E_CUDA,              \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                     \
  } while (0)

constexpr size_t SMEM_LIMIT = 227 * 1024;
// certified relative error of one kind::tf32 dot product (assign_tc.cu header): the
// tensor core truncates operands to 10 mantissa bits (tools/tf32_probe.py measures the
// rounding direction); the centroid operand is pre-rounded to nearest TF32 by
// tc_prep_kernel (<= 2^-11 + 2^-24 from the f64 means), so a product is off by
// < 2^-10 + 2^-11 + 2^-21 = 0.75 * 2^-9 relative and the f32 sums by < 2^-15 of
// sum |x_i c_i|; 0.9375 * 2^-9 covers both with the same ~20% margin as before
// (truncating both operands needed 1.25 * 2^-9)
constexpr double KNB_TF32_ERR = 0x1.ep-10;

}  // namespace

// error reporting shared with the context-free entry points (primitives.cu)
namespace knb {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace knb

struct knb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // one steady-state iteration (t >= 1: MTI / delta pass + finish) as a CUDA graph,
  // replayed by knb_run / knb_enqueue; rebuilt when buffers or options change
  cudaStream_t cap_stream = nullptr;
  cudaGraphExec_t graph = nullptr;
  bool graph_valid = false;
  long long n_global = 0, n_local = 0, row_lo = 0;
  int d = 0, k = 0, pruning = 0, max_iters = 1;
  double tolerance = 0.0;
  int sms = 148;

  const double* X = nullptr;
  double* X_own = nullptr;
  const void* host_registered = nullptr;  // knb_attach_host_rows: pinned + mapped caller rows
  CUtensorMap tmap;
  int use_tma = 0;

  // f32 rows on the tcgen05 path (assign_tc.cu + segsum.cu)
  int elem = 8;
  const float* X32 = nullptr;
  float* X32_own = nullptr;
  bool tc = false;
  CUtensorMap tmX32, tmC32;
  int kp = 0, dp = 0, nkc = 0, nnt = 0, G_tc = 1;
  float *c32 = nullptr, *chn32 = nullptr;
  double* xn2 = nullptr;
  bool xn_valid = false;
  int32_t* old_assign = nullptr;
  float* tc_bound = nullptr;
  TcHalf* tc_scratch = nullptr;
  int4* tcq = nullptr;
  int* tc_fullq = nullptr;
  int* tcq_count = nullptr;
  long long tcq_cap = 0;
  unsigned long long* tc_counters = nullptr;
  SegArgs seg;

  // f64 rows, d = 16: the split-TF32 tcgen05 MTI pass (mti_tc.cu)
  int tcx_nx = 0;                  // f64 ring stages, 0 = not applicable
  CUtensorMap tmX128;              // 128-row boxes of the f64 rows
  bool tcx_map = false;
  void* tcx_bimg = nullptr;        // B operand image
  unsigned char* tcx_recs = nullptr;  // per-tile moved-row records (mti_tc_delta_kernel)
  unsigned long long* tcx_counters = nullptr;
  long long* tcx_rq = nullptr;     // uncertified-row queue ({row, old id} pairs) and its count
  unsigned long long* tcx_rq_count = nullptr;
  long long tcx_rq_cap = 0;

  int DP = 0, DPm = 0, half_in_smem = 0;
  int G_dense = 1, G_mti = 1, G_mti_mma = 1;
  int mti_scan = 0;   // KNB_MTI_AUTO / KNB_MTI_EXACT / KNB_MTI_DENSE
  bool mti_mma_ok = false;

  int32_t* assign = nullptr;
  double* upper = nullptr;
  uint8_t* tight = nullptr;
  double *means = nullptr, *prev = nullptr, *drift = nullptr, *counts = nullptr, *chn = nullptr,
         *cn2 = nullptr, *half = nullptr, *half_min = nullptr, *wterm = nullptr, *run = nullptr,
         *stage = nullptr;
  double* exch = nullptr;
  bool own_exch = true;
  long long L = 0;
  double* partials = nullptr;  // allocated on first use by an f64 pass
  int G_alloc = 0;
  Ctrl* ctrl = nullptr;
  unsigned int* fin_sync = nullptr;
  IterStatsDev* stats = nullptr;
  long long* bad = nullptr;
  long long* ids_dev = nullptr;
  int ids_cap = 0;
  double* d2 = nullptr;
  double* kpp_bs = nullptr;
  double* kpp_scalar = nullptr;
  long long* kpp_idx = nullptr;
  int kpp_nblk = 0;

  // semi-external runs (knb_sem_configure): I/O accounting + HBM row cache (sem.cu)
  bool sem = false;
  SemArgs semA;
  int sem_nb = 0;

  long long t_host = 0;
  bool centroids_set = false;
  long long bytes = 0;
  std::unordered_set<void*> pooled;  // allocations from the library's stream-ordered pool
};

namespace {

// One stream-ordered memory pool per device for every context's buffers: a context's
// create / destroy then costs no cudaMalloc / cudaFree (each an implicit device
// synchronisation) once the pool holds the memory -- repeated kmeans() calls reuse it.
// Like torch's caching allocator, the pool keeps what it has mapped (returning ~100 GB to
// the driver took 0.6-0.8 s inside knb_destroy, i.e. inside every large kmeans() call;
// a background trim instead contended with the next call's mapping): knb_release_memory
// hands the unused part back (Python: release_memory(), as torch.cuda.empty_cache), and
// the pool's unused memory is reused by the next context's allocations.
cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static std::unordered_map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(device);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool = nullptr;
  if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
    cudaGetLastError();
    pool = nullptr;
  } else {
    uint64_t keep = ~0ULL;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  pools[device] = pool;
  return pool;
}

template <typename T>
int dev_alloc(knb_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  const size_t bytes = count * sizeof(T);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(c->stream, &cs);
  cudaMemPool_t pool = cs == cudaStreamCaptureStatusNone ? lib_pool(c->device) : nullptr;
  cudaError_t e;
  if (pool) {
    e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), bytes, pool, c->stream);
    if (e == cudaSuccess) {
      c->pooled.insert(*p);
      // usable from any stream and by synchronous copies from here on
      e = cudaStreamSynchronize(c->stream);
    }
  } else {
    e = cudaMalloc(reinterpret_cast<void**>(p), bytes);  // inside a capture: a plain allocation
  }
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? KNB_E_NOMEM : KNB_E_CUDA,
                std::string("device allocation (") + std::to_string(bytes) + " B): " + cudaGetErrorString(e));
  c->bytes += (long long)bytes;
  return KNB_OK;
}

void dev_free(knb_ctx* c, void* p) {
  if (!p) return;
  if (c->pooled.erase(p)) cudaFreeAsync(p, c->stream);
  else cudaFree(p);
}

FinalArgs final_args(knb_ctx* c) {
  FinalArgs f;
  f.k = c->k;
  f.d = c->d;
  f.n = c->n_global;
  f.pruning = c->pruning;
  f.exch = c->exch;
  f.run = c->run;
  f.means = c->means;
  f.prev = c->prev;
  f.drift = c->drift;
  f.counts = c->counts;
  f.chn = c->chn;
  f.cn2 = c->cn2;
  f.half = c->half;
  f.half_min = c->half_min;
  f.wterm = c->wterm;
  f.wcss_mode = c->tc ? 2 : (c->pruning ? 1 : 0);
  f.sync = c->fin_sync;
  f.ctrl = c->ctrl;
  f.stats = c->stats;
  return f;
}

// fresh run state: iteration 0, not stopped, assignment zero, running sums zero
int reset_run(knb_ctx* c) {
  Ctrl h;
  std::memset(&h, 0, sizeof(h));
  h.full_pass = 1;
  // the pruned pass streams every row (tcgen05 pass, or the DMMA block pass) while clause 1
  // skips fewer than this share of rows, and compacts the survivors above it (measured: the
  // tcgen05 pass at c2's 49% / c3's 41% skips runs 0.226 / 2.16 ms against the compacted
  // DMMA pass's 0.167 / 1.22 ms -- its per-row epilogue work does not shrink with skips)
  h.block_pct = 10;
  h.max_iters = c->max_iters;
  h.tolerance = c->tolerance;
  KNB_CUDA(cudaMemcpyAsync(c->ctrl, &h, offsetof(Ctrl, cmax2), cudaMemcpyHostToDevice, c->stream));
  KNB_CUDA(cudaMemsetAsync(c->assign, 0, sizeof(int32_t) * (c->n_local ? c->n_local : 1), c->stream));
  KNB_CUDA(cudaMemsetAsync(c->run, 0, sizeof(double) * c->L, c->stream));
  if (c->tc_counters) KNB_CUDA(cudaMemsetAsync(c->tc_counters, 0, 4 * sizeof(unsigned long long), c->stream));
  if (c->tcx_counters) KNB_CUDA(cudaMemsetAsync(c->tcx_counters, 0, sizeof(unsigned long long), c->stream));
  if (c->sem) {  // a new run starts with an empty cache and zero I/O counters
    KNB_CUDA(cudaMemsetAsync(c->semA.io, 0, sizeof(long long) * 4 * c->max_iters, c->stream));
    KNB_CUDA(cudaMemsetAsync(c->semA.cslot, 0xff, sizeof(int32_t) * (c->n_local ? c->n_local : 1), c->stream));
  }
  c->t_host = 0;
  return KNB_OK;
}

int build_tmap(knb_ctx* c) {
  c->use_tma = 0;
  c->tcx_map = false;
  if (c->host_registered) return KNB_OK;  // rows in host memory: cp.async gathers, no tensor maps
  if (c->DP == 0 || (c->d & 1) || (reinterpret_cast<uintptr_t>(c->X) & 15) || c->n_local < 1 ||
      c->n_local > 0x7fffffffLL)
    return KNB_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      fn == nullptr || q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return KNB_OK;  // cp.async loader instead (same layout)
  }
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int PW = c->DP < 16 ? c->DP : 16;
  const int R = dense_rows_per_tile(c->DP);
  const int BR = R < 256 ? R : 256;
  cuuint64_t gdim[2] = {(cuuint64_t)c->d, (cuuint64_t)c->n_local};
  cuuint64_t gstride[1] = {(cuuint64_t)c->d * 8};
  cuuint32_t box[2] = {(cuuint32_t)PW, (cuuint32_t)BR};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
  if (PW * 8 == 128) sw = CU_TENSOR_MAP_SWIZZLE_128B;
  else if (PW * 8 == 64) sw = CU_TENSOR_MAP_SWIZZLE_64B;
  else if (PW * 8 == 32) sw = CU_TENSOR_MAP_SWIZZLE_32B;
  CUresult r = encode(&c->tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(c->X), gdim, gstride,
                      box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r == CUDA_SUCCESS) c->use_tma = 1;
  c->tcx_map = false;
  if (c->use_tma && c->tcx_nx > 0) {
    // the tcgen05 MTI pass: 128-row boxes, 16 columns (128 B, SWIZZLE_128B; d = 32 takes
    // two per tile) or the whole 8-column row (64 B, SWIZZLE_64B)
    cuuint32_t box128[2] = {c->d == 8 ? 8u : 16u, 128u};
    r = encode(&c->tmX128, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(c->X), gdim, gstride, box128,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, c->d == 8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    c->tcx_map = r == CUDA_SUCCESS;
  }
  return KNB_OK;
}

int need_ready(knb_ctx* c, bool centroids) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (!c->X && !c->X32 && c->n_local > 0) return fail(KNB_E_STATE, "rows not uploaded or attached");
  if (centroids && !c->centroids_set) return fail(KNB_E_STATE, "centroids not initialised");
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(KNB_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return KNB_OK;
}

const void* rows_of(const knb_ctx* c) {
  return c->elem == 4 ? static_cast<const void*>(c->X32) : static_cast<const void*>(c->X);
}

int ensure_partials(knb_ctx* c) {
  if (c->partials) return KNB_OK;
  return dev_alloc(c, &c->partials, (size_t)c->G_alloc * c->L);
}

bool f32_supported(int d, int k, int pruning) {
  return !pruning && d % 4 == 0 && d >= 32 && d <= 256 && k >= 1 && k <= 16384;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || fn == nullptr ||
      q != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

// 2-D f32 map, 32-column (128 B) boxes with the 128-byte swizzle the UMMA
// descriptors expect; columns past `cols` read as zeros.
int encode_f32_map(CUtensorMap* m, const float* p, long long cols, long long rows, int box_rows) {
  auto encode = tensor_map_encoder();
  if (!encode) return fail(KNB_E_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old for the f32 path)");
  cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(p), gdim, gstride, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(KNB_E_CUDA, "cuTensorMapEncodeTiled failed for f32 rows (" + std::to_string((int)r) + ")");
  return KNB_OK;
}

// first f32 rows: switch the context to the tensor-core path and allocate its state
int tc_setup(knb_ctx* c) {
  if (c->tc) return KNB_OK;
  if (!f32_supported(c->d, c->k, c->pruning))
    return fail(KNB_E_ARG, "f32 rows need the dense tensor-core path: pruning off, d % 4 == 0, 32 <= d <= 256, k <= 16384");
  if (c->n_local > (1LL << 30)) return fail(KNB_E_ARG, "f32 path: at most 2^30 rows per GPU");
  if (c->X) return fail(KNB_E_STATE, "context already holds f64 rows");
  const long long nl = c->n_local ? c->n_local : 1;
  c->elem = 4;
  c->kp = (c->k + 255) / 256 * 256;
  c->dp = (c->d + 31) / 32 * 32;
  c->nkc = c->dp / 32;
  c->nnt = c->kp / 256;
  // CTA pairs over 256-row tiles: an even grid, every CTA one 128-row half per pair tile
  const long long ptiles = (nl + 2 * tc_rows_per_tile() - 1) / (2 * tc_rows_per_tile());
  const long long pairs = ptiles < c->sms / 2 ? ptiles : c->sms / 2;
  c->G_tc = (int)(2 * pairs);
  c->tcq_cap = (ptiles + pairs - 1) / pairs * 32;
  int rc;
  if ((rc = dev_alloc(c, &c->c32, (size_t)c->kp * c->dp))) return rc;
  if ((rc = dev_alloc(c, &c->chn32, c->kp))) return rc;
  if ((rc = dev_alloc(c, &c->xn2, nl))) return rc;
  if ((rc = dev_alloc(c, &c->old_assign, nl))) return rc;
  if ((rc = dev_alloc(c, &c->tc_bound, nl))) return rc;
  if ((rc = dev_alloc(c, &c->tc_fullq, nl))) return rc;
  if ((rc = dev_alloc(c, &c->tc_scratch, (size_t)c->G_tc * 2 * tc_rows_per_tile()))) return rc;
  if ((rc = dev_alloc(c, &c->tcq, (size_t)c->G_tc * 4 * 2 * c->tcq_cap))) return rc;
  if ((rc = dev_alloc(c, &c->tcq_count, (size_t)c->G_tc * 4))) return rc;
  if ((rc = dev_alloc(c, &c->tc_counters, 4))) return rc;
  KNB_CUDA(cudaMemsetAsync(c->tc_counters, 0, 4 * sizeof(unsigned long long), c->stream));
  KNB_CUDA(cudaMemsetAsync(c->tcq_count, 0, sizeof(int) * c->G_tc * 4, c->stream));
  KNB_CUDA(cudaMemsetAsync(c->c32, 0, sizeof(float) * (size_t)c->kp * c->dp, c->stream));
  if ((rc = encode_f32_map(&c->tmC32, c->c32, c->dp, c->kp, 128))) return rc;
  // cluster-sorted accumulation
  SegArgs& g = c->seg;
  std::memset(&g, 0, sizeof(g));
  g.n = c->n_local;
  g.d = c->d;
  g.k = c->k;
  g.B = seg_blocks(nl);
  if ((rc = dev_alloc(c, &g.counts, (size_t)c->k * g.B))) return rc;
  if ((rc = dev_alloc(c, &g.lrank, 2 * (size_t)nl))) return rc;
  if ((rc = dev_alloc(c, &g.ctot, c->k))) return rc;
  if ((rc = dev_alloc(c, &g.cstart, c->k + 1))) return rc;
  if ((rc = dev_alloc(c, &g.istart, c->k + 1))) return rc;
  if ((rc = dev_alloc(c, &g.sorted, 2 * (size_t)nl))) return rc;
  if ((rc = dev_alloc(c, &g.records, (size_t)seg_max_items(nl, c->k) * (c->d + 2)))) return rc;
  c->tc = true;
  return KNB_OK;
}

int tc_attach(knb_ctx* c, const float* p) {
  c->X32 = p;
  c->graph_valid = false;
  c->xn_valid = false;
  if (reinterpret_cast<uintptr_t>(p) & 15) return fail(KNB_E_ARG, "f32 rows must be 16-byte aligned");
  if (c->n_local > 0) return encode_f32_map(&c->tmX32, p, c->d, c->n_local, tc_rows_per_tile());
  return KNB_OK;
}

SegArgs seg_args(knb_ctx* c, int mode, const int32_t* labels) {
  SegArgs g = c->seg;
  g.X = rows_of(c);
  g.assign = labels;
  g.old_assign = c->old_assign;
  g.xn2 = c->xn2;
  g.mode = mode;
  g.exch = c->exch;
  g.ctrl = c->ctrl;
  return g;
}

int ensure_xn2(knb_ctx* c) {
  if (c->xn_valid) return KNB_OK;
  if (c->n_local) KNB_CUDA(launch_row_sqnorm_f32(c->X32, c->n_local, c->d, c->xn2, c->stream));
  c->xn_valid = true;
  return KNB_OK;
}

TcArgs tc_args(knb_ctx* c);

// one dense pass of f32 rows: TF32 scores + certificate, exact rerank of the
// uncertified rows, cluster-sorted accumulation (full on the first pass, signed
// deltas of the moved rows afterwards), scalars
int tc_local(knb_ctx* c) {
  int rc = ensure_xn2(c);
  if (rc) return rc;
  KNB_CUDA(cudaMemsetAsync(c->tc_counters, 0, sizeof(unsigned long long), c->stream));
  KNB_CUDA(cudaMemsetAsync(c->tc_counters + 3, 0, sizeof(unsigned long long), c->stream));
  KNB_CUDA(launch_tc_prep(c->means, c->cn2, c->k, c->d, c->kp, c->dp, c->c32, c->chn32, c->stream));
  TcArgs a = tc_args(c);
  if (c->n_local) {
    if (c->t_host == 0) {
      // no distance bounds yet: one scoring pass for each row's maximum, then the
      // collecting pass with the exact window
      a.mode = TC_MAX;
      KNB_CUDA(launch_tc_assign(&c->tmX32, &c->tmC32, a, c->G_tc, c->stream));
      a.mode = TC_COLLECT_SMAX;
    }
    KNB_CUDA(launch_tc_assign(&c->tmX32, &c->tmC32, a, c->G_tc, c->stream));
    KNB_CUDA(launch_tc_rerank(a, c->means, c->G_tc * 4, c->stream));
    KNB_CUDA(launch_tc_rerank_full(a, c->means, c->sms, c->stream));
  }
  SegArgs g = seg_args(c, c->t_host == 0 ? 0 : 1, c->assign);
  KNB_CUDA(launch_segsum(g, 4, c->stream));
  KNB_CUDA(launch_tc_scalars(c->tc_counters, c->n_local, c->k, c->d, c->exch, c->ctrl, c->stream));
  return KNB_OK;
}

TcArgs tc_args(knb_ctx* c) {
  TcArgs a;
  a.X = c->X32;
  a.n = c->n_local;
  a.d = c->d;
  a.k = c->k;
  a.kp = c->kp;
  a.nkc = c->nkc;
  a.nnt = c->nnt;
  a.assign = c->assign;
  a.old_assign = c->old_assign;
  a.xn2 = c->xn2;
  a.chn32 = c->chn32;
  a.queue = c->tcq;
  a.qcount = c->tcq_count;
  a.qcap = c->tcq_cap;
  a.counters = c->tc_counters;
  a.ctrl = c->ctrl;
  a.err_rel = KNB_TF32_ERR;
  a.dbg = nullptr;
  a.mode = TC_COLLECT_BOUND;
  a.bound = c->tc_bound;
  a.drift = c->drift;
  a.scratch = c->tc_scratch;
  a.fullq = c->tc_fullq;
  return a;
}

DenseArgs dense_args(knb_ctx* c) {
  DenseArgs a;
  a.X = c->X;
  a.n = c->n_local;
  a.d = c->d;
  a.k = c->k;
  a.assign = c->assign;
  a.upper = c->upper;
  a.tight = c->tight;
  a.mti_seed = 0;
  a.labels_only = 0;
  a.delta = 0;
  a.mti_filter = 0;
  a.gate = 0;
  a.drift = c->drift;
  a.half_min = c->half_min;
  a.means = c->means;
  a.chn = c->chn;
  a.partials = c->partials;
  a.ctrl = c->ctrl;
  a.use_tma = c->use_tma;
  return a;
}

int launch_pass(knb_ctx* c);

// the split-TF32 tcgen05 MTI pass applies: d = 16, k <= 128, HBM rows with a 128-row map
bool tcx_ready(const knb_ctx* c) {
  return c->tcx_nx > 0 && c->tcx_map && !c->host_registered && !c->sem && c->n_local > 0;
}

int launch_tcx(knb_ctx* c, int gate, float* dbg) {
  KNB_CUDA(launch_mti_tc_prep(c->means, c->d, c->k, c->tcx_bimg, dbg ? nullptr : c->tcx_rq_count, c->stream));
  MtiTcArgs t;
  t.X = c->X;
  t.n = c->n_local;
  t.d = c->d;
  t.k = c->k;
  t.nx = c->tcx_nx;
  t.gtc = c->G_dense < c->sms ? c->G_dense : c->sms;
  t.assign = c->assign;
  t.upper = c->upper;
  t.tight = c->tight;
  t.means = c->means;
  t.drift = c->drift;
  t.half_min = c->half_min;
  t.bimg = c->tcx_bimg;
  t.partials = c->partials;
  t.ctrl = c->ctrl;
  t.gate = gate;
  t.dbg = dbg;
  t.counters = c->tcx_counters;
  t.kmask = 0xFFFFFF80u;
  t.recs = c->tcx_recs;
  t.rq = c->tcx_rq;
  t.rq_count = c->tcx_rq_count;
  t.rq_cap = c->tcx_rq_cap;
  KNB_CUDA(launch_mti_tc(&c->tmX128, t, c->G_dense, c->stream));
  if (!dbg) {
    KNB_CUDA(launch_mti_tc_rerank(t, 2 * c->sms, c->stream));  // (two 8-warp CTAs per SM)
    KNB_CUDA(launch_mti_tc_delta(t, c->G_dense, c->stream));
  }
  return KNB_OK;
}

SemArgs sem_args(knb_ctx* c) {
  SemArgs s = c->semA;
  s.assign = c->assign;
  s.upper = c->upper;
  s.drift = c->drift;
  s.half_min = c->half_min;
  s.X = c->X;
  s.ctrl = c->ctrl;
  return s;
}

// one iteration's local work; semi-external runs add the I/O accounting before the
// pass (it needs the bounds the pass overwrites) and the cache refresh after it
int launch_local(knb_ctx* c) {
  if (!c->sem) return launch_pass(c);
  const SemArgs s = sem_args(c);
  KNB_CUDA(launch_sem_account(s, c->sms, c->stream));
  int rc = launch_pass(c);
  if (rc) return rc;
  KNB_CUDA(launch_sem_rebuild(s, c->sms, c->stream));
  return KNB_OK;
}

// the CTA partials of a pass -> the exchange vector (fixed order).  (Fusing this into
// the finalize, one warp per centroid, was measured slower: c1 0.023 -> 0.034 ms/iter,
// the per-centroid reductions serialise what reduce_kernel does in one round trip.)
int reduce_partials(knb_ctx* c, int G) {
  KNB_CUDA(launch_reduce(c->partials, G, c->L, c->exch, c->ctrl, c->stream));
  return KNB_OK;
}

int launch_pass(knb_ctx* c) {
  if (c->tc) return tc_local(c);
  int rc = ensure_partials(c);
  if (rc) return rc;
  const bool full = !c->pruning || c->t_host == 0;
  if (full) {
    DenseArgs a = dense_args(c);
    a.mti_seed = c->pruning;
    a.delta = (!c->pruning && c->t_host > 0) ? 1 : 0;
    KNB_CUDA(launch_dense(&c->tmap, a, c->DP, c->G_dense, c->stream));
    return reduce_partials(c, c->G_dense);
  }
  MtiArgs m;
  m.X = c->X;
  m.n = c->n_local;
  m.d = c->d;
  m.k = c->k;
  m.assign = c->assign;
  m.upper = c->upper;
  m.tight = c->tight;
  m.means = c->means;
  m.drift = c->drift;
  m.half = c->half;
  m.half_min = c->half_min;
  m.chn = c->chn;
  m.partials = c->partials;
  m.ctrl = c->ctrl;
  m.half_in_smem = c->half_in_smem;
  m.row_gather = c->host_registered ? 1 : 0;
  m.cslot = (c->sem && c->host_registered && c->semA.rows_per_part > 0) ? c->semA.cslot : nullptr;
  m.cache = c->semA.cache;
  m.gate = 0;
  int mode = (c->mti_mma_ok || c->mti_scan == KNB_MTI_TC) ? c->mti_scan : KNB_MTI_EXACT;
  const bool tcx_any = tcx_ready(c);
  // automatic choices take the tcgen05 pass for rows of 16 (config 4: 148.6 -> 45 ms per
  // pass against the DMMA block pass); rows of 8 / 32 run it when forced (mti_scan="tc")
  const bool tcx = tcx_any && (c->d == 16 || mode == KNB_MTI_TC);
  if (mode == KNB_MTI_TC && !tcx_any)
    return fail(KNB_E_ARG, "the tcgen05 MTI pass needs d in {8, 16, 32}, k <= 128 (k <= 32 for d = 32) and 16-byte aligned rows in HBM");
  // the compacted kernel's filter uses 32-bit row / block indices: larger shards take a
  // block MTI pass (64-bit indices, same results)
  if ((mode == KNB_MTI_AUTO || mode == KNB_MTI_DENSE) && !mti_compact_ok(c->n_local))
    mode = tcx ? KNB_MTI_TC : KNB_MTI_BLOCK;
  if (mode == KNB_MTI_EXACT) {
    KNB_CUDA(launch_mti(m, c->DPm, c->G_mti, c->stream));
    return reduce_partials(c, c->G_mti);
  }
  DenseArgs a = dense_args(c);
  a.mti_filter = 1;
  if (mode == KNB_MTI_TC) {
    int rc = launch_tcx(c, 0, nullptr);
    if (rc) return rc;
  } else if (mode == KNB_MTI_BLOCK) {
    KNB_CUDA(launch_dense(&c->tmap, a, c->DP, c->G_dense, c->stream));
  } else if (mode == KNB_MTI_DENSE) {
    KNB_CUDA(launch_mti_mma(m, c->DP, c->G_dense, c->stream));
  } else {
    // auto: both are queued; the device-side choice made by the previous finalize
    // (skip fraction) lets exactly one of them run, the other returns at once.  The
    // block form is the tcgen05 pass where it applies (d = 16: config 4)
    a.gate = 1;
    m.gate = 1;
    if (tcx) {
      int rc = launch_tcx(c, 1, nullptr);
      if (rc) return rc;
    } else {
      KNB_CUDA(launch_dense(&c->tmap, a, c->DP, c->G_dense, c->stream));
    }
    if (mti_compact_ok(c->n_local)) KNB_CUDA(launch_mti_mma(m, c->DP, c->G_dense, c->stream));
  }
  return reduce_partials(c, c->G_dense);
}

int launch_finish(knb_ctx* c) {
  FinalArgs f = final_args(c);
  KNB_CUDA(launch_finalize(f, c->stream));
  if (c->pruning) KNB_CUDA(launch_geometry(f, c->stream));
  c->t_host += 1;
  return KNB_OK;
}

int install_means(knb_ctx* c, const double* src_dev, int from_partition) {
  FinalArgs f = final_args(c);
  KNB_CUDA(launch_set_means(src_dev, c->k, c->d, f, from_partition, c->n_global, c->stream));
  int rc = reset_run(c);
  if (rc) return rc;
  c->centroids_set = true;
  return KNB_OK;
}

// Capture one steady-state iteration into c->graph (the kernels take every decision
// from device state, so the same graph serves every later iteration of the run).
int build_graph(knb_ctx* c) {
  if (c->graph_valid) return KNB_OK;
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  if (!c->cap_stream) KNB_CUDA(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  if (c->tc) {  // the f32 path computes its row norms once, outside the graph
    int rc = ensure_xn2(c);
    if (rc) return rc;
  }
  cudaStream_t user = c->stream;
  const long long t = c->t_host;
  c->stream = c->cap_stream;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal);
  int rc = KNB_OK;
  if (e == cudaSuccess) {
    rc = launch_local(c);
    if (!rc) rc = launch_finish(c);
    e = cudaStreamEndCapture(c->cap_stream, &g);
  }
  c->stream = user;
  c->t_host = t;
  if (rc) {
    if (g) cudaGraphDestroy(g);
    return rc;
  }
  if (e != cudaSuccess) return fail(KNB_E_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&c->graph, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return fail(KNB_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  c->graph_valid = true;
  return KNB_OK;
}

// enqueue one iteration: the captured graph once past the first (full) pass
int enqueue_iteration(knb_ctx* c) {
  if (c->t_host >= 1) {
    int rc = build_graph(c);
    if (rc) return rc;
    KNB_CUDA(cudaGraphLaunch(c->graph, c->stream));
    c->t_host += 1;
    return KNB_OK;
  }
  int rc = launch_local(c);
  if (rc) return rc;
  return launch_finish(c);
}

void to_host_stats(const IterStatsDev& s, knb_iter_stats* o) {
  o->t = s.t;
  o->reassignments = s.reassignments;
  o->wcss = s.wcss;
  o->dist_comps = s.dist_comps;
  o->skips = s.skips;
  o->pruned_stale = s.pruned_stale;
  o->pruned_tight = s.pruned_tight;
  o->converged = s.converged;
  o->stop = s.stop;
  o->count_total = s.count_total;
}

}  // namespace

extern "C" {

int knb_version(void) { return 1; }

const char* knb_last_error(void) { return g_err.c_str(); }

int knb_device_info(int device, int* sms, int64_t* hbm_bytes, int* cc_major, int* cc_minor) {
  cudaDeviceProp p;
  KNB_CUDA(cudaGetDeviceProperties(&p, device));
  if (sms) *sms = p.multiProcessorCount;
  if (hbm_bytes) *hbm_bytes = (int64_t)p.totalGlobalMem;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return KNB_OK;
}

int knb_create(int device, int64_t n_global, int64_t n_local, int64_t row_lo, int32_t d, int32_t k,
               int32_t pruning, int32_t max_iters, double tolerance, void* stream, knb_ctx** out) {
  if (!out) return fail(KNB_E_ARG, "null out");
  *out = nullptr;
  if (n_global < 1 || n_local < 0 || row_lo < 0 || row_lo + n_local > n_global)
    return fail(KNB_E_ARG, "bad shard geometry");
  if (d < 1) return fail(KNB_E_ARG, "d must be >= 1");
  if (k < 1) return fail(KNB_E_ARG, "k must be >= 1");
  if (max_iters < 1) return fail(KNB_E_ARG, "max_iters must be >= 1");
  if (!(tolerance >= 0.0)) return fail(KNB_E_ARG, "tolerance must be >= 0");
  KNB_CUDA(cudaSetDevice(device));
  knb_ctx* c = new knb_ctx();
  std::memset(&c->tmap, 0, sizeof(c->tmap));
  std::memset(&c->tmX32, 0, sizeof(c->tmX32));
  std::memset(&c->tmC32, 0, sizeof(c->tmC32));
  std::memset(&c->seg, 0, sizeof(c->seg));
  std::memset(&c->semA, 0, sizeof(c->semA));
  c->device = device;
  c->n_global = n_global;
  c->n_local = n_local;
  c->row_lo = row_lo;
  c->d = d;
  c->k = k;
  c->pruning = pruning ? 1 : 0;
  c->max_iters = max_iters;
  c->tolerance = tolerance;
  int rc = KNB_OK;
  auto bail = [&](int code) {
    knb_destroy(c);
    return code;
  };
  // (one attribute query: cudaGetDeviceProperties costs milliseconds per call)
  if (cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess)
    return bail(fail(KNB_E_CUDA, "cudaDeviceGetAttribute"));
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(KNB_E_CUDA, "cudaStreamCreate"));
    c->own_stream = true;
  }
  // kernel selection
  c->DP = dense_tile_dp(d);
  if (c->DP && dense_tile_smem(c->DP, k, d) > SMEM_LIMIT) c->DP = 0;
  c->DPm = dense_tile_dp(d);
  c->half_in_smem = 0;
  if (c->DPm) {
    if ((size_t)k * k * 8 <= 64 * 1024 && mti_tile_smem(c->DPm, k, 1) <= SMEM_LIMIT) c->half_in_smem = 1;
    else if (mti_tile_smem(c->DPm, k, 0) > SMEM_LIMIT) c->DPm = 0;
  }
  const long long nl = n_local > 0 ? n_local : 1;
  {
    const long long rows = dense_rows_per_tile(c->DP);
    const long long tiles = (nl + rows - 1) / rows;
    long long g = c->DP ? dense_tile_grid(c->DP, k, d, c->sms) : 4LL * c->sms;
    // small shards: one CTA per SM (a second CTA per SM only adds setup and partials;
    // measured c1, 200k rows: 0.029 -> 0.027 ms / iteration)
    if (c->DP && nl < 4096LL * c->sms) g = c->sms;
    c->G_dense = (int)(tiles < g ? tiles : g);
  }
  {
    const long long rows = c->DPm ? 4LL * KNB_NT : KNB_NT;
    const long long tiles = (nl + rows - 1) / rows;
    long long g = c->DPm ? mti_tile_grid(c->DPm, k, c->half_in_smem, c->sms) : 4LL * c->sms;
    c->G_mti = (int)(tiles < g ? tiles : g);
  }
  c->mti_mma_ok = c->DP != 0 && mti_mma_fits(c->DP, k, d);
  c->tcx_nx = c->pruning ? mti_tc_stages(d, k) : 0;
  {
    const long long tiles = (nl + 31) / 32;
    c->G_mti_mma = (int)(tiles < c->sms ? tiles : c->sms);
  }
  c->L = acc_len(k, d);
  c->G_alloc = c->G_dense > c->G_mti ? c->G_dense : c->G_mti;
  if (c->G_mti_mma > c->G_alloc) c->G_alloc = c->G_mti_mma;
  const size_t kd = (size_t)k * d;
  if ((rc = dev_alloc(c, &c->assign, nl))) return bail(rc);
  if (c->pruning) {
    if ((rc = dev_alloc(c, &c->upper, nl))) return bail(rc);
    if ((rc = dev_alloc(c, &c->tight, nl))) return bail(rc);
    if ((rc = dev_alloc(c, &c->half, (size_t)k * k))) return bail(rc);
    if ((rc = dev_alloc(c, &c->half_min, k))) return bail(rc);
    if (cudaMemsetAsync(c->tight, 0, nl, c->stream) != cudaSuccess) return bail(fail(KNB_E_CUDA, "memset"));
  }
  if (c->tcx_nx > 0) {
    if ((rc = dev_alloc(c, &c->tcx_counters, 1))) return bail(rc);
    double* bimg = nullptr;
    if ((rc = dev_alloc(c, &bimg, mti_tc_bimg_bytes(d, k) / sizeof(double)))) return bail(rc);
    c->tcx_bimg = bimg;
    double* recs = nullptr;
    const size_t rec_bytes = (size_t)((nl + 127) / 128) * TC_REC;
    if ((rc = dev_alloc(c, &recs, (rec_bytes + 7) / 8))) return bail(rc);
    c->tcx_recs = reinterpret_cast<unsigned char*>(recs);
    // the rerank queue: 1/128 of the rows (c4 flags ~0.3% per pass), at least 64K entries
    c->tcx_rq_cap = nl / 128 > 65536 ? nl / 128 : 65536;
    double* rq = nullptr;
    if ((rc = dev_alloc(c, &rq, (size_t)c->tcx_rq_cap * 2))) return bail(rc);
    c->tcx_rq = reinterpret_cast<long long*>(rq);
    if ((rc = dev_alloc(c, &c->tcx_rq_count, 1))) return bail(rc);
  }
  if ((rc = dev_alloc(c, &c->run, c->L))) return bail(rc);
  if ((rc = dev_alloc(c, &c->means, kd))) return bail(rc);
  if ((rc = dev_alloc(c, &c->prev, kd))) return bail(rc);
  if ((rc = dev_alloc(c, &c->stage, kd))) return bail(rc);
  if ((rc = dev_alloc(c, &c->drift, k))) return bail(rc);
  if ((rc = dev_alloc(c, &c->counts, k))) return bail(rc);
  if ((rc = dev_alloc(c, &c->chn, k))) return bail(rc);
  if ((rc = dev_alloc(c, &c->cn2, k))) return bail(rc);
  if ((rc = dev_alloc(c, &c->wterm, k))) return bail(rc);
  if ((rc = dev_alloc(c, &c->exch, c->L))) return bail(rc);
  if ((rc = dev_alloc(c, &c->ctrl, 1))) return bail(rc);
  if ((rc = dev_alloc(c, &c->fin_sync, 1))) return bail(rc);
  if (cudaMemsetAsync(c->fin_sync, 0, sizeof(unsigned int), c->stream) != cudaSuccess)
    return bail(fail(KNB_E_CUDA, "memset"));
  if ((rc = dev_alloc(c, &c->stats, max_iters))) return bail(rc);
  if ((rc = dev_alloc(c, &c->bad, 2))) return bail(rc);
  if (cudaMemsetAsync(c->ctrl, 0, sizeof(Ctrl), c->stream) != cudaSuccess) return bail(fail(KNB_E_CUDA, "memset"));
  if (cudaMemsetAsync(c->stats, 0, sizeof(IterStatsDev) * max_iters, c->stream) != cudaSuccess)
    return bail(fail(KNB_E_CUDA, "memset"));
  if ((rc = reset_run(c))) return bail(rc);
  *out = c;
  return KNB_OK;
}

int knb_destroy(knb_ctx* c) {
  if (!c) return KNB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  void* ptrs[] = {c->X_own, c->assign, c->upper, c->tight, c->means, c->prev, c->stage, c->drift, c->counts,
                  c->chn, c->cn2, c->half, c->half_min, c->wterm, c->run, c->partials, c->ctrl, c->fin_sync, c->stats,
                  c->bad, c->ids_dev, c->d2, c->kpp_bs, c->kpp_scalar, c->kpp_idx, c->X32_own, c->c32,
                  c->chn32, c->xn2, c->old_assign, c->tc_bound, c->tc_scratch, c->tc_fullq, c->tcq, c->tcq_count, c->tc_counters, c->tcx_bimg, c->tcx_recs, c->tcx_counters, c->tcx_rq, c->tcx_rq_count, c->seg.counts,
                  c->seg.lrank, c->seg.ctot, c->seg.cstart, c->seg.istart, c->seg.sorted, c->seg.records,
                  c->semA.fetched, c->semA.cslot, c->semA.crow, c->semA.cache, c->semA.bcount, c->semA.bpre,
                  c->semA.plo, c->semA.io};
  for (void* q : ptrs) dev_free(c, q);
  if (c->own_exch && c->exch) dev_free(c, c->exch);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  if (c->host_registered) cudaHostUnregister(const_cast<void*>(c->host_registered));
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return KNB_OK;
}

int knb_release_memory(int device) {
  KNB_CUDA(cudaSetDevice(device));
  if (cudaMemPool_t pool = lib_pool(device)) {
    KNB_CUDA(cudaDeviceSynchronize());
    KNB_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  return KNB_OK;
}

int knb_f32_supported(int32_t d, int32_t k, int32_t pruning) { return f32_supported(d, k, pruning) ? 1 : 0; }

int knb_mti_compact_ok(int64_t n_local) { return mti_compact_ok(n_local) ? 1 : 0; }

int knb_upload_rows_f32(knb_ctx* c, const float* host, int64_t lo, int64_t rows) {
  if (!c || (!host && rows > 0)) return fail(KNB_E_ARG, "null argument");
  if (lo < 0 || rows < 0 || lo + rows > c->n_local) return fail(KNB_E_ARG, "row range outside the shard");
  KNB_CUDA(cudaSetDevice(c->device));
  int rc;
  if (!c->X32_own) {
    if ((rc = tc_setup(c))) return rc;
    if ((rc = dev_alloc(c, &c->X32_own, (size_t)(c->n_local ? c->n_local : 1) * c->d))) return rc;
    if ((rc = tc_attach(c, c->X32_own))) return rc;
  }
  c->xn_valid = false;
  if (rows) {
    KNB_CUDA(cudaStreamSynchronize(c->stream));
    KNB_CUDA(staged_copy(c->device, c->X32_own + lo * c->d, host, sizeof(float) * rows * c->d, true));
  }
  return KNB_OK;
}

int knb_attach_rows_f32(knb_ctx* c, const float* dev) {
  if (!c || !dev) return fail(KNB_E_ARG, "null argument");
  KNB_CUDA(cudaSetDevice(c->device));
  int rc = tc_setup(c);
  if (rc) return rc;
  return tc_attach(c, dev);
}

int knb_tc_info(knb_ctx* c, int32_t* active, int64_t* flagged, int64_t* full_reranks) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (active) *active = c->tc ? 1 : 0;
  unsigned long long h[4] = {0, 0, 0, 0};
  if (c->tc) {
    KNB_CUDA(cudaSetDevice(c->device));
    KNB_CUDA(cudaMemcpyAsync(h, c->tc_counters, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (flagged) *flagged = (int64_t)h[1];
  if (full_reranks) *full_reranks = (int64_t)h[2];
  return KNB_OK;
}

int knb_mti_tc_info(knb_ctx* c, int32_t* available, int64_t* uncertified) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (available) *available = tcx_ready(c) ? 1 : 0;
  unsigned long long h = 0;
  if (c->tcx_counters) {
    KNB_CUDA(cudaSetDevice(c->device));
    KNB_CUDA(cudaMemcpyAsync(&h, c->tcx_counters, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (uncertified) *uncertified = (int64_t)h;
  return KNB_OK;
}

int knb_mti_tc_prof(int64_t* out16, int32_t* enabled) {
  if (!out16) return fail(KNB_E_ARG, "null output");
  unsigned long long h[16];
  const int rc = mti_tc_prof(h);
  if (rc < 0) return fail(KNB_E_CUDA, "reading the tcgen05 MTI profile counters");
  for (int i = 0; i < 16; ++i) out16[i] = (int64_t)h[i];
  if (enabled) *enabled = rc;
  return KNB_OK;
}

int knb_mti_tc_scores(knb_ctx* c, float* dev_out) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  if (!tcx_ready(c)) return fail(KNB_E_STATE, "the tcgen05 MTI pass does not apply to this context");
  if (!dev_out) return fail(KNB_E_ARG, "null output");
  if ((rc = ensure_partials(c))) return rc;
  if ((rc = launch_tcx(c, 0, dev_out))) return rc;
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_tc_scores(knb_ctx* c, float* dev_out, double* err_rel) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  if (!c->tc) return fail(KNB_E_STATE, "no f32 rows on the tensor-core path");
  if (!dev_out) return fail(KNB_E_ARG, "null output");
  if ((rc = ensure_xn2(c))) return rc;
  KNB_CUDA(launch_tc_prep(c->means, c->cn2, c->k, c->d, c->kp, c->dp, c->c32, c->chn32, c->stream));
  TcArgs a = tc_args(c);
  a.dbg = dev_out;
  a.mode = TC_MAX;
  if (c->n_local) KNB_CUDA(launch_tc_assign(&c->tmX32, &c->tmC32, a, c->G_tc, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (err_rel) *err_rel = KNB_TF32_ERR;
  return KNB_OK;
}

int knb_upload_rows(knb_ctx* c, const double* host, int64_t lo, int64_t rows) {
  if (!c || (!host && rows > 0)) return fail(KNB_E_ARG, "null argument");
  if (c->tc) return fail(KNB_E_STATE, "context holds f32 rows");
  if (lo < 0 || rows < 0 || lo + rows > c->n_local) return fail(KNB_E_ARG, "row range outside the shard");
  KNB_CUDA(cudaSetDevice(c->device));
  if (!c->X_own) {
    int rc = dev_alloc(c, &c->X_own, (size_t)(c->n_local ? c->n_local : 1) * c->d);
    if (rc) return rc;
    c->X = c->X_own;
    rc = build_tmap(c);
    if (rc) return rc;
  }
  if (rows) {  // (ordered after the stream's earlier work; synchronous)
    KNB_CUDA(cudaStreamSynchronize(c->stream));
    KNB_CUDA(staged_copy(c->device, c->X_own + lo * c->d, host, sizeof(double) * rows * c->d, true));
  }
  return KNB_OK;
}

int knb_attach_host_rows(knb_ctx* c, const double* host) {
  if (!c || (!host && c->n_local > 0)) return fail(KNB_E_ARG, "null argument");
  if (c->tc) return fail(KNB_E_STATE, "context holds f32 rows");
  KNB_CUDA(cudaSetDevice(c->device));
  if (c->host_registered) {
    cudaHostUnregister(const_cast<void*>(c->host_registered));
    c->host_registered = nullptr;
  }
  if (c->n_local == 0) return KNB_OK;
  const size_t bytes = sizeof(double) * (size_t)c->n_local * c->d;
  void* p = const_cast<double*>(host);
  cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly);
  if (e != cudaSuccess) {
    cudaGetLastError();
    e = cudaHostRegister(p, bytes, cudaHostRegisterMapped);  // read-only registration is optional
  }
  if (e != cudaSuccess) {
    cudaGetLastError();  // not sticky: keep it out of the next launch check
    return fail(KNB_E_CUDA, std::string("cudaHostRegister: ") + cudaGetErrorString(e));
  }
  c->host_registered = host;
  void* dptr = nullptr;
  KNB_CUDA(cudaHostGetDevicePointer(&dptr, p, 0));
  c->X = static_cast<const double*>(dptr);
  c->graph_valid = false;
  return build_tmap(c);
}

int knb_attach_rows(knb_ctx* c, const double* dev) {
  if (!c || !dev) return fail(KNB_E_ARG, "null argument");
  if (c->tc) return fail(KNB_E_STATE, "context holds f32 rows");
  KNB_CUDA(cudaSetDevice(c->device));
  c->X = dev;
  c->graph_valid = false;
  return build_tmap(c);
}

int knb_check_finite(knb_ctx* c, int64_t* first_bad) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  KNB_CUDA(cudaMemsetAsync(c->bad, 0xff, sizeof(long long), c->stream));
  if (c->n_local) KNB_CUDA(launch_check_finite(rows_of(c), c->elem, c->n_local, c->d, c->bad, c->stream));
  long long h;
  KNB_CUDA(cudaMemcpyAsync(&h, c->bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (first_bad) *first_bad = h;  // -1 (all ones) when every value is finite
  return KNB_OK;
}

int knb_exchange_len(knb_ctx* c, int64_t* len) {
  if (!c || !len) return fail(KNB_E_ARG, "null argument");
  *len = c->L;
  return KNB_OK;
}

int knb_set_exchange(knb_ctx* c, double* dev, int64_t len) {
  if (!c || !dev) return fail(KNB_E_ARG, "null argument");
  if (len < c->L) return fail(KNB_E_ARG, "exchange buffer too small");
  if (c->own_exch && c->exch) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    dev_free(c, c->exch);
    c->bytes -= (long long)(c->L * sizeof(double));
  }
  c->exch = dev;
  c->graph_valid = false;
  c->own_exch = false;
  return KNB_OK;
}

int knb_exchange_ptr(knb_ctx* c, double** dev) {
  if (!c || !dev) return fail(KNB_E_ARG, "null argument");
  *dev = c->exch;
  return KNB_OK;
}

int knb_set_centroids(knb_ctx* c, const double* host) {
  if (!c || !host) return fail(KNB_E_ARG, "null argument");
  KNB_CUDA(cudaSetDevice(c->device));
  KNB_CUDA(cudaMemcpyAsync(c->stage, host, sizeof(double) * c->k * c->d, cudaMemcpyHostToDevice, c->stream));
  int rc = install_means(c, c->stage, 0);
  if (rc) return rc;
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_init_gather(knb_ctx* c, const int64_t* ids, int32_t count) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if (count < 1 || count > c->k || !ids) return fail(KNB_E_ARG, "gather count must be in [1, k]");
  if (count > c->ids_cap) {
    dev_free(c, c->ids_dev);
    c->ids_dev = nullptr;
    if ((rc = dev_alloc(c, &c->ids_dev, c->k))) return rc;
    c->ids_cap = c->k;
  }
  KNB_CUDA(cudaMemcpyAsync(c->ids_dev, ids, sizeof(long long) * count, cudaMemcpyHostToDevice, c->stream));
  KNB_CUDA(cudaMemsetAsync(c->exch, 0, sizeof(double) * count * c->d, c->stream));
  if (c->n_local)
    KNB_CUDA(launch_gather_rows(rows_of(c), c->elem, c->n_local, c->row_lo, c->d, c->ids_dev, count, c->exch,
                                c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));  // ids is a caller buffer
  return KNB_OK;
}

int knb_init_from_exchange(knb_ctx* c, int32_t first, int32_t count) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (first < 0 || count < 1 || first + count > c->k) return fail(KNB_E_ARG, "rows outside [0, k)");
  KNB_CUDA(cudaSetDevice(c->device));
  KNB_CUDA(cudaMemcpyAsync(c->stage + (size_t)first * c->d, c->exch, sizeof(double) * count * c->d,
                           cudaMemcpyDeviceToDevice, c->stream));
  if (first + count == c->k) {
    int rc = install_means(c, c->stage, 0);
    if (rc) return rc;
  }
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_init_partition_local(knb_ctx* c, const int32_t* labels) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if (!labels && c->n_local) return fail(KNB_E_ARG, "null labels");
  rc = reset_run(c);  // also clears a stop flag left by an earlier run
  if (rc) return rc;
  if (c->n_local)
    KNB_CUDA(cudaMemcpyAsync(c->assign, labels, sizeof(int32_t) * c->n_local, cudaMemcpyHostToDevice, c->stream));
  if (c->tc) {
    if ((rc = ensure_xn2(c))) return rc;
    KNB_CUDA(launch_segsum(seg_args(c, 0, c->assign), 4, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));  // labels is a caller buffer
    return KNB_OK;
  }
  if ((rc = ensure_partials(c))) return rc;
  DenseArgs a = dense_args(c);
  a.labels_only = 1;
  KNB_CUDA(launch_dense(&c->tmap, a, c->DP, c->G_dense, c->stream));
  KNB_CUDA(launch_reduce(c->partials, c->G_dense, c->L, c->exch, c->ctrl, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));  // labels is a caller buffer
  return KNB_OK;
}

int knb_init_partition_finish(knb_ctx* c) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  int rc = install_means(c, c->exch, 1);
  if (rc) return rc;
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

static int kpp_buffers(knb_ctx* c) {
  if (c->d2) return KNB_OK;
  int rc;
  c->kpp_nblk = (int)((c->n_local + KPP_BLOCK - 1) / KPP_BLOCK);
  if (c->kpp_nblk < 1) c->kpp_nblk = 1;
  if ((rc = dev_alloc(c, &c->d2, c->n_local ? c->n_local : 1))) return rc;
  if ((rc = dev_alloc(c, &c->kpp_bs, c->kpp_nblk))) return rc;
  if ((rc = dev_alloc(c, &c->kpp_scalar, 1))) return rc;
  if ((rc = dev_alloc(c, &c->kpp_idx, 1))) return rc;
  return KNB_OK;
}

int knb_kpp_update(knb_ctx* c, int32_t first, double* local_total) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if ((rc = kpp_buffers(c))) return rc;
  double h = 0.0;
  if (c->n_local) {
    KNB_CUDA(launch_kpp_update(rows_of(c), c->elem, c->n_local, c->d, c->exch, c->d2, first, c->kpp_bs,
                               c->kpp_nblk, c->stream));
    KNB_CUDA(launch_sum_blocks(c->kpp_bs, c->kpp_nblk, c->kpp_scalar, c->stream));
    KNB_CUDA(cudaMemcpyAsync(&h, c->kpp_scalar, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (local_total) *local_total = h;
  return KNB_OK;
}

int knb_kpp_psum(knb_ctx* c, double total, double* local_psum) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if ((rc = kpp_buffers(c))) return rc;
  double h = 0.0;
  if (c->n_local) {
    KNB_CUDA(launch_kpp_psums(c->d2, c->n_local, total, c->kpp_bs, c->kpp_nblk, c->stream));
    KNB_CUDA(launch_sum_blocks(c->kpp_bs, c->kpp_nblk, c->kpp_scalar, c->stream));
    KNB_CUDA(cudaMemcpyAsync(&h, c->kpp_scalar, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
  }
  if (local_psum) *local_psum = h;
  return KNB_OK;
}

int knb_kpp_search(knb_ctx* c, double total, double threshold, int64_t* local_idx) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if (!c->d2 || c->n_local < 1) return fail(KNB_E_STATE, "kmeans++ search without psum / rows");
  KNB_CUDA(launch_kpp_search(c->d2, c->n_local, total, c->kpp_bs, c->kpp_nblk, threshold, c->kpp_idx, c->stream));
  long long h;
  KNB_CUDA(cudaMemcpyAsync(&h, c->kpp_idx, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (local_idx) *local_idx = h;
  return KNB_OK;
}

// The whole kmeans++ loop on one GPU (centroids.py:174-189): the host supplies the
// first pick and the k - 1 uniform draws of its RNG stream; every D^2 update, total,
// probability block sum and search runs on the device back to back, with one
// synchronisation at the end.  A step whose D^2 total is 0 (the reference then
// draws an integer instead) is reported as degenerate and nothing is installed.
int knb_kpp_run(knb_ctx* c, int64_t first_pick, const double* u_host, int32_t k, int64_t* picks_out,
                int32_t* degenerate) {
  int rc = need_ready(c, false);
  if (rc) return rc;
  if (k != c->k || !u_host || !picks_out) return fail(KNB_E_ARG, "kpp_run: k must be the context's k");
  if (c->n_local != c->n_global) return fail(KNB_E_STATE, "kpp_run is single-GPU; sharded runs use kpp_update/psum/search");
  if (first_pick < 0 || first_pick >= c->n_local) return fail(KNB_E_ARG, "first pick outside [0, n)");
  if ((rc = kpp_buffers(c))) return rc;
  long long* picks = nullptr;
  double* u = nullptr;
  int* degen = nullptr;
  double* scal = nullptr;
  if ((rc = dev_alloc(c, &picks, (size_t)k))) return rc;
  auto cleanup = [&]() {
    dev_free(c, picks);
    dev_free(c, u);
    dev_free(c, degen);
    dev_free(c, scal);
    c->bytes -= (long long)(k * 8 + (k > 1 ? (k - 1) * 8 : 8) + 4 + 16);
  };
  if ((rc = dev_alloc(c, &u, (size_t)(k > 1 ? k - 1 : 1))) || (rc = dev_alloc(c, &degen, 1)) ||
      (rc = dev_alloc(c, &scal, 2))) {
    cleanup();
    return rc;
  }
  long long p0 = first_pick;
  cudaError_t e = cudaMemcpyAsync(picks, &p0, sizeof(p0), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess && k > 1)
    e = cudaMemcpyAsync(u, u_host, sizeof(double) * (k - 1), cudaMemcpyHostToDevice, c->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(degen, 0, sizeof(int), c->stream);
  const void* X = rows_of(c);
  const int d = c->d;
  if (e == cudaSuccess) e = launch_gather_row_dev(X, c->elem, d, picks, c->stage, c->stream);
  for (int i = 1; i < k && e == cudaSuccess; ++i) {
    // D^2 against centroid i - 1, its fixed-order total, p-block sums, their end, search
    e = launch_kpp_update(X, c->elem, c->n_local, d, c->stage + (size_t)(i - 1) * d, c->d2, i == 1, c->kpp_bs,
                          c->kpp_nblk, c->stream);
    if (e == cudaSuccess) e = launch_sum_blocks(c->kpp_bs, c->kpp_nblk, scal, c->stream);
    if (e == cudaSuccess) e = launch_kpp_psums_dev(c->d2, c->n_local, scal, c->kpp_bs, c->kpp_nblk, c->stream);
    if (e == cudaSuccess) e = launch_sum_blocks(c->kpp_bs, c->kpp_nblk, scal + 1, c->stream);
    if (e == cudaSuccess)
      e = launch_kpp_search_dev(c->d2, c->n_local, scal, c->kpp_bs, c->kpp_nblk, scal + 1, u + (i - 1), picks + i,
                                degen, c->stream);
    if (e == cudaSuccess) e = launch_gather_row_dev(X, c->elem, d, picks + i, c->stage + (size_t)i * d, c->stream);
  }
  std::vector<long long> hp((size_t)k);
  int hd = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(hp.data(), picks, sizeof(long long) * k, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&hd, degen, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cleanup();
  if (e != cudaSuccess) return fail(KNB_E_CUDA, std::string("kpp_run: ") + cudaGetErrorString(e));
  for (int i = 0; i < k; ++i) picks_out[i] = hp[(size_t)i];
  if (degenerate) *degenerate = hd;
  if (hd) return KNB_OK;
  rc = install_means(c, c->stage, 0);
  if (rc) return rc;
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_kpp_release(knb_ctx* c) {
  if (!c) return fail(KNB_E_ARG, "null context");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->d2) {
    dev_free(c, c->d2);
    c->bytes -= (long long)(sizeof(double) * (c->n_local ? c->n_local : 1));
  }
  c->d2 = nullptr;
  return KNB_OK;
}

int knb_iter_local(knb_ctx* c) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  return launch_local(c);
}

int knb_iter_finish(knb_ctx* c) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  return launch_finish(c);
}

int knb_iterate(knb_ctx* c, knb_iter_stats* out) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  const long long t = c->t_host;
  if ((rc = launch_local(c))) return rc;
  if ((rc = launch_finish(c))) return rc;
  IterStatsDev s;
  Ctrl h;
  KNB_CUDA(cudaMemcpyAsync(&h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  if (t < c->max_iters)
    KNB_CUDA(cudaMemcpyAsync(&s, c->stats + t, sizeof(s), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (h.count_error)
    return fail(KNB_E_COUNT, "iteration " + std::to_string(h.t - 1) + ": accumulator counts sum to " +
                                 std::to_string(h.count_seen) + ", expected " + std::to_string(c->n_global));
  if (out && t < c->max_iters) to_host_stats(s, out);
  return KNB_OK;
}

int knb_run(knb_ctx* c, int32_t batch, int32_t* done) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  if (batch < 1) batch = 1;
  Ctrl h;
  for (;;) {
    for (int b = 0; b < batch && c->t_host < c->max_iters; ++b)
      if ((rc = enqueue_iteration(c))) return rc;
    KNB_CUDA(cudaMemcpyAsync(&h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
    if (h.count_error)
      return fail(KNB_E_COUNT, "accumulator counts sum to " + std::to_string(h.count_seen) + ", expected " +
                                   std::to_string(c->n_global));
    if ((h.stop && !h.ignore_stop) || c->t_host >= c->max_iters) break;
  }
  if (done) *done = (int32_t)h.t;
  return KNB_OK;
}

int knb_enqueue(knb_ctx* c, int32_t count) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  for (int b = 0; b < count && c->t_host < c->max_iters; ++b)
    if ((rc = enqueue_iteration(c))) return rc;
  return KNB_OK;
}

int knb_sem_configure(knb_ctx* c, int32_t T, int64_t task_size, int64_t page_size, int32_t cache_enabled,
                      int64_t cache_capacity, int32_t refresh_start) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (c->sem) return fail(KNB_E_STATE, "semi-external accounting already configured");
  if (c->n_local != c->n_global) return fail(KNB_E_ARG, "semi-external runs use one GPU (the whole matrix)");
  if (c->elem != 8) return fail(KNB_E_ARG, "semi-external runs read f64 rows");
  if (T < 1) return fail(KNB_E_ARG, "T must be >= 1");
  if (task_size < 1) return fail(KNB_E_ARG, "task_size must be >= 1");
  if (page_size < 1) return fail(KNB_E_ARG, "page_size must be >= 1");
  if (cache_capacity < 0) return fail(KNB_E_ARG, "capacity must be >= 0");
  if (refresh_start < 1) return fail(KNB_E_ARG, "refresh start must be >= 1");
  KNB_CUDA(cudaSetDevice(c->device));
  SemArgs& s = c->semA;
  s.n = c->n_local;
  s.d = c->d;
  s.T = T;
  s.pruning = c->pruning;
  s.cache_enabled = cache_enabled ? 1 : 0;
  s.refresh_start = refresh_start;
  s.max_iters = c->max_iters;
  s.task_size = task_size;
  s.page_size = page_size;
  s.row_bytes = 8LL * c->d;
  s.pbase = c->n_local / T;
  s.prem = c->n_local % T;
  s.rows_per_part = cache_enabled ? (cache_capacity / T) / s.row_bytes : 0;  // RowCache.__init__
  const long long n = c->n_local;
  int rc;
  c->sem_nb = sem_rebuild_blocks(n);
  if ((rc = dev_alloc(c, &s.fetched, n))) return rc;
  if ((rc = dev_alloc(c, &s.cslot, n))) return rc;
  if ((rc = dev_alloc(c, &s.io, 4 * (size_t)c->max_iters))) return rc;
  if (s.rows_per_part > 0) {
    const size_t slots = (size_t)T * s.rows_per_part;
    if ((rc = dev_alloc(c, &s.crow, slots))) return rc;
    if ((rc = dev_alloc(c, &s.cache, slots * c->d))) return rc;
    if ((rc = dev_alloc(c, &s.bcount, c->sem_nb))) return rc;
    if ((rc = dev_alloc(c, &s.bpre, c->sem_nb))) return rc;
    if ((rc = dev_alloc(c, &s.plo, T))) return rc;
    KNB_CUDA(cudaMemsetAsync(s.crow, 0xff, sizeof(long long) * slots, c->stream));
  }
  KNB_CUDA(cudaMemsetAsync(s.cslot, 0xff, sizeof(int32_t) * n, c->stream));
  KNB_CUDA(cudaMemsetAsync(s.io, 0, sizeof(long long) * 4 * c->max_iters, c->stream));
  c->sem = true;
  c->graph_valid = false;
  return KNB_OK;
}

int knb_sem_io(knb_ctx* c, int64_t* out, int32_t count) {
  if (!c || !out) return fail(KNB_E_ARG, "null argument");
  if (!c->sem) return fail(KNB_E_STATE, "no semi-external accounting configured");
  if (count < 0 || count > c->max_iters) return fail(KNB_E_ARG, "count outside [0, max_iters]");
  std::vector<long long> h(4 * (size_t)(count ? count : 1));
  KNB_CUDA(cudaMemcpyAsync(h.data(), c->semA.io, sizeof(long long) * 4 * count, cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  const SemArgs& s = c->semA;
  for (int i = 0; i < count; ++i) {
    out[5 * i + 0] = h[4 * i + 0] * s.row_bytes;   // bytes_requested
    out[5 * i + 1] = h[4 * i + 1] * s.page_size;   // bytes_read
    out[5 * i + 2] = h[4 * i + 2];                 // cache_hits
    out[5 * i + 3] = h[4 * i + 3];                 // cache_misses
    out[5 * i + 4] = h[4 * i + 0];                 // rows fetched
  }
  return KNB_OK;
}

int knb_sem_cache(knb_ctx* c, int64_t* ids, double* rows, int64_t cap, int64_t* count) {
  if (!c || !count) return fail(KNB_E_ARG, "null argument");
  if (!c->sem) return fail(KNB_E_STATE, "no semi-external accounting configured");
  const SemArgs& s = c->semA;
  const long long slots = (long long)s.T * s.rows_per_part;
  *count = 0;
  if (slots == 0) return KNB_OK;
  std::vector<long long> crow(slots);
  KNB_CUDA(cudaMemcpyAsync(crow.data(), s.crow, sizeof(long long) * slots, cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  long long m = 0;
  for (long long j = 0; j < slots; ++j) {
    if (crow[j] < 0) continue;
    if (m < cap) {
      if (ids) ids[m] = crow[j];
      if (rows)
        KNB_CUDA(cudaMemcpyAsync(rows + m * s.d, s.cache + j * s.d, sizeof(double) * s.d, cudaMemcpyDeviceToHost,
                                 c->stream));
    }
    ++m;
  }
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  *count = m;
  return KNB_OK;
}

int knb_validate(knb_ctx* c, int64_t* bad_assign, int64_t* bad_bound) {
  int rc = need_ready(c, true);
  if (rc) return rc;
  if (!c->pruning) return fail(KNB_E_STATE, "validate needs a pruning run");
  KNB_CUDA(cudaMemsetAsync(c->bad, 0xff, 2 * sizeof(long long), c->stream));
  if (c->n_local)
    KNB_CUDA(launch_validate(c->X, c->n_local, c->d, c->k, c->assign, c->upper, c->means, c->bad, c->stream));
  long long h[2];
  KNB_CUDA(cudaMemcpyAsync(h, c->bad, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (bad_assign) *bad_assign = h[0];
  if (bad_bound) *bad_bound = h[1];
  return KNB_OK;
}

int knb_get_stats(knb_ctx* c, knb_iter_stats* out, int32_t max_count, int32_t* count) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  Ctrl h;
  KNB_CUDA(cudaMemcpyAsync(&h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  long long nt = h.t < c->max_iters ? h.t : c->max_iters;
  if (nt > max_count) nt = max_count;
  std::vector<IterStatsDev> tmp((size_t)(nt > 0 ? nt : 1));
  if (nt > 0) {
    KNB_CUDA(cudaMemcpyAsync(tmp.data(), c->stats, sizeof(IterStatsDev) * nt, cudaMemcpyDeviceToHost, c->stream));
    KNB_CUDA(cudaStreamSynchronize(c->stream));
  }
  for (long long i = 0; i < nt; ++i) to_host_stats(tmp[i], out + i);
  if (count) *count = (int32_t)nt;
  return KNB_OK;
}

int knb_get_state(knb_ctx* c, int32_t* stop, int32_t* converged, int64_t* t, int32_t* count_error) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  Ctrl h;
  KNB_CUDA(cudaMemcpyAsync(&h, c->ctrl, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (stop) *stop = h.stop;
  if (converged) *converged = h.converged;
  if (t) *t = h.t;
  if (count_error) *count_error = h.count_error;
  return KNB_OK;
}

int knb_get_centroids(knb_ctx* c, double* means, double* prev, int64_t* counts, double* drift) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  const size_t kd = (size_t)c->k * c->d;
  std::vector<double> cnt(c->k);
  if (means) KNB_CUDA(cudaMemcpyAsync(means, c->means, kd * 8, cudaMemcpyDeviceToHost, c->stream));
  if (prev) KNB_CUDA(cudaMemcpyAsync(prev, c->prev, kd * 8, cudaMemcpyDeviceToHost, c->stream));
  if (drift) KNB_CUDA(cudaMemcpyAsync(drift, c->drift, (size_t)c->k * 8, cudaMemcpyDeviceToHost, c->stream));
  if (counts) KNB_CUDA(cudaMemcpyAsync(cnt.data(), c->counts, (size_t)c->k * 8, cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (counts)
    for (int j = 0; j < c->k; ++j) counts[j] = (int64_t)cnt[j];
  return KNB_OK;
}

int knb_get_assignments(knb_ctx* c, int32_t* out, int64_t lo, int64_t count) {
  if (!c || (!out && count > 0)) return fail(KNB_E_ARG, "null argument");
  if (lo < 0 || count < 0 || lo + count > c->n_local) return fail(KNB_E_ARG, "range outside the shard");
  KNB_CUDA(cudaSetDevice(c->device));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  if (count) KNB_CUDA(staged_copy(c->device, out, c->assign + lo, sizeof(int32_t) * count, false));
  return KNB_OK;
}

int knb_staging_reserve(int device) {
  KNB_CUDA(staging_reserve(device));
  return KNB_OK;
}

int knb_get_bounds(knb_ctx* c, double* upper, uint8_t* tight) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (!c->pruning) return fail(KNB_E_STATE, "bounds exist only for pruning runs");
  KNB_CUDA(cudaSetDevice(c->device));
  if (upper && c->n_local)
    KNB_CUDA(cudaMemcpyAsync(upper, c->upper, sizeof(double) * c->n_local, cudaMemcpyDeviceToHost, c->stream));
  if (tight && c->n_local)
    KNB_CUDA(cudaMemcpyAsync(tight, c->tight, c->n_local, cudaMemcpyDeviceToHost, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_sync(knb_ctx* c) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_set_stream(knb_ctx* c, void* stream) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  if (c->own_stream && c->stream && c->stream != s) {
    KNB_CUDA(cudaStreamSynchronize(c->stream));
    cudaStreamDestroy(c->stream);
    c->own_stream = false;
  }
  c->stream = s;
  c->graph_valid = false;
  return KNB_OK;
}

int knb_set_ignore_stop(knb_ctx* c, int32_t on) {
  if (!c) return fail(KNB_E_ARG, "null context");
  KNB_CUDA(cudaSetDevice(c->device));
  int v = on ? 1 : 0;
  KNB_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(c->ctrl) + offsetof(Ctrl, ignore_stop), &v, sizeof(int),
                           cudaMemcpyHostToDevice, c->stream));
  KNB_CUDA(cudaStreamSynchronize(c->stream));
  return KNB_OK;
}

int knb_set_option(knb_ctx* c, int32_t option, int64_t value) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (option == KNB_OPT_MTI_SCAN) {
    if (value < KNB_MTI_AUTO || value > KNB_MTI_TC) return fail(KNB_E_ARG, "bad MTI scan mode");
    if (value == KNB_MTI_TC && c->tcx_nx == 0)
      return fail(KNB_E_ARG, "the tcgen05 MTI pass needs a pruned run with d in {8, 16, 32} and k <= 128 (k <= 32 for d = 32)");
    if ((value == KNB_MTI_DENSE || value == KNB_MTI_BLOCK) && !c->mti_mma_ok)
      return fail(KNB_E_ARG, "dense MTI scan needs d <= 64 and centroids that fit shared memory");
    c->mti_scan = (int)value;
    c->graph_valid = false;
    return KNB_OK;
  }
  return fail(KNB_E_ARG, "unknown option " + std::to_string(option));
}

int knb_state_bytes(knb_ctx* c, int64_t* bytes) {
  if (!c || !bytes) return fail(KNB_E_ARG, "null argument");
  *bytes = c->bytes;
  return KNB_OK;
}

int knb_describe(knb_ctx* c, int32_t* dp, int32_t* tma, int32_t* gd, int32_t* gm) {
  if (!c) return fail(KNB_E_ARG, "null context");
  if (dp) *dp = c->tc ? -c->dp : c->DP;  // negative: f32 rows on the tcgen05 path
  if (tma) *tma = c->use_tma;
  if (gd) *gd = c->G_dense;
  if (gm) *gm = (c->mti_scan != KNB_MTI_EXACT && c->mti_mma_ok) ? -c->G_dense : c->G_mti;
  return KNB_OK;
}

}  // extern "C"
