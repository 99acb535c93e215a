// Internal launcher interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "state.cuh"

#ifndef KNB_PDL_LAUNCH
#define KNB_PDL_LAUNCH 1
#endif

namespace knb {

// launch with programmatic stream serialization (see pdl_enter in common.cuh)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = KNB_PDL_LAUNCH;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

struct DenseArgs {
  const double* X;       // n x d row-major (shard-local rows)
  long long n;
  int d, k;
  int32_t* assign;
  double* upper;         // MTI seeding (pruning runs): nearest distance
  uint8_t* tight;
  int mti_seed;          // 1 on the full pass of a pruned run
  int labels_only;       // accumulate by the labels already in assign (random-partition init)
  int delta;             // dense passes after the first: accumulate signed deltas of moved rows only
  int mti_filter;        // block-dense MTI pass (clause-1 filter per row, see assign_mma.cu)
  int gate;              // run only when ctrl->mti_choice == 1
  const double* drift;   // MTI: per-centroid drift (bound inflation)
  const double* half_min;
  const double* means;   // k x d
  const double* chn;     // k: -0.5 * ||c_j||^2
  double* partials;      // G x acc_len(k, d)
  const Ctrl* ctrl;
  int use_tma;
};

struct MtiArgs {
  const double* X;
  long long n;
  int d, k;
  int32_t* assign;
  double* upper;
  uint8_t* tight;
  const double* means;
  const double* drift;
  const double* half;      // k x k
  const double* half_min;  // k
  const double* chn;       // -0.5 ||c||^2 (tensor-core scan)
  int gate;                // run only when ctrl->mti_choice == 0
  double* partials;
  const Ctrl* ctrl;
  int half_in_smem;
  int row_gather;          // rows in host memory: the warp fetches one row per request
  const int32_t* cslot;    // semi-external runs: HBM cache slot per row (-1: read X), or null
  const double* cache;     // [slots][d]
};

// semi-external I/O accounting + HBM row cache (sem.cu)
struct SemArgs {
  long long n;
  int d, T, pruning, cache_enabled, refresh_start;
  long long max_iters;
  long long task_size, page_size, row_bytes;
  long long pbase, prem;       // partition_rows: n / T, n % T
  long long rows_per_part;     // (capacity / T) / row_bytes
  const int32_t* assign;
  const double* upper;
  const double* drift;
  const double* half_min;
  const double* X;             // rows (host-mapped or HBM)
  uint8_t* fetched;            // [n] rows fetched by the current iteration
  int32_t* cslot;              // [n] cache slot or -1
  long long* crow;             // [slots] row id or -1
  double* cache;               // [slots][d]
  long long* bcount;           // [rebuild blocks]
  long long* bpre;             // [rebuild blocks]
  long long* plo;              // [T]
  long long* io;               // [max_iters][4]: rows requested, pages read, hits, misses
  const Ctrl* ctrl;
};
int sem_rebuild_blocks(long long n);
cudaError_t launch_sem_account(const SemArgs& s, int sms, cudaStream_t st);
cudaError_t launch_sem_rebuild(const SemArgs& s, int sms, cudaStream_t st);

struct FinalArgs {
  int k, d;
  long long n;           // global rows
  int pruning;
  double* exch;          // reduced (and all-reduced) accumulator vector
  double* run;           // pruned runs: running sums/counts/sq (acc layout, no scalars used)
  double* means;
  double* prev;
  double* drift;
  double* counts;        // k, as f64
  double* chn;           // -0.5 ||c||^2
  double* cn2;           // ||c||^2 (for cmax2)
  double* half;
  double* half_min;
  double* wterm;         // k: per-centroid WCSS terms (pruned runs)
  int wcss_mode;         // 0: K1's scalar, 1: pruned formula, 2: dense from running sums
  unsigned int* sync;    // finalize's arrival counter (reset by its last CTA)
  Ctrl* ctrl;
  IterStatsDev* stats;   // [max_iters]
};

// f32 rows on the tcgen05 tensor cores (assign_tc.cu)
struct TcHalf {          // one row's window result from the second epilogue half
  float best, dropped;
  float v[8];            // its TOPK largest window scores, descending
  int j[8];
};
struct TcArgs {
  const float* X;        // n x d row-major f32 (shard-local rows)
  long long n;
  int d, k;
  int kp, nkc, nnt;      // centroids padded to 256s; 32-column K chunks; 256-column N tiles
  int32_t* assign;
  int32_t* old_assign;   // assignment before this pass (delta accumulation)
  const double* xn2;     // ||x||^2 per row
  const float* chn32;    // -||c||^2 / 2 per padded centroid (-inf padding)
  int4* queue;           // rerank entries (2 x int4: row + up to 7 candidates), qcap per epilogue warp
  int* qcount;           // entries per epilogue warp
  long long qcap;
  unsigned long long* counters;  // [0] reassigned this pass, [1] flagged rows, [2] full reranks (cumulative),
                                 // [3] rows in fullq this pass
  int* fullq;            // rows whose candidate window overflowed (re-scored against all k)
  const Ctrl* ctrl;
  double err_rel;        // certified relative error of a TF32 dot product
  float* dbg;            // non-null: dump the n x kp f32 scores instead of assigning
  int mode;              // TC_MAX / TC_COLLECT_SMAX / TC_COLLECT_BOUND
  float* bound;          // per row: max score (TC_MAX out) or distance upper bound (in/out)
  const double* drift;   // per centroid: distance moved by the last finalize
  TcHalf* scratch;       // [grid][2][128] hand-over between the epilogue halves
};
enum TcMode { TC_MAX = 0, TC_COLLECT_SMAX = 1, TC_COLLECT_BOUND = 2 };
size_t tc_smem_bytes(int nkc);
int tc_rows_per_tile();
cudaError_t launch_tc_assign(const CUtensorMap* tmX, const CUtensorMap* tmC, const TcArgs& a, int grid,
                             cudaStream_t s);
cudaError_t launch_tc_rerank(const TcArgs& a, const double* means, int regions, cudaStream_t s);
cudaError_t launch_tc_rerank_full(const TcArgs& a, const double* means, int grid, cudaStream_t s);
cudaError_t launch_tc_prep(const double* means, const double* cn2, int k, int d, int kp, int dp, float* c32,
                           float* chn32, cudaStream_t s);
cudaError_t launch_row_sqnorm_f32(const float* X, long long n, int d, double* out, cudaStream_t s);
cudaError_t launch_tc_scalars(const unsigned long long* counters, long long n_local, int k, int d,
                              double* exch, const Ctrl* ctrl, cudaStream_t s);

// f64 rows (d = 16) on the tcgen05 tensor cores: the MTI block pass with split-TF32
// scores and a certified argmin (mti_tc.cu)
struct MtiTcArgs {
  const double* X;       // n x 16 rows (the epilogue's exact recipe reads them through L2)
  long long n;
  int d, k;
  int nx;                // f64 ring stages (mti_tc_stages)
  int gtc;               // CTAs that take tiles (<= gridDim.x; the rest write zero partials)
  int32_t* assign;
  double* upper;
  uint8_t* tight;
  const double* means;   // k x 16
  const double* drift;
  const double* half_min;
  const void* bimg;      // B operand image (launch_mti_tc_prep)
  double* partials;
  const Ctrl* ctrl;
  int gate;              // run only when ctrl->mti_choice == 1
  float* dbg;            // non-null: dump the n x N scores D~ and change nothing
  unsigned long long* counters;  // [0] uncertified (re-ranked) rows, cumulative
  uint32_t kmask;        // 0xFFFFFF80 (key mask, passed at run time)
  unsigned char* recs;   // per 128-row tile: moved-row masks (4 x u32) + old ids (u8 x 128)
  long long* rq;         // uncertified rows queued for mti_tc_rerank_kernel: {row, old id} pairs
  unsigned long long* rq_count;  // entries claimed this pass (zeroed by the prep kernel)
  long long rq_cap;      // queue capacity (rows beyond it are re-ranked inside the pass)
};
constexpr int TC_REC = 16 + 128;
cudaError_t launch_mti_tc_delta(const MtiTcArgs& a, int grid, cudaStream_t s);
int mti_tc_stages(int d, int k);
int mti_tc_prof(unsigned long long* out);  // 16 counters; returns 1 in a -DKNB_TCX_PROF=1 build
size_t mti_tc_bimg_bytes(int d, int k);
cudaError_t launch_mti_tc_prep(const double* means, int d, int k, void* bimg, unsigned long long* rq_count,
                               cudaStream_t s);
cudaError_t launch_mti_tc_rerank(const MtiTcArgs& a, int grid, cudaStream_t s);
cudaError_t launch_mti_tc(const CUtensorMap* tm, const MtiTcArgs& a, int grid, cudaStream_t s);

// staged copies between pageable host memory and HBM (hostcopy.cu)
constexpr size_t STAGE_MIN = 16ull << 20;  // smaller copies go straight through cudaMemcpy
cudaError_t staged_copy(int device, void* dst, const void* src, size_t bytes, bool h2d);
cudaError_t staging_reserve(int device);

// deterministic cluster-sorted accumulation (segsum.cu)
struct SegArgs {
  const void* X;         // f32 or f64 rows
  long long n;
  int d, k;
  const int32_t* assign;      // new labels
  const int32_t* old_assign;  // mode 1: labels before the pass
  const double* xn2;          // per-row ||x||^2 for the sq slot (or null)
  int mode;                   // 0: every row +x to assign; 1: moved rows +x new, -x old
  int B;                      // local blocks
  int* counts;                // [k][B]
  int* lrank;                 // [2n]
  int* ctot;                  // [k]
  int* cstart;                // [k + 1]
  int* istart;                // [k + 1]
  long long* sorted;          // [2n]
  double* records;            // [items][d + 2]
  double* exch;               // out: sums, counts, sq
  const Ctrl* ctrl;
};
int seg_blocks(long long n);
long long seg_max_items(long long n, int k);
cudaError_t launch_segsum(const SegArgs& a, int elem, cudaStream_t s);

// kernel selection helpers
int dense_mma_dp(int d);
size_t dense_mma_smem(int DP, int k, int d);
int dense_mma_rows();
cudaError_t launch_dense_mma(const CUtensorMap* tmap, const DenseArgs& a, int DP, int grid, cudaStream_t s);
int dense_tile_dp(int d);                       // padded dim for the register path, 0 = generic
size_t dense_tile_smem(int DP, int k, int d);
size_t mti_tile_smem(int DP, int k, int half_in_smem);

cudaError_t launch_dense(const CUtensorMap* tmap, const DenseArgs& a, int DP, int grid, cudaStream_t s);
cudaError_t launch_mti(const MtiArgs& a, int DP, int grid, cudaStream_t s);
bool mti_mma_fits(int DP, int k, int d);
bool mti_compact_ok(long long n_local);
cudaError_t launch_mti_mma(const MtiArgs& a, int DP, int grid, cudaStream_t s);
int dense_tile_grid(int DP, int k, int d, int sms);  // CTAs per device for the tensor-core path
int mti_tile_grid(int DP, int k, int half_in_smem, int sms);
int dense_rows_per_tile(int DP);

cudaError_t launch_reduce(const double* partials, int G, long long L, double* out, const Ctrl* ctrl,
                          cudaStream_t s);
cudaError_t launch_finalize(const FinalArgs& f, cudaStream_t s);
cudaError_t launch_geometry(const FinalArgs& f, cudaStream_t s);

// init helpers
// X is f64 (elem 8) or f32 (elem 4) rows
cudaError_t launch_gather_rows(const void* X, int elem, long long n_local, long long row_lo, int d,
                               const long long* ids, int count, double* out, cudaStream_t s);
cudaError_t launch_kpp_update(const void* X, int elem, long long n, int d, const double* c, double* d2,
                              int first, double* block_sums, int nblk, cudaStream_t s);
cudaError_t launch_kpp_psums(const double* d2, long long n, double total, double* block_sums,
                             int nblk, cudaStream_t s);
cudaError_t launch_kpp_search(const double* d2, long long n, double total, const double* block_sums,
                              int nblk, double threshold, long long* out, cudaStream_t s);
cudaError_t launch_sum_blocks(const double* block_sums, int nblk, double* out, cudaStream_t s);
// kmeans++ with every scalar on the device (single-GPU loop, no host round trips)
cudaError_t launch_kpp_psums_dev(const double* d2, long long n, const double* total, double* block_sums, int nblk,
                                 cudaStream_t s);
cudaError_t launch_kpp_search_dev(const double* d2, long long n, const double* total, const double* block_sums,
                                  int nblk, const double* cdf_end, const double* u, long long* out, int* degenerate,
                                  cudaStream_t s);
cudaError_t launch_gather_row_dev(const void* X, int elem, int d, const long long* idx, double* dst, cudaStream_t s);
cudaError_t launch_set_means(const double* src, int k, int d, FinalArgs f, int from_partition,
                             long long n, cudaStream_t s);
cudaError_t launch_validate(const double* X, long long n, int d, int k, const int32_t* assign,
                            const double* upper, const double* means, long long* bad,
                            cudaStream_t s);
cudaError_t launch_check_finite(const void* X, int elem, long long n, int d, long long* first_bad,
                                cudaStream_t s);

constexpr int KPP_BLOCK = 2048;  // rows per kmeans++ probability block (about 7 waves of CTAs at c2)

}  // namespace knb
