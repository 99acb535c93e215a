// Internal launcher interface between the C-ABI layer (capi.cu) and the kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "state.cuh"

namespace knb {

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
};

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
  Ctrl* ctrl;
  IterStatsDev* stats;   // [max_iters]
};

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
cudaError_t launch_mti_mma(const MtiArgs& a, int DP, int grid, cudaStream_t s);
int dense_tile_grid(int DP, int k, int d, int sms);  // CTAs per device for the tensor-core path
int mti_tile_grid(int DP, int k, int half_in_smem, int sms);
int dense_rows_per_tile(int DP);

cudaError_t launch_reduce(const double* partials, int G, long long L, double* out, const Ctrl* ctrl,
                          cudaStream_t s);
cudaError_t launch_finalize(const FinalArgs& f, cudaStream_t s);
cudaError_t launch_geometry(const FinalArgs& f, cudaStream_t s);

// init helpers
cudaError_t launch_gather_rows(const double* X, long long n_local, long long row_lo, int d,
                               const long long* ids, int count, double* out, cudaStream_t s);
cudaError_t launch_kpp_update(const double* X, long long n, int d, const double* c, double* d2,
                              int first, double* block_sums, int nblk, cudaStream_t s);
cudaError_t launch_kpp_psums(const double* d2, long long n, double total, double* block_sums,
                             int nblk, cudaStream_t s);
cudaError_t launch_kpp_search(const double* d2, long long n, double total, const double* block_sums,
                              int nblk, double threshold, long long* out, cudaStream_t s);
cudaError_t launch_sum_blocks(const double* block_sums, int nblk, double* out, cudaStream_t s);
cudaError_t launch_set_means(const double* src, int k, int d, FinalArgs f, int from_partition,
                             long long n, cudaStream_t s);
cudaError_t launch_validate(const double* X, long long n, int d, int k, const int32_t* assign,
                            const double* upper, const double* means, long long* bad,
                            cudaStream_t s);
cudaError_t launch_check_finite(const double* X, long long n, int d, long long* first_bad,
                                cudaStream_t s);

constexpr int KPP_BLOCK = 4096;  // rows per kmeans++ probability block

}  // namespace knb
