// Device-side run state shared by every kernel of one context (one GPU shard).
#pragma once

#include <stdint.h>

#define KNB_NT 256  // threads per CTA for the streaming kernels
#define KNB_WARPS (KNB_NT / 32)

namespace knb {

// Control block, resident in device memory so that a whole iteration (and a
// CUDA graph of iterations) runs without reading anything back to the host.
struct Ctrl {
  long long t;           // iteration about to run (or just finalized)
  int stop;              // convergence / max_iters reached (engine.py:413-416)
  int converged;
  int full_pass;         // 1 until the first finalize of a pruned run
  int count_error;       // Sigma counts != n (engine.py:378-380)
  int ignore_stop;       // bench: keep iterating after convergence (never set by kmeans())
  int max_iters;
  double tolerance;      // reassigned <= tolerance converges
  int mti_choice;        // next pruned pass: 1 = block-dense (few skips), 0 = compacted survivors
  int block_pct;         // the block (or tcgen05) pass runs while clause 1 skips < block_pct % of rows
  double cmax2;          // max_j ||c_j||^2 of the current means (dense certificate)
  long long count_seen;  // last Sigma counts
};

// One row of per-iteration statistics (IterationStats, engine.py:124-144).
struct IterStatsDev {
  long long t;
  long long reassignments;
  double wcss;
  long long dist_comps;
  long long skips;
  long long pruned_stale;
  long long pruned_tight;
  int converged;
  int stop;
  long long count_total;
};

// Layout of one accumulator vector (a per-CTA partial, or the exchange
// buffer that is all-reduced across GPUs): all doubles.
//   [0, k*d)        sums
//   [k*d, k*d+k)    counts (exact integers in f64)
//   [k*d+k, +k)     sq (sum of squared row norms, pruned runs)
//   then NSCAL scalars:
enum Scalar { S_REASSIGNED = 0, S_WCSS, S_COMPUTED, S_SKIPS, S_PSTALE, S_PTIGHT, S_ROWS, S_SPARE, NSCAL };

__host__ __device__ inline long long acc_len(int k, int d) { return (long long)k * d + 2LL * k + NSCAL; }

}  // namespace knb
