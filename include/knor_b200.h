/* knor_b200.h -- C ABI of libknorb200.so, the B200 (sm_100a) Lloyd / MTI k-means path.
 *
 * The reference (numakmeans, knor arXiv 1606.08905) is a pure-Python package whose
 * only public entry to this path is
 *     kmeans(matrix, EngineConfig) -> KmeansResult           engine.py:489-500
 * with no FFI of its own.  This header is the plain-pointer boundary that a ctypes
 * (or cffi / C++) binding calls instead of the reference's in-process engine; the
 * Python package paper_1606_08905_b200 is such a binding and mirrors the reference API.
 * Each entry point names the reference code it replaces.
 *
 * Conventions: every function returns 0 on success or a negative KNB_E* code;
 * knb_last_error() returns a thread-local message for the last failure.  A context
 * (knb_ctx) owns one GPU's contiguous row shard [row_lo, row_lo + n_local) of an
 * n_global x d matrix (partition_rows, matrix.py:196-213) and all per-point state;
 * it is not thread-safe.  All work is enqueued on the context's CUDA stream; the
 * functions that return host data synchronise it.  Host pointers are plain,
 * C-contiguous arrays; device pointers are marked "dev".
 */
#ifndef KNOR_B200_H
#define KNOR_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KNB_OK 0
#define KNB_E_ARG (-1)     /* invalid argument            -> ValueError      */
#define KNB_E_CUDA (-2)    /* CUDA runtime / driver error -> RuntimeError    */
#define KNB_E_STATE (-3)   /* call out of order           -> RuntimeError    */
#define KNB_E_COUNT (-4)   /* Sigma counts != n            -> RuntimeError (engine.py:378-380) */
#define KNB_E_NOMEM (-5)   /* device allocation failed    -> MemoryError     */

typedef struct knb_ctx knb_ctx;

/* One row of IterationStats (engine.py:124-144). */
typedef struct {
  int64_t t;
  int64_t reassignments;
  double wcss;
  int64_t dist_comps;
  int64_t skips;
  int64_t pruned_stale;
  int64_t pruned_tight;
  int32_t converged;
  int32_t stop;
  int64_t count_total;
} knb_iter_stats;

int knb_version(void);
const char* knb_last_error(void);
/* SM count, HBM bytes and compute capability of a device. */
int knb_device_info(int device, int* sms, int64_t* hbm_bytes, int* cc_major, int* cc_minor);

/* _Engine.__init__ (engine.py:212-254) for one shard: allocates assignment (int32, zeroed
 * as at engine.py:226), and for pruning runs the upper bound (f64) and tight flag (u8)
 * state (engine.py:227-235) plus running sums.  stream may be NULL (a private stream is
 * created).  max_iters / tolerance are EngineConfig's (engine.py:63-72). */
int knb_create(int device, int64_t n_global, int64_t n_local, int64_t row_lo, int32_t d,
               int32_t k, int32_t pruning, int32_t max_iters, double tolerance, void* stream,
               knb_ctx** out);
int knb_destroy(knb_ctx* ctx);
/* Device memory of destroyed contexts stays in the library's pool for the next context
 * (no reference counterpart: the reference allocates numpy arrays per call).  This hands
 * the unused part back to the driver -- torch.cuda.empty_cache's counterpart. */
int knb_release_memory(int device);

/* Rows of the shard: copy from host (any pointer; pinned is faster) into a context-owned
 * buffer, or attach caller-owned device rows.  Replaces _MemorySource (engine.py:162-191). */
int knb_upload_rows(knb_ctx* ctx, const double* host, int64_t row_lo_local, int64_t rows);
int knb_attach_rows(knb_ctx* ctx, const double* dev_rows);
/* Rows that stay in host memory (larger than HBM): the caller's array is page-locked and
 * mapped (cudaHostRegister) and every kernel reads it over the host link; clause-1
 * skipped rows of a pruned pass are never fetched -- the B200 form of the reference's
 * semi-external mode with row elision (outofcore.py:163-225, §8(f) f2).  The array must
 * outlive the context (unregistered by knb_destroy). */
int knb_attach_host_rows(knb_ctx* ctx, const double* host_rows);
/* Semi-external run (kmeans_ondisk, outofcore.py:440-455; _DiskSource :293-355): from now
 * on every iteration (1) marks the rows the reference would fetch -- all rows on a full
 * pass (task_rows), the survivors of clause 1 on a pruned pass (rows_by_ids) -- and keeps
 * the reference's I/O counters for it exactly (fetch_rows, :163-225: bytes requested, cache
 * hits/misses against the published cache, page_size x distinct pages of each task's
 * uncached rows), and (2) at the refresh iterations start, 3 start, 7 start, ...
 * (should_refresh, :282-290) rebuilds an HBM row cache like RowCache.rebuild (:250-270):
 * each of the T worker partitions keeps its smallest (capacity / T) / row_bytes fetched row
 * ids.  Pruned passes over host rows gather cached rows from HBM instead of the host link.
 * One GPU holding the whole matrix (n_local == n_global), f64 rows; call before the
 * centroids are installed.  Same argument errors as the reference (T, task_size,
 * page_size >= 1, capacity >= 0, refresh start >= 1). */
int knb_sem_configure(knb_ctx* ctx, int32_t T, int64_t task_size, int64_t page_size,
                      int32_t cache_enabled, int64_t cache_capacity, int32_t refresh_start);
/* Per-iteration IoDelta (engine.py:112-118) of the first `count` iterations, 5 int64 per
 * iteration: bytes_requested, bytes_read, cache_hits, cache_misses, rows fetched
 * (rows_elided is the iteration's skips). */
int knb_sem_io(knb_ctx* ctx, int64_t* out, int32_t count);
/* The published cache: row ids (slot order: partition, then ascending id) and, if rows is
 * non-null, their cached values (cap x d); *count = cached rows (may exceed cap). */
int knb_sem_cache(knb_ctx* ctx, int64_t* ids, double* rows, int64_t cap, int64_t* count);
/* f32 rows (BASELINE config 5), kept as f32 in HBM -- the reference upcasts them to f64
 * (matrix.py:40), which is exact, and every result here equals the f64 upcast's.  Only the
 * dense tensor-core path takes them: knb_f32_supported(d, k, pruning) says whether it
 * applies (pruning off, d % 4 == 0, 32 <= d <= 256); elsewhere the caller upcasts.
 * Scores come from tcgen05 kind::tf32 with a certified bound; uncertified rows are
 * re-scored with the exact f64 recipe (distance.py:28-39, :94-116). */
int knb_f32_supported(int32_t d, int32_t k, int32_t pruning);
int knb_upload_rows_f32(knb_ctx* ctx, const float* host, int64_t row_lo_local, int64_t rows);
int knb_attach_rows_f32(knb_ctx* ctx, const float* dev_rows);
/* Tensor-core path counters since the last centroid install: rows whose certificate
 * failed (re-scored exactly) and, of those, rows re-scored against all k. */
int knb_tc_info(knb_ctx* ctx, int32_t* active, int64_t* flagged_rows, int64_t* full_reranks);
/* Diagnostics of the certificate: the tensor-core scores x.c_j - ||c_j||^2/2 (f32) of every
 * shard row against the current centroids into dev_out (n_local x k_pad, k rounded up to
 * 256; padding scores are -inf), and the relative error e the certificate assumes
 * (|score error| <= e ||x|| max_j ||c_j|| + rounding terms).  Assignments are untouched. */
int knb_tc_scores(knb_ctx* ctx, float* dev_out, double* err_rel);
/* check_matrix's finite scan (matrix.py:46-48): *first_bad = first shard-local row with a
 * NaN/inf, or -1. */
int knb_check_finite(knb_ctx* ctx, int64_t* first_bad);

/* Exchange vector: the per-shard accumulator that crosses GPUs once per iteration
 * (sums k*d, counts k, sq k, 8 scalars: the merged Accumulator of centroids.py:55-107 plus
 * the counters).  A caller doing multi-GPU all-reduces it in place between the *_local and
 * *_finish calls; it may supply its own device buffer (e.g. a torch tensor). */
int knb_exchange_len(knb_ctx* ctx, int64_t* len);
int knb_set_exchange(knb_ctx* ctx, double* dev, int64_t len);
int knb_exchange_ptr(knb_ctx* ctx, double** dev);

/* init_centroids (centroids.py:131-189).  given: knb_set_centroids.  forgy / kmeans++ rows:
 * knb_init_gather writes the requested global rows this shard owns into the exchange
 * (zeros elsewhere; all-reduce across shards), then knb_init_from_exchange installs the
 * first `count` rows as centroids 0..count-1.  random-partition: knb_init_partition_local
 * accumulates the shard's rows by group label into the exchange, knb_init_partition_finish
 * installs group means (empty group -> global mean) and resets the assignment to zero. */
int knb_set_centroids(knb_ctx* ctx, const double* host_means);
int knb_init_gather(knb_ctx* ctx, const int64_t* global_ids, int32_t count);
int knb_init_from_exchange(knb_ctx* ctx, int32_t first, int32_t count);
int knb_init_partition_local(knb_ctx* ctx, const int32_t* host_labels_local);
int knb_init_partition_finish(knb_ctx* ctx);
/* kmeans++ (centroids.py:175-189): d2 = min(d2, dist(x, c)^2) against the row in
 * exchange[0:d]; returns the shard's sum of d2.  psum returns the shard's sum of d2/total;
 * search returns the first shard-local row whose running sum of d2/total exceeds
 * `threshold` (the sampled index of Generator.choice). */
int knb_kpp_update(knb_ctx* ctx, int32_t first, double* local_total);
int knb_kpp_psum(knb_ctx* ctx, double total, double* local_psum);
int knb_kpp_search(knb_ctx* ctx, double total, double threshold, int64_t* local_idx);
/* Single-GPU kmeans++ in one call: first_pick = rng.integers(n) and u[0..k-2] = the next
 * k - 1 rng.random() draws of the host stream (centroids.py:174-189 consumes exactly these
 * while the D^2 total stays > 0); the D^2 updates, totals, cumulative sums and searches run
 * on the device without host round trips, then the k rows are installed.  *degenerate = 1
 * (nothing installed) when a total is 0 -- the caller replays the reference's draw order
 * with the step-wise calls below. */
int knb_kpp_run(knb_ctx* ctx, int64_t first_pick, const double* u, int32_t k, int64_t* picks, int32_t* degenerate);
int knb_kpp_release(knb_ctx* ctx);

/* One Lloyd iteration, split around the cross-GPU exchange:
 *   local  -- engine._task_full / _task_pruned over every row of the shard (K1 or
 *             K6/K7) and the fixed-order merge of CTA partials into the exchange;
 *   finish -- the barrier action (engine.py:358-426): running sums, Sigma counts == n,
 *             finalize, WCSS, stats row, convergence, MTI geometry.
 * knb_iterate = local + finish + the stats row (single shard). */
int knb_iter_local(knb_ctx* ctx);
int knb_iter_finish(knb_ctx* ctx);
int knb_iterate(knb_ctx* ctx, knb_iter_stats* out);
/* Iterate a single-shard run until it stops (converged or max_iters), synchronising with
 * the host only every `batch` iterations (the stop flag lives on the device). */
int knb_run(knb_ctx* ctx, int32_t batch, int32_t* iterations_done);
/* EngineConfig.validate_bounds test mode (engine.py:428-445), between local and finish:
 * first row whose assignment != exhaustive argmin and first row whose bound is below its
 * true distance (-1 when none). */
/* Enqueue up to `count` iterations (fewer at max_iters) without synchronising: iterations
 * after the first replay one captured CUDA graph (local pass + finish, every decision on
 * device).  Single-GPU only -- a multi-GPU caller all-reduces between knb_iter_local and
 * knb_iter_finish instead.  The bench's timed loop. */
int knb_enqueue(knb_ctx* ctx, int32_t count);
int knb_validate(knb_ctx* ctx, int64_t* bad_assign_row, int64_t* bad_bound_row);

/* Results: IterationStats rows so far, CentroidSet (centroids.py:15-52), assignments
 * (KmeansResult.assignments, engine.py:480), MTI bounds (PruneState, pruning.py:64-81). */
int knb_get_stats(knb_ctx* ctx, knb_iter_stats* out, int32_t max_count, int32_t* count);
int knb_get_state(knb_ctx* ctx, int32_t* stop, int32_t* converged, int64_t* t, int32_t* count_error);
int knb_get_centroids(knb_ctx* ctx, double* means, double* prev_means, int64_t* counts, double* drift);
int knb_get_assignments(knb_ctx* ctx, int32_t* out, int64_t lo, int64_t count);
/* Host transfers of 16 MB or more between pageable caller memory and HBM (the rows of
 * knb_upload_rows / _f32, the assignments of knb_get_assignments) are staged through a
 * pool of pinned chunks by eight threads, overlapping CPU copies with DMA.  The pool is
 * allocated on first use; knb_staging_reserve allocates it ahead of a timed call. */
int knb_staging_reserve(int device);
int knb_get_bounds(knb_ctx* ctx, double* upper, uint8_t* tight);
int knb_sync(knb_ctx* ctx);
/* Benchmark hook: keep running full iterations after convergence (kmeans() never sets it). */
int knb_set_ignore_stop(knb_ctx* ctx, int32_t on);
/* Enqueue this context's work on `stream` from now on (NULL = the legacy default
 * stream).  Lets a caller capture whole iterations -- local pass, its own all-reduce,
 * finish -- into one CUDA graph on its capture stream (bench.py does at N > 1). */
int knb_set_stream(knb_ctx* ctx, void* stream);
/* Options.  KNB_OPT_MTI_SCAN selects how a pruned iteration re-assigns the survivors of the
 * point-skip test (clause 1): KNB_MTI_EXACT walks the candidates with clauses 2/3 exactly like
 * scan_block (pruning.py:163-204), reproducing its dist_comps / pruned_* counters;
 * KNB_MTI_DENSE compacts survivors per warp and scores them on the FP64 tensor cores
 * (certified argmin, exact bound) -- identical assignments, bounds, skips and centroids,
 * dist_comps = k per survivor; KNB_MTI_BLOCK streams every block through the tensor-core
 * pass and skips only blocks whose rows all pass clause 1 (same outputs); KNB_MTI_AUTO
 * (default, d <= 64 and centroids in shared memory) picks BLOCK or DENSE on the device each
 * iteration from the previous iteration's skip fraction. */
#define KNB_OPT_MTI_SCAN 1
#define KNB_MTI_AUTO 0
#define KNB_MTI_EXACT 1
#define KNB_MTI_DENSE 2
#define KNB_MTI_BLOCK 3
/* KNB_MTI_TC: the block pass on the tcgen05 tensor cores for f64 rows with d == 16 and
 * k <= 128 (split-TF32 scores, certified argmin, exact re-rank of uncertified rows; same
 * outputs as BLOCK).  Under KNB_MTI_AUTO it replaces BLOCK wherever it applies. */
#define KNB_MTI_TC 4
int knb_set_option(knb_ctx* ctx, int32_t option, int64_t value);
/* 1 when a shard of n_local rows may run the compacted (DENSE) MTI kernel, whose filter
 * uses 32-bit row indices (n_local <= 2^31 - 2^26); larger shards run the BLOCK pass under
 * KNB_MTI_AUTO / KNB_MTI_DENSE (same results).  Host-only, no device needed. */
int knb_mti_compact_ok(int64_t n_local);
/* Device bytes held by the context (the GPU analogue of KmeansResult.peak_state_bytes). */
int knb_state_bytes(knb_ctx* ctx, int64_t* bytes);
/* Which kernels the context uses: padded width (0 = generic, < 0: f32 rows on the tcgen05
 * path with that padded width), TMA on/off, grid sizes (grid_mti < 0: the tensor-core MTI
 * kernel with -grid_mti CTAs). */
int knb_describe(knb_ctx* ctx, int32_t* dense_dp, int32_t* use_tma, int32_t* grid_dense, int32_t* grid_mti);
/* The tcgen05 MTI pass (KNB_MTI_TC): whether it applies to this context, and how many
 * rows it could not certify (re-ranked with the exact recipe) since the run started. */
int knb_mti_tc_info(knb_ctx* ctx, int32_t* available, int64_t* uncertified);
/* Test hook: the pass's split-TF32 scores D~ (n_local x N floats, N = k rounded up to 16,
 * ~ ||x - c_j||^2) against the current centroids, into device memory; no state changes. */
int knb_mti_tc_scores(knb_ctx* ctx, float* dev_out);
/* Profiling builds (-DKNB_TCX_PROF=1): cycles each role of the tcgen05 MTI kernel spent
 * waiting / working, summed over CTAs since the last call (then cleared); *enabled = 0 and
 * zeros in normal builds.  Slots: producer [0 wait x_empty, 1 issue], issuer [2 wait A,
 * 3 wait TMEM, 4 issue], converter [5 wait x_full, 6 wait A slot, 7 work], epilogue [8 wait
 * TMEM full, 9 keys, 10 wait rows, 11 certify + bound + state, 12 accumulate, 13 other]. */
int knb_mti_tc_prof(int64_t* out16, int32_t* enabled);

/* numpy's default_rng(seed).random(...) on the device: writes draws [first_draw,
 * first_draw + count) of the PCG64 stream whose (state, inc) the host read from
 * Generator.bit_generator.state into dev_out, bit-identical to the host stream (config 4's
 * U[0,1)^16 input).  Context-free; stream may be NULL. */
int knb_fill_uniform_pcg64(double* dev_out, int64_t count, int64_t first_draw, uint64_t state_hi,
                           uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, void* stream);

/* The reference's distance primitives on the device (context-free, host pointers, same
 * exact recipe as the engine): block_distances / nearest_centroid (distance.py:42-82) --
 * dist_out (m x k) and/or ids_out / best_out (ascending strict-less argmin per row); any
 * output may be NULL.  knb_rowwise: rowwise_distances (distance.py:36-39, refs m x d or one
 * shared row) or, with refs NULL, row_sqnorms (distance.py:66-72); take_sqrt selects the
 * distance or the squared sum. */
int knb_block_distances(int device, const double* rows, int64_t m, const double* cents, int32_t k, int32_t d,
                        double* dist_out, int32_t* ids_out, double* best_out);
int knb_rowwise(int device, const double* rows, int64_t m, const double* refs, int32_t shared_ref, int32_t d,
                int32_t take_sqrt, double* out);

/* Roofline denominators measured on the device: FP64 FMA rate (DFMA/s, 8 independent chains
 * per thread over 8 CTAs/SM) and a 1 GiB device copy (read + write bytes/s). */
int knb_measure_peaks(int device, double* dfma_per_s, double* copy_bytes_per_s);

#ifdef __cplusplus
}
#endif

#endif /* KNOR_B200_H */
