/*
 * bandmatch_gpu.h -- C ABI of the B200-native cascade-hashing matcher.
 *
 * Drop-in boundary for the hot path of the reference "bandmatch" library
 * (/root/reference/proj; citations are file:line in that tree).  The entry
 * points are what the reference's C++ API for this path binds to:
 *
 *   reference                                          | this ABI
 *   ---------------------------------------------------+------------------------------
 *   HashFunctions / make_hash_functions                | bmg_create (planes are host-
 *     include/bandmatch/hashmatch.hpp:19-34,             |   generated and passed in),
 *     src/hashmatch.cpp:53-69                           |   bmg_make_hash_functions
 *   DeviceArena::upload / evict + DeviceBackend hooks  | bmg_upload / bmg_evict /
 *     engine.hpp:20-44, 98-104; engine.cpp:18-40,       |   bmg_arena_stats
 *     438-444, 491-494                                  |
 *   execute_plan row body: centering mean + codes      | bmg_row / bmg_row_mean /
 *     engine.cpp:433-465                                |   bmg_codes
 *   compute_codes  hashmatch.hpp:58-61, .cpp:71-100     | bmg_compute_codes
 *   match_pair     hashmatch.hpp:82-90, .cpp:102-211    | bmg_match_pair, bmg_match
 *   execute_plan   engine.hpp:121-131, .cpp:411-527     | bmg_execute_plan
 *   bandmatch::Error codes  common.hpp:13-26            | bmg_status / bmg_status_name
 *
 * Conventions (mirroring the reference):
 *   - descriptors are float[n][128], row-major (Descriptor = std::array<float,128>,
 *     features.hpp:23-44), i.e. &fs.descriptors[0].v[0];
 *   - coarse codes are uint32[n][tables] (bucket ids), fine codes are
 *     uint64[n][ceil(fine_bits/64)] with fine bit b in word b/64, bit b%64
 *     (HashCodeSet, hashmatch.hpp:36-56);
 *   - matches are int32 (query_idx, train_idx) pairs in ascending query_idx
 *     (PairMatches, hashmatch.hpp:70-75); image pairs are (lower id, higher id)
 *     with query = lower id (IdPair, common.hpp:50-59; engine.cpp:469-472);
 *   - no C++ exception crosses this boundary: every call returns a bmg_status;
 *     bmg_status_name() gives the reference's stable error code string and
 *     bmg_last_error() the message.
 *
 * Results are bit-exact with the reference on the same inputs (hash codes,
 * bucket ids, Hamming ranking and the final match index sets).
 */
#ifndef BANDMATCH_GPU_H
#define BANDMATCH_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BMG_DIM 128 /* kDescriptorDim, features.hpp:14 */
#define BMG_ABI_VERSION 1

typedef enum {
  BMG_OK = 0,
  BMG_INVALID_ARGUMENT = 1,   /* "InvalidArgument"  */
  BMG_HASH_MISMATCH = 2,      /* "HashMismatch"     */
  BMG_CAPACITY_EXCEEDED = 3,  /* "CapacityExceeded" */
  BMG_NOT_RESIDENT = 4,       /* "NotResident"      */
  BMG_CUDA_ERROR = 5,         /* "CudaError"        */
  BMG_OUT_OF_MEMORY = 6,      /* "OutOfMemory"      */
  BMG_UNSUPPORTED = 7,        /* "Unsupported"      */
  BMG_INVALID_SCENE = 8,      /* "InvalidScene" / "ZeroVector" (features.cpp:60, 69-78) */
  BMG_FORMAT_ERROR = 9,       /* "FormatError"   (binary_io.hpp:63-67, features.cpp, hashmatch.cpp) */
  BMG_TRUNCATED_FILE = 10,    /* "TruncatedFile" (binary_io.hpp:37-43) */
  BMG_TOO_FEW_DESCRIPTORS = 11 /* "TooFewDescriptors" (retrieval.cpp:62-64, 94-96) */
} bmg_status;

typedef struct bmg_context bmg_context;
typedef struct bmg_result bmg_result;

/* HashParams, hashmatch.hpp:11-15 (defaults 6 / 8 / 128). */
typedef struct {
  int32_t tables;
  int32_t coarse_bits;
  int32_t fine_bits;
} bmg_hash_params;

/* MatchParams, hashmatch.hpp:77-80 (defaults 8 / 0.5). */
typedef struct {
  int32_t k_nearest;
  double ratio;
} bmg_match_params;

typedef struct {
  int32_t device;                 /* CUDA ordinal */
  bmg_hash_params hash;
  const float* coarse_planes;     /* [tables][coarse_bits][128] (HashFunctions::coarse) */
  const float* fine_planes;       /* [fine_bits][128]          (HashFunctions::fine)   */
  uint64_t function_seed;         /* HashFunctions::seed, tags every code set */
  uint64_t capacity_units;        /* DeviceArena capacity in descriptor units */
} bmg_config;

/* HashCodeSet view, hashmatch.hpp:36-56 */
typedef struct {
  uint64_t image_id;
  uint64_t function_seed;
  bmg_hash_params params;
  uint64_t count;
  const uint32_t* coarse;         /* [count][tables] */
  const uint64_t* fine;           /* [count][ceil(fine_bits/64)] */
} bmg_code_set;

/* FeatureSet view (descriptors only; keypoints stay on the host) */
typedef struct {
  uint64_t image_id;
  const float* descriptors;       /* [count][128] */
  uint64_t count;
} bmg_feature_view;

/* DeviceArena counters, engine.hpp:24-31 */
typedef struct {
  uint64_t capacity, occupancy, peak_occupancy, uploads, evictions, units_uploaded;
  uint64_t resident_count;
} bmg_arena_stats;

/* SchedulePlan flattened (mbr.hpp:26-68).  Rows are listed iteration by
 * iteration; row r's block pairs are pairs[2*row_pair_offsets[r] ..
 * 2*row_pair_offsets[r+1]) as (a,b) with a<b in block order, its
 * `needed` set is derived as row_images ∪ all blocks' col_images
 * (engine.cpp:434-436) and passed explicitly (ascending), and its eviction
 * directives are evict_ids[row_evict_offsets[r] .. row_evict_offsets[r+1]). */
typedef struct {
  uint64_t n_iterations;
  const uint64_t* rows_per_iteration;  /* [n_iterations] */
  uint64_t n_rows;
  const uint64_t* row_needed_offsets;  /* [n_rows+1] */
  const uint64_t* needed_ids;
  const uint64_t* row_pair_offsets;    /* [n_rows+1] */
  const uint64_t* pairs;               /* [2*total pairs] */
  const uint64_t* row_evict_offsets;   /* [n_rows+1] */
  const uint64_t* evict_ids;
} bmg_plan;

/* The hand-off point to host-side verification (VerifyPool::push,
 * engine.cpp:478-479): called on the executor's collector thread -- not the
 * caller's -- for every matched pair of a block row as soon as that row's
 * matches are in host memory, while later rows still run on the GPU.  Rows
 * come in the order the executor ran them, a row's pairs in plan (block)
 * order; a pair planned twice is handed over twice, like the reference's
 * push per match_pair call.  `matches` stays valid until bmg_result_free.
 * The callback may block (backpressure from a bounded verification queue)
 * without stalling the GPU; bmg_execute_plan returns after the last call. */
typedef void (*bmg_pair_callback)(void* user, uint64_t query_image, uint64_t train_image,
                                  const int32_t* matches, uint64_t n_matches);

/* DeviceBackend hooks (engine.hpp:98-104), called after each successful
 * arena transition. */
typedef void (*bmg_upload_hook)(void* user, uint64_t image_id, uint64_t units);
typedef void (*bmg_evict_hook)(void* user, uint64_t image_id);

typedef struct {
  bmg_match_params match;
  bmg_pair_callback on_pair;      /* may be NULL */
  void* on_pair_user;
  bmg_upload_hook on_upload;      /* may be NULL */
  bmg_evict_hook on_evict;        /* may be NULL */
  void* hook_user;
  uint32_t flags;                 /* BMG_EXEC_* */
} bmg_execute_options;

/* Keep every image resident: eviction directives are skipped (no free, no
 * bookkeeping).  Used to measure the row body on HBM-resident inputs. */
#define BMG_EXEC_RETAIN 1u
/* Row means (engine.cpp:446-461) are reconstructed exactly in parallel from
 * 128-bit fixed-point prefix sums plus the chain's rare rounding steps; this
 * flag computes them with the literal sequential FP64 chain instead (the
 * fallback path, exposed as a test hook -- results are identical). */
#define BMG_EXEC_MEAN_CHAIN 2u
/* Run every row on one stream (no overlap of consecutive rows): used to time
 * kernels in isolation; results are identical. */
#define BMG_EXEC_SERIAL 4u
/* Recompute the (mean-independent, per-residency) descriptor projections of
 * every resident image inside the call: used to time the complete row work
 * on HBM-resident inputs; results are identical. */
#define BMG_EXEC_REPROJECT 8u

/* ---- status ------------------------------------------------------------ */
const char* bmg_status_name(int status);              /* "InvalidArgument", ... */
const char* bmg_last_error(void);                     /* thread-local message */
int bmg_abi_version(void);

/* ---- host helpers mirroring the reference's host-side generation ------- */
/* seed_for, common.hpp:38-45 */
uint64_t bmg_seed_for(uint64_t root, const char* stage);
/* make_hash_functions, hashmatch.cpp:53-69 (libstdc++ <random>, host only) */
int bmg_make_hash_functions(uint64_t seed, const bmg_hash_params* params, float* coarse_out,
                            float* fine_out);

/* Synthetic band-overlap scene, generate_synthetic (features.cpp:68-197):
 * counts_out[n_images] first, then descriptors [sum counts][128] and
 * optionally keypoints [sum counts][4] (x, y, scale, orientation). */
int bmg_synthetic_counts(int n_images, int points_per_image, int overlap_band, double noise_sigma,
                         double outlier_fraction, uint64_t* counts_out);
int bmg_generate_synthetic(int n_images, int points_per_image, int overlap_band,
                           double noise_sigma, double outlier_fraction, uint64_t seed,
                           float* descriptors_out, float* keypoints_out);
/* The same scene keeping only the images with keep[i] != 0, stored back to
 * back in image order (a rank of a sharded plan generates what its shard
 * needs; the draws of the other images are still made, the observation
 * stream being shared, features.cpp:131-171). */
int bmg_generate_synthetic_subset(int n_images, int points_per_image, int overlap_band,
                                  double noise_sigma, double outlier_fraction, uint64_t seed,
                                  const uint8_t* keep, float* descriptors_out,
                                  float* keypoints_out);

/* ---- context ----------------------------------------------------------- */
int bmg_create(const bmg_config* config, bmg_context** out);
int bmg_destroy(bmg_context* ctx);
int bmg_synchronize(bmg_context* ctx);

/* ---- DeviceArena (HBM descriptor cache) --------------------------------- */
/* Uploads `count` descriptors for `image_id` (no-op when resident, engine.cpp:19);
 * CapacityExceeded when occupancy would exceed capacity (:20-24).  The copy is
 * asynchronous; `desc` must stay valid until the next bmg_row/bmg_synchronize. */
int bmg_upload(bmg_context* ctx, uint64_t image_id, const float* desc, uint64_t count);
int bmg_evict(bmg_context* ctx, uint64_t image_id);        /* NotResident (:34-36) */
int bmg_is_resident(bmg_context* ctx, uint64_t image_id);  /* 1 / 0 */
int bmg_arena_stats_get(bmg_context* ctx, bmg_arena_stats* out);

/* ---- row body (engine.cpp:446-465) --------------------------------------- */
/* Computes the centering mean over `needed` (ascending ids, all resident)
 * unless `mean` is non-NULL, then the codes and bucket tables of every
 * needed image relative to it.  Replaces the previous row's codes. */
int bmg_row(bmg_context* ctx, const uint64_t* needed, uint64_t n_needed, const float* mean);
int bmg_row_mean(bmg_context* ctx, float mean_out[BMG_DIM]);
/* Parity hook: copy the current row's codes of a needed image to the host. */
int bmg_codes(bmg_context* ctx, uint64_t image_id, uint32_t* coarse_out, uint64_t* fine_out);
/* match_pair over resident images of the current row: writes per-pair match
 * offsets [n_pairs+1] and (query_idx, train_idx) int32 pairs; capacity is in
 * pairs (int32 pairs, i.e. matches_out holds 2*capacity ints). */
int bmg_match(bmg_context* ctx, const uint64_t* query_ids, const uint64_t* train_ids,
              uint64_t n_pairs, const bmg_match_params* params, uint64_t* offsets_out,
              int32_t* matches_out, uint64_t capacity);

/* ---- stateless mirrors of the reference functions ------------------------ */
/* compute_codes(fs, hf, mean), hashmatch.cpp:71-100 */
int bmg_compute_codes(bmg_context* ctx, const float* desc, uint64_t count,
                      const float mean[BMG_DIM], uint32_t* coarse_out, uint64_t* fine_out);
/* match_pair(qf, qc, tf, tc, mp), hashmatch.cpp:102-211; HashMismatch on
 * seed / params / count disagreement, InvalidArgument on k_nearest < 1. */
int bmg_match_pair(bmg_context* ctx, const float* qdesc, const bmg_code_set* qc,
                   const float* tdesc, const bmg_code_set* tc, const bmg_match_params* params,
                   int32_t* matches_out, uint64_t* n_matches_out);

/* ---- full executor (engine.cpp:411-527, verification off) ---------------- */
int bmg_execute_plan(bmg_context* ctx, const bmg_plan* plan, const bmg_feature_view* features,
                     uint64_t n_features, const bmg_execute_options* options,
                     bmg_result** out);
/* A feature file (the "BMF1" layout of write_features, features.cpp:199-220)
 * as the source of an image: execute_plan reads it when the image uploads
 * -- the header checked like read_features (features.cpp:222-236), the
 * records read in blocks by host threads and de-interleaved straight into
 * pinned staging slots that the copy engine moves to HBM -- so the feature
 * map of a large plan need not sit in host memory (
 * load_features_dir, bandmatch_cli.cpp:56-74, reads everything up front).
 * `count` is the file's feature count (bmg_read_features_header); a file
 * that disagrees fails with InvalidArgument, a damaged one with the
 * reference's FormatError / TruncatedFile. */
typedef struct {
  uint64_t image_id;
  const char* path;
  uint64_t count;
} bmg_feature_file;
int bmg_execute_plan_files(bmg_context* ctx, const bmg_plan* plan, const bmg_feature_file* files,
                           uint64_t n_files, const bmg_execute_options* options, bmg_result** out);

/* ExecutionResult accessors: pairs sorted by IdPair (engine.cpp:506-512). */
uint64_t bmg_result_pair_count(const bmg_result* r);
uint64_t bmg_result_match_count(const bmg_result* r);
/* pair_ids[2*n_pairs], offsets[n_pairs+1], matches[2*n_matches] */
int bmg_result_copy(const bmg_result* r, uint64_t* pair_ids, uint64_t* offsets, int32_t* matches);
/* Zero-copy view, valid until bmg_result_free: pair_ids[2*n_pairs] (sorted
 * by IdPair), ranges[2*n_pairs] = [begin, end) of each pair's matches in
 * `log`, an int32 (query_idx, train_idx) array in pinned host memory. */
int bmg_result_view(const bmg_result* r, const uint64_t** pair_ids, const uint64_t** ranges,
                    const int32_t** log);
/* PipelineMetrics, engine.hpp:57-78: pairs_matched, initial_matches, uploads,
 * evictions, units_uploaded, peak_occupancy (6 values) + wall seconds */
int bmg_result_metrics(const bmg_result* r, uint64_t counters_out[6], double* wall_s_out);
/* per-iteration metrics: pairs, uploads, units_uploaded (3 values each) */
uint64_t bmg_result_iteration_count(const bmg_result* r);
int bmg_result_iteration(const bmg_result* r, uint64_t i, uint64_t out[3]);
/* Device time (CUDA events on the compute stream) from the first operation of
 * the first row to the last kernel of the last row. */
int bmg_result_device_ms(const bmg_result* r, double* ms_out);
/* Overlap diagnostics for plan row `row`, both in ms since the call's first
 * device operation was issued (host and device clocks aligned to within the
 * launch latency): out[0] = when its pairs were handed to on_pair (-1
 * without on_pair), out[1] = when its last kernel / copy finished. */
int bmg_result_row_timing(const bmg_result* r, uint64_t row, double out[2]);
void bmg_result_free(bmg_result* r);
/* write_matches_binary (hashmatch.cpp:311-332) of the result: the "BMMT" file
 * the reference writes for the same ExecutionResult, byte for byte (pairs in
 * IdPair order, stage Initial), straight from the pinned log. */
int bmg_result_write_matches(const bmg_result* r, const char* path);

/* ---- file formats either side of the path ------ */
/* read_features (features.cpp:222-249): header only (image id, count). */
int bmg_read_features_header(const char* path, uint64_t* image_id, uint64_t* count);
/* read_features into caller buffers (e.g. pinned host memory for the H2D):
 * descriptors_out[count][128], keypoints_out[count][4] (x, y, scale,
 * orientation; may be NULL), capacity = features the buffers hold; the
 * records are read in large blocks by `threads` threads.  Same checks and
 * error codes / messages as the reference (FormatError, TruncatedFile). */
int bmg_read_features(const char* path, uint64_t capacity, float* descriptors_out,
                      float* keypoints_out, int threads, uint64_t* image_id, uint64_t* count);
/* write_matches_binary (hashmatch.cpp:311-332) from flat arrays: pair_ids
 * [2*n_pairs] sorted by IdPair, ranges[2*n_pairs] = [begin, end)
 * into log (int32 (qi, ti) pairs), stages[n_pairs] (0 = Initial, 1 =
 * Verified; NULL = all Initial). */
int bmg_write_matches_binary(const char* path, uint64_t n_pairs, const uint64_t* pair_ids,
                             const uint64_t* ranges, const int32_t* log, const uint8_t* stages);

/* ---- host verification, stage 1 --------------------- */
/* sao_filter (verify.cpp:303-341) with the reference's results: the spatial-
 * angular-order filter over the pair's initial matches, its Bowyer-Watson
 * Delaunay (verify.cpp:47-107) run with adjacency (walking point location +
 * cavity growth) instead of the reference's all-triangle scan per point.
 * matches[2*m] = (query_idx, train_idx); keypoints [n][4] = (x, y, scale,
 * orientation) as Keypoint (features.hpp); SaoParams n_neighbors (>= 1) and
 * score_threshold (>= 0) as in verify.hpp.  Outputs per input match: keep
 * (score <= threshold) and the score; flags: BMG_SAO_*.  InvalidArgument as
 * the reference raises it.  Host code: no device needed. */
/* Retrieval: encode_vlad (retrieval.hpp:36-47, retrieval.cpp:160-205) for a
 * batch of images -- what select_pairs (retrieval.cpp:386-399) calls once per
 * image.  centroids: float[k_words][128] (Codebook::centroids); images[i]:
 * its descriptors (pinned or pageable host memory; image_id is ignored);
 * values_out: float[n_images][k_words*128] (VladVector::values);
 * degenerate_out: uint8[n_images].  Bit-exact with the reference (nearest
 * centroid, FP64 residual sums in descriptor order, signed square root,
 * sequential norm).  InvalidArgument "codebook has no words" for k_words < 1;
 * Unsupported for k_words > 1024. */
int bmg_encode_vlad(bmg_context* ctx, const float* centroids, int k_words, const bmg_feature_view* images,
                    uint64_t n_images, float* values_out, uint8_t* degenerate_out);
/* train_codebook (retrieval.hpp:26-34, retrieval.cpp:56-158) on the B200:
 * Lloyd iterations over descriptors[n][128] with the reference's seeding
 * (mt19937_64 shuffle, k distinct values), nearest-centroid assignment
 * (FP64 semantics, certified FP32 filter), FP64 cluster sums in point order,
 * empty clusters reseeded from the farthest point, stop at an assignment
 * fixpoint or max_iters.  centroids_out: float[k_words][128]; sse_out (may be
 * NULL): the within-cluster SSE of every assignment step (at most max_iters),
 * *n_sse_out their number.  Bit-exact with the reference.  Errors as the
 * reference: InvalidArgument (k_words < 1, max_iters < 1), TooFewDescriptors
 * (n < k_words, or fewer than k_words distinct values); Unsupported for
 * k_words > 1024. */
int bmg_train_codebook(bmg_context* ctx, const float* descriptors, uint64_t n, int k_words, int max_iters,
                       uint64_t seed, float* centroids_out, double* sse_out, int* n_sse_out);

/* knn_from_delaunay (verify.cpp:135-196): per point its k neighbours by
 * Delaunay rings (neighbors_out[n][k], -1 padded); *fallback = 1 when the
 * set could not be triangulated (duplicates, collinear) and plain nearest
 * neighbours were used.  xy[n][2] doubles (Point2). */
int bmg_delaunay_knn(const double* xy, uint64_t n, int k, int32_t* neighbors_out, int* fallback);
#define BMG_SAO_PASSTHROUGH 1u       /* fewer than n_neighbors + 1 matches: all kept */
#define BMG_SAO_DELAUNAY_FALLBACK 2u /* a side could not be triangulated: plain k-NN */
int bmg_sao_filter(const int32_t* matches, uint64_t n_matches, const float* query_keypoints,
                   uint64_t n_query, const float* train_keypoints, uint64_t n_train, int n_neighbors,
                   double score_threshold, uint8_t* keep_out, double* scores_out, uint32_t* flags_out);

/* ---- instrumentation ------------------------------------------------------ */
/* Number of kernels this context has launched so far. */
uint64_t bmg_launch_count(bmg_context* ctx);
/* Device time of the most recent bmg_execute_plan / bmg_match, per kernel
 * class ("mean", "codes", "fixup", "tables", "match", "compact"): total
 * milliseconds and launch count, measured with CUDA events on the launching
 * stream.  Enabled by bmg_set_profiling(ctx, 1). */
int bmg_set_profiling(bmg_context* ctx, int enabled);
int bmg_kernel_time(bmg_context* ctx, const char* kernel_class, double* total_ms,
                    uint64_t* launches);
/* Number of projection bits / ratio decisions resolved by the FP64 fixup
 * path in the last row / match (diagnostics). */
int bmg_fixup_counts(bmg_context* ctx, uint64_t* code_bits, uint64_t* rerank_queries);
/* Number of queries of the last row / match whose candidate top-K was redone
 * on the matcher's exact insertion path (a lane's short key list may have
 * dropped a top-K key; diagnostics). */
int bmg_exact_walk_count(bmg_context* ctx, uint64_t* queries);
/* How the last computed row mean was obtained (diagnostics): `rounds` =
 * 1 + the largest number of tiles any channel had to walk (tiles the F96
 * certificate could not clear; every rounding step lies in one of them),
 * `used_chain` = 1 when the sequential FP64 chain produced it (fallback or
 * BMG_EXEC_MEAN_CHAIN). */
int bmg_row_mean_info(bmg_context* ctx, uint32_t* rounds, int* used_chain);
/* Test hooks: route every query of later matches through the exact top-K
 * walk (the path a lane's dropped key triggers) and / or every ratio
 * decision through the FP64 reference re-rank (the path near ties take).
 * Results are identical; only speed changes. */
#define BMG_TEST_FORCE_EXACT_WALK 1u
#define BMG_TEST_FORCE_FP64_RERANK 2u
int bmg_set_test_flags(bmg_context* ctx, uint32_t flags);

#ifdef __cplusplus
}
#endif

#endif /* BANDMATCH_GPU_H */
