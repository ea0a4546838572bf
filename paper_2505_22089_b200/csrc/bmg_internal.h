// bmg_internal.h -- device-side data layout shared by the sm_100a kernels and
// the host runtime (bmg_api.cpp).  See DESIGN.md §3 for the HBM layout.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace bmg {

constexpr int kDim = 128;

// One image as seen by the kernels during a block row: descriptors live in
// the HBM arena; codes and bucket tables live in the row scratch buffer.
struct ImgDev {
  const float* desc;   // [n][128] row-major (Descriptor layout, features.hpp:23-44)
  uint32_t* coarse;    // [n][tables] bucket ids            (HashCodeSet::coarse)
  uint64_t* fine;      // [n][fwp] fine code words, fwp >= ceil(fine_bits/64), zero padded
  uint32_t* offsets;   // [tables][n_buckets+1] bucket starts (hashmatch.cpp:125-135)
  uint32_t* cursor;    // [tables][n_buckets]   scatter cursors (scratch)
  uint32_t* slots;     // [tables][ns] train indices grouped by bucket (:136-145),
                       // buckets padded to 8 entries (pad index 0xffffffff); the
                       // last 8 entries of each table are an all-pad sentinel chunk
  uint64_t* bfine;     // [tables][ns][fwp] fine codes in slot order (coalesced candidate walk)
  float* proj;          // [n][proj_stride] fl32(d . p) for every plane (mean-independent, per residency)
  float* dnorm;         // [n] ||d||_2 rounded up
  // row-mean tile statistics of the image (kernels.cu K1), per 128-
  // descriptor tile and channel, computed with its projections: F96 sum
  // (i128), range of the partial sums (2 x i128), lowest set F96 bit
  // (kNoLow: all zeros, kBadTile: a value outside F96); null when absent
  void* tsum;
  void* trng;
  uint32_t* tlow;
  uint32_t n;
  uint32_t overflow;   // set by the codes kernel when its fixup list overflowed
  uint32_t ns;         // slot stride per table: slot_stride(n, n_buckets)
  uint32_t pad_;
};

struct HashDev {
  int tables, coarse_bits, fine_bits;
  int n_planes;        // tables*coarse_bits + fine_bits
  int fw;              // ceil(fine_bits/64)
  int fwp;             // padded words (1,2,4,8,16)
  int n_buckets;       // 1 << coarse_bits
  const float* planes_t;   // [128][n_planes_pad] transposed planes, zero padded
  const float* planes;     // [n_planes][128] planes (coarse first, then fine)
  const float* plane_norm; // [n_planes_pad] ||p||_2 rounded up, 0 for padding
  int n_planes_pad;
  int proj_stride;         // floats per descriptor row of ImgDev::proj (n_planes rounded up to 4)
  int bucket_pad;          // buckets padded to a multiple of this (kBucketPad)
  // tensor-core K2 (kernels.cu project_tc_kernel), null when n_planes > 192:
  const signed char* tc_b; // [3 digits][tc_npad planes][128 B], K-major 128-byte-swizzle image
  const int* tc_fexp;      // [tc_npad] per-plane exponent f (2^(f-1) <= max|p| < 2^f)
  int tc_npad;             // planes rounded up to 16
  int tc_pass0;            // planes in the first MMA pass (<= 96); the rest in the second
};

// An ambiguous projection whose sign the FP32 pass could not certify; the
// fixup kernel recomputes it in the reference's FP64 order.
struct Fixup {
  uint32_t img, desc, plane, pad;
};

// One CTA of the match kernel: a query range of one image pair.
struct PairWork {
  uint32_t q_img, t_img;  // row-slot indices into the ImgDev table
  uint32_t q_begin, q_end;
  uint32_t pair;          // index of the pair within the launch
  uint32_t pad[3];
};

struct MatchLaunch {
  const ImgDev* imgs;
  const PairWork* work;
  const uint64_t* dense_off;   // [n_pairs] offset of each pair's dense result array
  int32_t* dense;              // train idx or -1 per query
  uint32_t* pair_count;        // [n_pairs] number of matches per pair
  unsigned long long* exact_queries;  // diagnostics: queries that took the FP64 path
  int tables, n_buckets, k, idx_bits;
  double ratio;
  uint32_t test_flags;  // BMG_TEST_* (bmg_set_test_flags): force the rare exact paths
};
constexpr uint32_t kTestForceExactWalk = 1u;   // BMG_TEST_FORCE_EXACT_WALK
constexpr uint32_t kTestForceFp64Rerank = 2u;  // BMG_TEST_FORCE_FP64_RERANK

// Device state of the exact parallel row mean (kernels.cu K1).
struct MeanState {
  uint32_t bad;         // a descriptor value outside the F96 range
  uint32_t need_chain;  // gate of the sequential fallback
  uint32_t rounds;      // max over channels of walked tiles + 1
  uint32_t events;      // rounding steps replayed (all channels)
};

// Small device-side copies / zero fills on a compute stream (kernels.cu
// meta_kernel); src == nullptr means zero fill.  src may be mapped pinned
// host memory.  dst and src 16-byte aligned.
struct MetaOp {
  void* dst;
  const void* src;
  size_t bytes;
};
constexpr int kMetaOps = 8;
struct MetaBatch {
  MetaOp op[kMetaOps];
  int n;
};
void launch_meta(const MetaBatch& b, cudaStream_t s);

// Buckets are padded to whole 8-entry chunks (the candidate walk's unit), so
// every chunk a query walks is full and a lane's entry needs no bounds test.
constexpr int kBucketPad = 8;
constexpr uint32_t kSentinel = 8;  // all-pad chunk at the end of each table
// per-table slot capacity with every bucket padded to a multiple of `pad`,
// plus the sentinel chunk
inline uint32_t slot_stride(uint64_t n, int n_buckets, int pad) {
  return static_cast<uint32_t>(((n + (pad - 1ull) * static_cast<uint64_t>(n_buckets) + 7ull) & ~7ull) + kSentinel);
}

// ---- launchers (kernels.cu) ----
// Row mean into mean_out (and the FP64 accumulators into acc_out): the exact
// parallel reconstruction with the sequential chain as gated fallback, or the
// chain alone.  scratch: mean_scratch_bytes(n_tiles); *st must be zeroed by
// the caller (stream-ordered).  Returns kernel launches.
inline size_t mean_scratch_bytes(size_t n_tiles) {
  return n_tiles * kDim * 16;  // exclusive prefix of the F96 tile sums
}
// bytes of an image's tile statistics (ImgDev::tsum / trng / tlow)
inline size_t tile_stats_bytes(uint64_t n) {
  return ((n + kDim - 1) / kDim) * kDim * (16 + 32 + 4);
}
// `sums_resident`: every image's tile statistics were computed with its
// projections, so only the resolve runs; otherwise mean_sums computes them
int launch_row_mean(const ImgDev* imgs, int n_imgs, const uint32_t* tile_img,
                    const uint32_t* tile_start, int n_tiles, unsigned long long total, void* scratch,
                    MeanState* st, float* mean_out, double* acc_out, bool chain_only, bool sums_resident,
                    cudaStream_t s);
// whether launch_project writes the tile statistics (the tensor-core K2)
bool project_writes_tile_stats(const HashDev& h);
// fl32 projections + norms of one image (tile t = descriptors [128t, 128t+128))
// or of a tile list (ImgDev::proj / dnorm are the outputs)
void launch_project(const HashDev& h, const ImgDev& one, cudaStream_t s);
void launch_project_tiles(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                          const uint32_t* tile_start, int n_tiles, cudaStream_t s);
inline size_t proj_bytes(uint64_t n, int proj_stride) { return n * (sizeof(float) * proj_stride + sizeof(float)); }
// mproj: scratch of n_planes + 1 floats (m . p per plane, ||m||)
void launch_codes(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                  const uint32_t* tile_start, int n_tiles, const float* mean, float* mproj, Fixup* fix,
                  uint32_t* fix_count, uint32_t fix_cap, cudaStream_t s);
void launch_codes_fixup(const HashDev& h, const ImgDev* imgs_dev, int n_imgs, const float* mean,
                        const Fixup* fix, const uint32_t* fix_count, uint32_t fix_cap,
                        unsigned long long* fixed_bits, cudaStream_t s);
int launch_tables(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                  const uint32_t* tile_start, int n_tiles, int n_imgs, cudaStream_t s);  // returns launches
void launch_match(const MatchLaunch& a, int fwp, int n_work, cudaStream_t s);

void launch_scan_counts(const uint32_t* counts, int n, uint64_t* ranges_out, uint64_t base, cudaStream_t s);
void launch_compact(const int32_t* dense, const uint64_t* dense_off, const uint32_t* nq,
                    const uint64_t* out_off, int n_pairs, int32_t* out, cudaStream_t s);

constexpr int kCodesTile = 128;   // descriptors per codes CTA
constexpr int kPlaneChunk = 180;  // planes per codes CTA: 15 warps x 12 (grid.y covers the rest)
#ifndef BMG_MATCH_THREADS
#define BMG_MATCH_THREADS 1024
#endif
constexpr int kMatchThreads = BMG_MATCH_THREADS;  // one query per warp at a time
#ifndef BMG_MATCH_QUERIES
#define BMG_MATCH_QUERIES 2048
#endif
constexpr int kMatchQueries = BMG_MATCH_QUERIES;  // queries per match CTA
// queries per CTA of the match kernel launch_match picks for (fwp, k)
int match_queries_per_cta(int fwp, int k);
int device_sm_count();

// ---- VLAD encoding (vlad.cu; retrieval.cpp:160-205) ----
struct VladImg {
  const float* desc;    // [n][128] in the batch buffer
  uint32_t n, pad_;
  uint64_t assign_off;  // offset of the image's descriptors in VladBatch::assign
};
struct VladBatch {
  const VladImg* imgs;
  const uint32_t* tile_img;    // per 128-descriptor tile: image, first descriptor
  const uint32_t* tile_start;
  const float* centroids;      // [k_words][128] (Codebook::centroids)
  int k_words;
  int32_t* assign;             // nearest centroid per descriptor
  uint2* fix;                  // (image, descriptor) the FP32 filter could not certify
  uint32_t* fix_count;         // zeroed before the launch
  uint32_t fix_cap;
  uint32_t* members;           // descriptors grouped by cluster, descriptor order (per image at assign_off)
  uint32_t* member_off;        // [images][k_words+1] cluster starts
  double* acc;                 // [images][k_words*128] residual sums
  float* values;               // [images][k_words*128] VladVector::values
  uint8_t* degenerate;         // [images] VladVector::degenerate
  // k-means assignment (train_codebook, retrieval.cpp:99-117): the centroids
  // are doubles (cent64; `centroids` holds them rounded to float for the FP32
  // filter, whose bound then adds cnorm_max * sqrt(s) terms), the FP64 loop
  // starts from centroid 0's distance, and point_d2 gets every point's FP64
  // distance to its centroid.  Null for encode_vlad.
  const double* cent64;
  float cnorm_max;             // max ||c||_2 over the centroids, rounded up
  double* point_d2;
};
constexpr int kVladTile = 128;
constexpr int kVladMaxWords = 1024;  // codebook words the GPU encoder supports
void launch_vlad(const VladBatch& b, int n_imgs, int n_tiles, cudaStream_t s);
// k-means: nearest centroid (+ FP64 fixups) and every point's FP64 distance;
// then the cluster sums (sort + residual chains with zero centroids: acc =
// sum of (double)d in point order) when `sums`
void launch_kmeans_assign(const VladBatch& b, int n_tiles, cudaStream_t s);
void launch_kmeans_sums(const VladBatch& b, cudaStream_t s);
// certified / FP64 assignments of the last launches (diagnostics)
size_t vlad_assign_smem_bytes();

}  // namespace bmg
