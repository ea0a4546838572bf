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
  uint32_t* slots;     // [tables][n] train indices grouped by bucket (:136-145)
  uint32_t n;
  uint32_t overflow;   // set by the codes kernel when its fixup list overflowed
  // upload completion flag written by the copy stream after the image's H2D
  // (value = upload generation); the row-mean producer waits on it so the
  // mean chain overlaps the transfers.  nullptr = already resident.
  const uint32_t* ready;
  uint32_t ready_gen;
  uint32_t pad_;
  // channel-major FP64 copy [128][n] made once per upload (exact widening),
  // streamed by the row-mean chain; nullptr for non-arena images
  const double* dt;
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
  // when non-null, kernels return immediately unless *gate != 0 (the
  // re-do pass after a mean speculation miss; see bmg_api.cpp)
  const uint32_t* gate;
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
  const uint32_t* gate;        // see HashDev::gate
};

// ---- launchers (kernels.cu) ----
// float [n][128] -> double [128][n] (exact), for the row-mean chain
void launch_widen_transpose(const float* desc, uint32_t n, double* dt, cudaStream_t s);
void launch_row_mean(const ImgDev* imgs, int n_imgs, float* mean_out, double* acc_out,
                     cudaStream_t s);
void launch_codes(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                  const uint32_t* tile_start, int n_tiles, const float* mean, Fixup* fix,
                  uint32_t* fix_count, uint32_t fix_cap, cudaStream_t s);
void launch_codes_fixup(const HashDev& h, const ImgDev* imgs_dev, int n_imgs, const float* mean,
                        const Fixup* fix, const uint32_t* fix_count, uint32_t fix_cap,
                        unsigned long long* fixed_bits, cudaStream_t s);
void launch_tables(const HashDev& h, const ImgDev* imgs_dev, const uint32_t* tile_img,
                   const uint32_t* tile_start, int n_tiles, int n_imgs, cudaStream_t s);
void launch_match(const MatchLaunch& a, int fwp, int n_work, const ImgDev& any_train_max,
                  uint32_t max_train_n, cudaStream_t s, int* smem_used);
void launch_scan_counts(const uint32_t* counts, int n, uint64_t* offsets_out,
                        unsigned long long* running_total, const uint32_t* gate, cudaStream_t s);
void launch_compact(const int32_t* dense, const uint64_t* dense_off, const uint32_t* nq,
                    const uint64_t* out_off, int n_pairs, int32_t* out, const uint32_t* gate,
                    cudaStream_t s);
// speculative row mean: order-free FP64 sums per 128-descriptor tile, then a
// fixed-order reduction -> float(sum / total)
void launch_mean_fast(const ImgDev* imgs, const uint32_t* tile_img, const uint32_t* tile_start,
                      int n_tiles, double* partial, unsigned long long total, float* mean_out,
                      cudaStream_t s);
// *redo = any bit of the speculative mean differs from the exact one
void launch_mean_check(const float* fast, const float* exact, uint32_t* redo, cudaStream_t s);
void launch_gated_clear(void* p, size_t bytes, const uint32_t* gate, cudaStream_t s);

constexpr int kCodesTile = 128;   // descriptors per codes CTA
constexpr int kPlaneChunk = 192;  // planes per codes CTA (grid.y covers the rest)
constexpr int kMatchThreads = 1024;  // 32 warps, one query per warp at a time
constexpr int kMatchQueries = 1024;  // queries per match CTA

}  // namespace bmg
