/*
 * oracle.h -- CPU restatement of the bandmatch cascade-hashing hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2505_22089_b200/,
 * include/, the C-ABI library) links, loads or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may use it, and
 * only as the checker / the timed CPU baseline.
 *
 * Every function restates one reference function (file:line relative to
 * /root/reference/proj) in plain C99 with the same IEEE-754 operation order.
 * Build flags pin -ffp-contract=off so no multiply-add is ever fused, which is
 * what the reference's CMake Release build (x86-64 baseline ISA, no FMA)
 * produces.  Parity of this restatement with the compiled reference is pinned
 * by tests/test_oracle.py against oracle/_ref and tests/golden/.
 */
#ifndef BANDMATCH_ORACLE_H
#define BANDMATCH_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_DIM 128 /* kDescriptorDim, include/bandmatch/features.hpp:14 */

/* status codes mirror bandmatch::Error codes (common.hpp:13-26) */
enum {
  ORC_OK = 0,
  ORC_INVALID_ARGUMENT = 1,
  ORC_HASH_MISMATCH = 2,
  ORC_OUT_OF_MEMORY = 3
};

typedef struct {
  int32_t tables;      /* HashParams::tables      hashmatch.hpp:12 */
  int32_t coarse_bits; /* HashParams::coarse_bits hashmatch.hpp:13 */
  int32_t fine_bits;   /* HashParams::fine_bits   hashmatch.hpp:14 */
} orc_hash_params;

/* seed_for / splitmix64 -- common.hpp:29-45 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_seed_for(uint64_t root, const char* stage);

/* make_hash_functions -- hashmatch.cpp:53-69.  Restates libstdc++ 13's
 * std::mt19937_64, generate_canonical<float,24> (random.tcc:3349-3381) and the
 * Marsaglia polar normal_distribution<float> (random.tcc:1811-1844).
 * coarse_out: tables*coarse_bits*128 floats; fine_out: fine_bits*128 floats. */
int orc_make_hash_functions(uint64_t seed, const orc_hash_params* p, float* coarse_out,
                            float* fine_out);

/* Row centering mean -- engine.cpp:446-461.  images in ascending id order,
 * descriptors in index order, double accumulation, float(acc/total). */
void orc_row_mean(const float* const* descs, const uint64_t* counts, size_t n_images,
                  float mean_out[ORC_DIM]);

/* compute_codes -- hashmatch.cpp:71-100 with centered_dot :27-33.
 * coarse_out: n*tables u32, fine_out: n*ceil(fine_bits/64) u64. */
int orc_compute_codes(const float* desc, uint64_t n, const orc_hash_params* p,
                      const float* coarse_planes, const float* fine_planes,
                      const float mean[ORC_DIM], uint32_t* coarse_out, uint64_t* fine_out);

/* One projection exactly as centered_dot (hashmatch.cpp:27-33). */
double orc_centered_dot(const float* d, const float* mean, const float* plane);

/* euclidean -- hashmatch.cpp:35-42 */
double orc_euclidean(const float* a, const float* b);

/* match_pair -- hashmatch.cpp:102-211.  Writes (query_idx, train_idx) int32
 * pairs to out_pairs (capacity >= 2*nq ints) in ascending query order and the
 * match count to *out_count.  Optional diagnostics (may be NULL):
 *   cand_count[nq]      size of the deduplicated candidate union (:147-169)
 *   topk[nq*k]          (hamming<<32 | train_idx) of the Hamming top-K (:171-200),
 *                       unused slots = UINT64_MAX. */
int orc_match_pair(const float* qdesc, uint64_t nq, const uint32_t* qcoarse,
                   const uint64_t* qfine, const float* tdesc, uint64_t nt,
                   const uint32_t* tcoarse, const uint64_t* tfine, const orc_hash_params* p,
                   int32_t k_nearest, double ratio, int32_t* out_pairs, uint64_t* out_count,
                   uint32_t* cand_count, uint64_t* topk);

/* brute_force_match -- hashmatch.cpp:213-239 */
int orc_brute_force_match(const float* qdesc, uint64_t nq, const float* tdesc, uint64_t nt,
                          double ratio, int32_t* out_pairs, uint64_t* out_count);

/* encode_vlad -- retrieval.cpp:160-205.  centroids
 * [k_words][128]; values_out[k_words*128]; returns ORC_INVALID_ARGUMENT for
 * k_words < 1 ("codebook has no words"). */
int orc_encode_vlad(const float* centroids, int k_words, const float* desc, uint64_t n,
                    float* values_out, uint8_t* degenerate_out);

#ifdef __cplusplus
}
#endif

#endif
