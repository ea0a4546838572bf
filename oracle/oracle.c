/*
 * oracle.c -- CPU restatement of the cascade-hashing hot path (TEST
 * INFRASTRUCTURE ONLY; see oracle.h).  Citations are file:line relative to
 * /root/reference/proj.  Compile with -ffp-contract=off.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- common.hpp:29-45 ------------------------------------------------- */

uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_seed_for(uint64_t root, const char* stage) {
  uint64_t h = 0xcbf29ce484222325ULL; /* FNV-1a over the tag */
  for (const unsigned char* c = (const unsigned char*)stage; *c; ++c) {
    h ^= *c;
    h *= 0x100000001b3ULL;
  }
  return orc_splitmix64(root ^ orc_splitmix64(h));
}

/* ---- std::mt19937_64 (ISO C++ [rand.eng.mers], libstdc++ 13) ------------ */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & upper) | (s->mt[(i + 1) % 312] & lower);
      s->mt[i] = s->mt[(i + 156) % 312] ^ (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* generate_canonical<float, 24>(mt19937_64): one engine call
 * (random.tcc:3349-3381): sum = float(u) * 1, tmp = float(2^64), ret = sum/tmp. */
static float canonical_f(mt64* s) {
  const float sum = (float)mt64_next(s) * 1.0f;
  const float tmp = (float)(1.0L * 18446744073709551616.0L);
  float ret = sum / tmp;
  if (ret >= 1.0f) ret = nextafterf(1.0f, 0.0f);
  return ret;
}

/* normal_distribution<float>::operator() -- random.tcc:1811-1844 (polar). */
typedef struct {
  int saved_available;
  float saved;
} normal_f;

static float normal_f_next(normal_f* nd, mt64* s) {
  float ret;
  if (nd->saved_available) {
    nd->saved_available = 0;
    ret = nd->saved;
  } else {
    float x, y, r2;
    do {
      x = (float)((double)(2.0f * canonical_f(s)) - 1.0);
      y = (float)((double)(2.0f * canonical_f(s)) - 1.0);
      r2 = x * x + y * y;
    } while ((double)r2 > 1.0 || (double)r2 == 0.0);
    const float mult = sqrtf(-2.0f * logf(r2) / r2);
    nd->saved = x * mult;
    nd->saved_available = 1;
    ret = y * mult;
  }
  return ret * 1.0f + 0.0f; /* stddev 1, mean 0 */
}

/* ---- hashmatch.cpp:20-25 ------------------------------------------------ */

static int check_params(const orc_hash_params* p) {
  if (p->tables < 1) return ORC_INVALID_ARGUMENT;
  if (p->coarse_bits < 1 || p->coarse_bits > 32) return ORC_INVALID_ARGUMENT;
  if (p->fine_bits < 1) return ORC_INVALID_ARGUMENT;
  return ORC_OK;
}

/* ---- hashmatch.cpp:53-69 ------------------------------------------------ */

int orc_make_hash_functions(uint64_t seed, const orc_hash_params* p, float* coarse_out,
                            float* fine_out) {
  if (check_params(p) != ORC_OK) return ORC_INVALID_ARGUMENT;
  /* one distribution object shared by both engines (hashmatch.cpp:59), so a
   * saved polar value can carry from the coarse stream into the fine one */
  normal_f gauss = {0, 0.0f};
  mt64* rng = (mt64*)malloc(sizeof(mt64));
  if (!rng) return ORC_OUT_OF_MEMORY;
  mt64_seed(rng, orc_seed_for(seed, "hash.coarse"));
  const size_t nc = (size_t)p->tables * (size_t)p->coarse_bits * ORC_DIM;
  for (size_t i = 0; i < nc; ++i) coarse_out[i] = normal_f_next(&gauss, rng);
  mt64_seed(rng, orc_seed_for(seed, "hash.fine"));
  const size_t nf = (size_t)p->fine_bits * ORC_DIM;
  for (size_t i = 0; i < nf; ++i) fine_out[i] = normal_f_next(&gauss, rng);
  free(rng);
  return ORC_OK;
}

/* ---- engine.cpp:446-461 ------------------------------------------------- */

void orc_row_mean(const float* const* descs, const uint64_t* counts, size_t n_images,
                  float mean_out[ORC_DIM]) {
  double acc[ORC_DIM];
  uint64_t total = 0;
  for (int c = 0; c < ORC_DIM; ++c) acc[c] = 0.0;
  for (size_t im = 0; im < n_images; ++im) {
    const float* d = descs[im];
    for (uint64_t i = 0; i < counts[im]; ++i)
      for (int c = 0; c < ORC_DIM; ++c) acc[c] += (double)d[i * ORC_DIM + c];
    total += counts[im];
  }
  for (int c = 0; c < ORC_DIM; ++c)
    mean_out[c] = total > 0 ? (float)(acc[c] / (double)total) : 0.0f;
}

/* ---- hashmatch.cpp:27-33 ------------------------------------------------ */

double orc_centered_dot(const float* d, const float* mean, const float* plane) {
  double s = 0.0;
  for (int c = 0; c < ORC_DIM; ++c) s += ((double)d[c] - (double)mean[c]) * (double)plane[c];
  return s;
}

/* ---- hashmatch.cpp:35-42 ------------------------------------------------ */

double orc_euclidean(const float* a, const float* b) {
  double s = 0.0;
  for (int c = 0; c < ORC_DIM; ++c) {
    const double d = (double)a[c] - (double)b[c];
    s += d * d;
  }
  return sqrt(s);
}

/* ---- hashmatch.cpp:71-100 ----------------------------------------------- */

int orc_compute_codes(const float* desc, uint64_t n, const orc_hash_params* p,
                      const float* coarse_planes, const float* fine_planes,
                      const float mean[ORC_DIM], uint32_t* coarse_out, uint64_t* fine_out) {
  if (check_params(p) != ORC_OK) return ORC_INVALID_ARGUMENT;
  const int fw = (p->fine_bits + 63) / 64;
  memset(coarse_out, 0, (size_t)n * (size_t)p->tables * sizeof(uint32_t));
  memset(fine_out, 0, (size_t)n * (size_t)fw * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) {
    const float* d = desc + i * ORC_DIM;
    for (int t = 0; t < p->tables; ++t) {
      uint32_t bucket = 0;
      for (int b = 0; b < p->coarse_bits; ++b) {
        const float* plane = coarse_planes + ((size_t)t * p->coarse_bits + b) * ORC_DIM;
        if (orc_centered_dot(d, mean, plane) > 0.0) bucket |= 1u << b;
      }
      coarse_out[i * p->tables + t] = bucket;
    }
    uint64_t* fine = fine_out + i * fw;
    for (int b = 0; b < p->fine_bits; ++b) {
      if (orc_centered_dot(d, mean, fine_planes + (size_t)b * ORC_DIM) > 0.0)
        fine[b / 64] |= 1ULL << (b % 64);
    }
  }
  return ORC_OK;
}

/* ---- hashmatch.cpp:102-211 ---------------------------------------------- */

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct {
  int train_idx;
  int hamming;
  double euclidean;
} cand_t;

int orc_match_pair(const float* qdesc, uint64_t nq, const uint32_t* qcoarse,
                   const uint64_t* qfine, const float* tdesc, uint64_t nt,
                   const uint32_t* tcoarse, const uint64_t* tfine, const orc_hash_params* p,
                   int32_t k_nearest, double ratio, int32_t* out_pairs, uint64_t* out_count,
                   uint32_t* cand_count, uint64_t* topk) {
  *out_count = 0;
  if (check_params(p) != ORC_OK) return ORC_HASH_MISMATCH;
  if (k_nearest < 1) return ORC_INVALID_ARGUMENT; /* :113 */
  if (cand_count)
    for (uint64_t q = 0; q < nq; ++q) cand_count[q] = 0;
  if (topk)
    for (uint64_t i = 0; i < nq * (uint64_t)k_nearest; ++i) topk[i] = UINT64_MAX;
  if (nq == 0 || nt == 0) return ORC_OK; /* :118 */

  const int tables = p->tables;
  const size_t n_buckets = (size_t)1 << p->coarse_bits;
  const int fw = (p->fine_bits + 63) / 64;
  const int max_ham = p->fine_bits;

  /* bucket index over train features (:125-145) */
  uint32_t* offsets = (uint32_t*)calloc((size_t)tables * (n_buckets + 1), sizeof(uint32_t));
  uint32_t* slots = (uint32_t*)malloc((size_t)tables * nt * sizeof(uint32_t));
  uint32_t* cursor = (uint32_t*)malloc((size_t)tables * (n_buckets + 1) * sizeof(uint32_t));
  int* last_seen = (int*)malloc(nt * sizeof(int));
  uint32_t* candidates = (uint32_t*)malloc(((size_t)tables * nt + 1) * sizeof(uint32_t));
  int* ham = (int*)malloc(((size_t)tables * nt + 1) * sizeof(int));
  int* by_distance = (int*)malloc(((size_t)tables * nt + 1) * sizeof(int));
  uint32_t* dist_start = (uint32_t*)malloc((size_t)(max_ham + 2) * sizeof(uint32_t));
  uint32_t* dcursor = (uint32_t*)malloc((size_t)(max_ham + 2) * sizeof(uint32_t));
  cand_t* top = (cand_t*)malloc((size_t)k_nearest * sizeof(cand_t));
  if (!offsets || !slots || !cursor || !last_seen || !candidates || !ham || !by_distance ||
      !dist_start || !dcursor || !top) {
    free(offsets); free(slots); free(cursor); free(last_seen); free(candidates); free(ham);
    free(by_distance); free(dist_start); free(dcursor); free(top);
    return ORC_OUT_OF_MEMORY;
  }
  for (uint64_t j = 0; j < nt; ++j)
    for (int t = 0; t < tables; ++t) ++offsets[t * (n_buckets + 1) + tcoarse[j * tables + t] + 1];
  for (int t = 0; t < tables; ++t) {
    uint32_t* row = offsets + (size_t)t * (n_buckets + 1);
    for (size_t b = 0; b < n_buckets; ++b) row[b + 1] += row[b];
  }
  memcpy(cursor, offsets, (size_t)tables * (n_buckets + 1) * sizeof(uint32_t));
  for (uint64_t j = 0; j < nt; ++j)
    for (int t = 0; t < tables; ++t) {
      uint32_t* c = &cursor[t * (n_buckets + 1) + tcoarse[j * tables + t]];
      slots[(size_t)t * nt + (*c)++] = (uint32_t)j;
    }
  for (uint64_t j = 0; j < nt; ++j) last_seen[j] = -1;

  uint64_t n_out = 0;
  for (uint64_t qi = 0; qi < nq; ++qi) {
    /* candidate union (:154-169) */
    size_t nc = 0;
    for (int t = 0; t < tables; ++t) {
      const uint32_t* row = offsets + (size_t)t * (n_buckets + 1);
      const uint32_t bucket = qcoarse[qi * tables + t];
      const uint32_t* slot_row = slots + (size_t)t * nt;
      for (uint32_t s = row[bucket]; s < row[bucket + 1]; ++s) {
        const uint32_t j = slot_row[s];
        if (last_seen[j] != (int)qi) {
          last_seen[j] = (int)qi;
          candidates[nc++] = j;
        }
      }
    }
    if (cand_count) cand_count[qi] = (uint32_t)nc;
    if (nc == 0) continue;
    qsort(candidates, nc, sizeof(uint32_t), cmp_u32); /* std::sort ascending (:169) */
    /* Hamming + stable counting sort by distance (:171-190) */
    memset(dist_start, 0, (size_t)(max_ham + 2) * sizeof(uint32_t));
    const uint64_t* qcode = qfine + qi * fw;
    for (size_t c = 0; c < nc; ++c) {
      const uint64_t* tcode = tfine + (size_t)candidates[c] * fw;
      int h = 0;
      for (int w = 0; w < fw; ++w) h += __builtin_popcountll(qcode[w] ^ tcode[w]);
      ham[c] = h;
      ++dist_start[h + 1];
    }
    for (int h = 0; h <= max_ham; ++h) dist_start[h + 1] += dist_start[h];
    memcpy(dcursor, dist_start, (size_t)(max_ham + 2) * sizeof(uint32_t));
    for (size_t c = 0; c < nc; ++c) by_distance[dcursor[ham[c]]++] = (int)c;

    /* top-K, Euclidean re-rank, sort by (euclid, train_idx) (:192-204) */
    const size_t keep = nc < (size_t)k_nearest ? nc : (size_t)k_nearest;
    for (size_t r = 0; r < keep; ++r) {
      const int c = by_distance[r];
      const int tj = (int)candidates[c];
      top[r].train_idx = tj;
      top[r].hamming = ham[c];
      top[r].euclidean = orc_euclidean(qdesc + qi * ORC_DIM, tdesc + (size_t)tj * ORC_DIM);
      if (topk) topk[qi * (uint64_t)k_nearest + r] = ((uint64_t)ham[c] << 32) | (uint32_t)tj;
    }
    for (size_t a = 1; a < keep; ++a) {
      const cand_t v = top[a];
      size_t b = a;
      while (b > 0 && (top[b - 1].euclidean > v.euclidean ||
                       (top[b - 1].euclidean == v.euclidean && top[b - 1].train_idx > v.train_idx))) {
        top[b] = top[b - 1];
        --b;
      }
      top[b] = v;
    }
    /* ratio_accept (:47-49, :206-208) */
    const int lone = keep == 1;
    const double d1 = top[0].euclidean, d2 = lone ? 0.0 : top[1].euclidean;
    if (lone || d1 < d2 * ratio) {
      out_pairs[2 * n_out] = (int32_t)qi;
      out_pairs[2 * n_out + 1] = top[0].train_idx;
      ++n_out;
    }
  }
  *out_count = n_out;
  free(offsets); free(slots); free(cursor); free(last_seen); free(candidates); free(ham);
  free(by_distance); free(dist_start); free(dcursor); free(top);
  return ORC_OK;
}

/* ---- hashmatch.cpp:213-239 ---------------------------------------------- */

int orc_brute_force_match(const float* qdesc, uint64_t nq, const float* tdesc, uint64_t nt,
                          double ratio, int32_t* out_pairs, uint64_t* out_count) {
  *out_count = 0;
  if (nq == 0 || nt == 0) return ORC_OK;
  uint64_t n_out = 0;
  for (uint64_t qi = 0; qi < nq; ++qi) {
    int best = -1, second = -1;
    double best_d = 0.0, second_d = 0.0;
    for (uint64_t tj = 0; tj < nt; ++tj) {
      const double d = orc_euclidean(qdesc + qi * ORC_DIM, tdesc + tj * ORC_DIM);
      if (best < 0 || d < best_d) {
        second = best;
        second_d = best_d;
        best = (int)tj;
        best_d = d;
      } else if (second < 0 || d < second_d) {
        second = (int)tj;
        second_d = d;
      }
    }
    const int lone = second < 0;
    if (lone || best_d < second_d * ratio) {
      out_pairs[2 * n_out] = (int32_t)qi;
      out_pairs[2 * n_out + 1] = best;
      ++n_out;
    }
  }
  *out_count = n_out;
  return ORC_OK;
}

/* encode_vlad -- retrieval.cpp:160-205.  Nearest centroid by the sequential
 * FP64 squared distance with strict < from +inf (:170-183), residuals summed
 * in FP64 in descriptor order (:184-187), signed square root and sequential
 * norm (:189-195), degenerate on an empty image or norm2 <= 0 (:165-168,
 * :196-199), then float(acc * (1/sqrt(norm2))) (:200-202). */
int orc_encode_vlad(const float* centroids, int k_words, const float* desc, uint64_t n,
                    float* values_out, uint8_t* degenerate_out) {
  if (k_words < 1) return ORC_INVALID_ARGUMENT;
  const size_t dim = (size_t)k_words * ORC_DIM;
  for (size_t i = 0; i < dim; ++i) values_out[i] = 0.0f;
  *degenerate_out = 0;
  if (n == 0) {
    *degenerate_out = 1;
    return ORC_OK;
  }
  double* acc = (double*)calloc(dim, sizeof(double));
  if (!acc) return ORC_INVALID_ARGUMENT;
  for (uint64_t i = 0; i < n; ++i) {
    const float* d = desc + i * ORC_DIM;
    int best = 0;
    double best_d2 = INFINITY;
    for (int k = 0; k < k_words; ++k) {
      const float* c = centroids + (size_t)k * ORC_DIM;
      double s = 0.0;
      for (int j = 0; j < ORC_DIM; ++j) {
        const double diff = (double)d[j] - (double)c[j];
        s += diff * diff;
      }
      if (s < best_d2) {
        best_d2 = s;
        best = k;
      }
    }
    double* slot = acc + (size_t)best * ORC_DIM;
    const float* c = centroids + (size_t)best * ORC_DIM;
    for (int j = 0; j < ORC_DIM; ++j) slot[j] += (double)d[j] - (double)c[j];
  }
  double norm2 = 0.0;
  for (size_t i = 0; i < dim; ++i) {
    double v = acc[i];
    v = v >= 0.0 ? sqrt(v) : -sqrt(-v);
    acc[i] = v;
    norm2 += v * v;
  }
  if (norm2 <= 0.0) {
    *degenerate_out = 1;
    free(acc);
    return ORC_OK;
  }
  const double inv = 1.0 / sqrt(norm2);
  for (size_t i = 0; i < dim; ++i) values_out[i] = (float)(acc[i] * inv);
  free(acc);
  return ORC_OK;
}
