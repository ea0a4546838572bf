// host_random.cpp -- host-side generation the reference performs on the CPU:
// seed splitting (common.hpp:29-45) and the LSH hyperplanes
// (make_hash_functions, hashmatch.cpp:53-69).  The planes are defined by
// libstdc++'s <random> (std::normal_distribution<float> over std::mt19937_64),
// so they are generated here with the same standard library and uploaded once
// per context; they are never regenerated on the device (SURVEY §7 hard part 7).
#include <cstdint>
#include <random>
#include <string_view>

#include "../../include/bandmatch_gpu.h"

namespace bmg {

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t seed_for(uint64_t root, std::string_view stage) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (char c : stage) {
    h ^= static_cast<unsigned char>(c);
    h *= 0x100000001b3ULL;
  }
  return splitmix64(root ^ splitmix64(h));
}

bool valid_hash_params(const bmg_hash_params& p) {
  return p.tables >= 1 && p.coarse_bits >= 1 && p.coarse_bits <= 32 && p.fine_bits >= 1;
}

void make_planes(uint64_t seed, const bmg_hash_params& p, float* coarse, float* fine) {
  // A single distribution object serves both engines: a cached polar-method
  // value carries over from the coarse stream to the fine stream.
  std::normal_distribution<float> gauss(0.0f, 1.0f);
  std::mt19937_64 rng_coarse(seed_for(seed, "hash.coarse"));
  const size_t nc = static_cast<size_t>(p.tables) * p.coarse_bits * BMG_DIM;
  for (size_t i = 0; i < nc; ++i) coarse[i] = gauss(rng_coarse);
  std::mt19937_64 rng_fine(seed_for(seed, "hash.fine"));
  const size_t nf = static_cast<size_t>(p.fine_bits) * BMG_DIM;
  for (size_t i = 0; i < nf; ++i) fine[i] = gauss(rng_fine);
}

}  // namespace bmg
