// host_synthetic.cpp -- the feature-input surface of the reference on the
// host: normalize (features.cpp:57-66) and the band-overlap synthetic scene
// (generate_synthetic, features.cpp:68-197, SyntheticScene features.hpp:56-64).
// Scenes are defined by libstdc++ <random>, so they are produced here on the
// CPU (bit-identical to the reference, pinned by tests/test_host.py) and then
// staged to HBM by the arena like any real feature set.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <random>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/bandmatch_gpu.h"

#include "../../include/bandmatch_gpu.h"

namespace bmg {

uint64_t seed_for(uint64_t root, std::string_view stage);
void set_last_error(const std::string& msg);

namespace {

constexpr int kD = BMG_DIM;
using Vec = std::array<float, kD>;

float wrap_angle(double a) {
  constexpr double two_pi = 2.0 * std::numbers::pi;
  a = std::fmod(a, two_pi);
  if (a < 0.0) a += two_pi;
  if (a >= two_pi) a = 0.0;
  return static_cast<float>(a);
}

// unit L2 norm with a double accumulator; false on an all-zero input
bool normalize_into(const Vec& raw, float* out) {
  double s = 0.0;
  for (float c : raw) s += static_cast<double>(c) * c;
  if (s == 0.0) return false;
  const double inv = 1.0 / std::sqrt(s);
  for (int i = 0; i < kD; ++i) out[i] = static_cast<float>(raw[i] * inv);
  return true;
}

Vec gaussian_vector(std::mt19937_64& rng, double sigma) {
  std::normal_distribution<double> g(0.0, sigma);  // fresh per vector
  Vec v{};
  for (float& c : v) c = static_cast<float>(g(rng));
  return v;
}

void random_unit(std::mt19937_64& rng, float* out) {
  for (;;) {
    const Vec raw = gaussian_vector(rng, 1.0);
    double s = 0.0;
    for (float c : raw) s += static_cast<double>(c) * c;
    if (s > 1e-12) {
      normalize_into(raw, out);
      return;
    }
  }
}

struct Scene {
  int n, ppi, band;
  double sigma, of;
  uint64_t seed;
  int ppa, opi;
};

int check_scene(const Scene& s) {
  const char* bad = nullptr;
  if (s.n < 1) bad = "n_images must be at least 1";
  else if (s.band < 0 || s.band >= s.n) bad = "overlap_band must satisfy 0 <= overlap_band < n_images";
  else if (s.ppi < 0) bad = "points_per_image must be non-negative";
  else if (!(s.of >= 0.0 && s.of <= 1.0)) bad = "outlier_fraction must lie in [0,1]";
  else if (!(s.sigma >= 0.0)) bad = "noise_sigma must be non-negative";
  if (bad) {
    set_last_error(std::string("InvalidScene: ") + bad);
    return BMG_INVALID_SCENE;
  }
  return BMG_OK;
}

Scene make_scene(int n, int ppi, int band, double sigma, double of, uint64_t seed) {
  Scene s{n, ppi, band, sigma, of, seed, 0, 0};
  if (ppi > 0 && band >= 0) {
    const double budget = ppi * (1.0 - of);
    s.ppa = std::max(1, static_cast<int>(std::llround(budget / (band + 1))));
  }
  s.opi = static_cast<int>(std::llround(ppi * of));
  return s;
}

}  // namespace
}  // namespace bmg

using namespace bmg;

extern "C" {

int bmg_synthetic_counts(int n_images, int ppi, int band, double sigma, double outlier_fraction,
                         uint64_t* counts_out) {
  const Scene s = make_scene(n_images, ppi, band, sigma, outlier_fraction, 0);
  if (const int rc = check_scene(s)) return rc;
  for (int i = 0; i < s.n; ++i)
    counts_out[i] = static_cast<uint64_t>(std::min(i, s.band) + 1) * s.ppa + s.opi;
  return BMG_OK;
}

int bmg_generate_synthetic(int n_images, int ppi, int band, double sigma, double outlier_fraction,
                           uint64_t seed, float* desc_out, float* keypoints_out) {
  return bmg_generate_synthetic_subset(n_images, ppi, band, sigma, outlier_fraction, seed, nullptr,
                                       desc_out, keypoints_out);
}

// The same scene, storing only the images with keep[i] != 0 (back to back,
// in image order).  Every image's random draws are still made -- the
// observation stream is shared by all images (features.cpp:131-171) -- but
// generation stops after the last kept image.
int bmg_generate_synthetic_subset(int n_images, int ppi, int band, double sigma,
                                  double outlier_fraction, uint64_t seed, const uint8_t* keep,
                                  float* desc_out, float* keypoints_out) {
  const Scene s = make_scene(n_images, ppi, band, sigma, outlier_fraction, seed);
  if (const int rc = check_scene(s)) return rc;
  struct World {
    double x, y, scale, orientation;
    float center[kD];
  };
  std::mt19937_64 rng_world(seed_for(seed, "scene.world"));
  std::uniform_real_distribution<double> upos(0.0, 1000.0), uscale(1.0, 4.0),
      uangle(0.0, 2.0 * std::numbers::pi);
  std::vector<World> world(static_cast<size_t>(s.n) * s.ppa);
  for (World& w : world) {
    w.x = upos(rng_world);
    w.y = upos(rng_world);
    w.scale = uscale(rng_world);
    w.orientation = uangle(rng_world);
    random_unit(rng_world, w.center);
  }
  struct Pose {
    double theta, sc, tx, ty, c, sn;
  };
  std::mt19937_64 rng_pose(seed_for(seed, "scene.poses"));
  std::uniform_real_distribution<double> uscale_img(0.8, 1.25), ushift(-100.0, 100.0);
  std::vector<Pose> poses(s.n);
  for (Pose& p : poses) {
    p.theta = uangle(rng_pose);
    p.sc = uscale_img(rng_pose);
    p.tx = ushift(rng_pose);
    p.ty = ushift(rng_pose);
    p.c = std::cos(p.theta);
    p.sn = std::sin(p.theta);
  }
  std::mt19937_64 rng_obs(seed_for(seed, "scene.observations"));
  int last = s.n - 1;
  if (keep) {
    last = -1;
    for (int i = 0; i < s.n; ++i)
      if (keep[i]) last = i;
  }
  float scratch_desc[kD], scratch_kp[4];
  size_t k = 0;
  for (int i = 0; i <= last; ++i) {
    const Pose& p = poses[i];
    const bool store = !keep || keep[i];
    for (int a = std::max(0, i - s.band); a <= i; ++a) {
      for (int q = 0; q < s.ppa; ++q) {
        const World& w = world[static_cast<size_t>(a) * s.ppa + q];
        float* kp = keypoints_out ? (store ? keypoints_out + 4 * k : scratch_kp) : nullptr;
        if (kp) {
          kp[0] = static_cast<float>(p.sc * (p.c * w.x - p.sn * w.y) + p.tx);
          kp[1] = static_cast<float>(p.sc * (p.sn * w.x + p.c * w.y) + p.ty);
          kp[2] = static_cast<float>(w.scale * p.sc);
          kp[3] = wrap_angle(w.orientation + p.theta);
        }
        Vec raw;
        std::memcpy(raw.data(), w.center, sizeof(raw));
        if (s.sigma > 0.0) {
          const Vec noise = gaussian_vector(rng_obs, s.sigma);
          for (int c = 0; c < kD; ++c) raw[c] += noise[c];
        }
        if (!normalize_into(raw, store ? desc_out + k * kD : scratch_desc)) {
          set_last_error("ZeroVector: cannot normalize an all-zero descriptor");
          return BMG_INVALID_SCENE;
        }
        k += store;
      }
    }
    for (int o = 0; o < s.opi; ++o) {
      const float x = static_cast<float>(upos(rng_obs));
      const float y = static_cast<float>(upos(rng_obs));
      const float sc = static_cast<float>(uscale(rng_obs));
      const float th = wrap_angle(uangle(rng_obs));
      float* kp = keypoints_out ? (store ? keypoints_out + 4 * k : scratch_kp) : nullptr;
      if (kp) {
        kp[0] = x;
        kp[1] = y;
        kp[2] = sc;
        kp[3] = th;
      }
      random_unit(rng_obs, store ? desc_out + k * kD : scratch_desc);
      k += store;
    }
  }
  return BMG_OK;
}

}  // extern "C"
