// ref_shim.cpp -- extern "C" wrapper around the UNMODIFIED reference library
// (bandmatch, /root/reference/proj/src), compiled in place by oracle/Makefile
// into oracle/_ref/libbandmatch_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin the C restatement (oracle.c) and to
// generate tests/golden fixtures in this container, and as the timed CPU
// baseline ("kind": "reference") in bench.py.  Never linked by the product.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "bandmatch/engine.hpp"
#include "bandmatch/features.hpp"
#include "bandmatch/hashmatch.hpp"
#include "bandmatch/mbr.hpp"
#include "bandmatch/retrieval.hpp"
#include "bandmatch/verify.hpp"
#include "bandmatch/view_graph.hpp"

using namespace bandmatch;

namespace {

thread_local std::string g_last_error;

int status_of(const std::string& code) {
  if (code == "InvalidArgument") return 1;
  if (code == "HashMismatch") return 2;
  if (code == "CapacityExceeded") return 3;
  if (code == "NotResident") return 4;
  if (code == "FormatError") return 5;
  if (code == "BudgetTooSmall") return 6;
  if (code == "EmptyGraph") return 7;
  if (code == "TruncatedFile") return 8;
  if (code == "TooFewDescriptors") return 9;
  if (code == "EmptyInput") return 10;
  return 99;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return status_of(e.code());
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 98;
  }
}

HashFunctions hf_from(uint64_t seed, int tables, int cb, int fb, const float* coarse,
                      const float* fine) {
  HashFunctions hf;
  hf.params = {tables, cb, fb};
  hf.seed = seed;
  hf.coarse.assign(coarse, coarse + static_cast<size_t>(tables) * cb * kDescriptorDim);
  hf.fine.assign(fine, fine + static_cast<size_t>(fb) * kDescriptorDim);
  return hf;
}

FeatureSet fs_from(uint64_t id, const float* desc, uint64_t n) {
  FeatureSet fs;
  fs.image_id = id;
  fs.descriptors.resize(n);
  fs.keypoints.resize(n);
  if (n) std::memcpy(fs.descriptors.data(), desc, n * sizeof(Descriptor));
  return fs;
}

HashCodeSet cs_from(const FeatureSet& fs, uint64_t seed, int tables, int cb, int fb,
                    const uint32_t* coarse, const uint64_t* fine) {
  HashCodeSet cs;
  cs.image_id = fs.image_id;
  cs.function_seed = seed;
  cs.params = {tables, cb, fb};
  cs.count = fs.size();
  cs.fine_words = (fb + 63) / 64;
  cs.coarse.assign(coarse, coarse + cs.count * tables);
  cs.fine.assign(fine, fine + cs.count * cs.fine_words);
  return cs;
}

void put_matches(const PairMatches& pm, int32_t* out, uint64_t* count) {
  for (size_t i = 0; i < pm.matches.size(); ++i) {
    out[2 * i] = pm.matches[i].first;
    out[2 * i + 1] = pm.matches[i].second;
  }
  *count = pm.matches.size();
}

struct Synth {
  SyntheticDataset data;
};

struct FeatureTable {
  std::map<ImageId, FeatureSet> features;
};

struct Results {
  std::map<IdPair, PairMatches> r;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

uint64_t ref_seed_for(uint64_t root, const char* tag) { return seed_for(root, tag); }

int ref_make_hash_functions(uint64_t seed, int tables, int cb, int fb, float* coarse_out,
                            float* fine_out) {
  return guarded([&] {
    const HashFunctions hf = make_hash_functions(seed, {tables, cb, fb});
    std::copy(hf.coarse.begin(), hf.coarse.end(), coarse_out);
    std::copy(hf.fine.begin(), hf.fine.end(), fine_out);
  });
}

int ref_compute_codes(const float* desc, uint64_t n, uint64_t seed, int tables, int cb, int fb,
                      const float* coarse, const float* fine, const float* mean,
                      uint32_t* coarse_out, uint64_t* fine_out) {
  return guarded([&] {
    const HashFunctions hf = hf_from(seed, tables, cb, fb, coarse, fine);
    const FeatureSet fs = fs_from(0, desc, n);
    std::array<float, kDescriptorDim> m;
    std::copy(mean, mean + kDescriptorDim, m.begin());
    const HashCodeSet cs = compute_codes(fs, hf, m);
    std::copy(cs.coarse.begin(), cs.coarse.end(), coarse_out);
    std::copy(cs.fine.begin(), cs.fine.end(), fine_out);
  });
}

int ref_match_pair(const float* qdesc, uint64_t nq, const uint32_t* qcoarse,
                   const uint64_t* qfine, const float* tdesc, uint64_t nt,
                   const uint32_t* tcoarse, const uint64_t* tfine, uint64_t seed, int tables,
                   int cb, int fb, int k, double ratio, int32_t* out, uint64_t* count) {
  return guarded([&] {
    const FeatureSet qf = fs_from(1, qdesc, nq);
    const FeatureSet tf = fs_from(2, tdesc, nt);
    const HashCodeSet qc = cs_from(qf, seed, tables, cb, fb, qcoarse, qfine);
    const HashCodeSet tc = cs_from(tf, seed, tables, cb, fb, tcoarse, tfine);
    MatchParams mp;
    mp.k_nearest = k;
    mp.ratio = ratio;
    put_matches(match_pair(qf, qc, tf, tc, mp), out, count);
  });
}

int ref_brute_force_match(const float* qdesc, uint64_t nq, const float* tdesc, uint64_t nt,
                          double ratio, int32_t* out, uint64_t* count) {
  return guarded([&] {
    put_matches(brute_force_match(fs_from(1, qdesc, nq), fs_from(2, tdesc, nt), ratio), out,
                count);
  });
}

// ---- synthetic scenes (features.cpp:68-197) --------------------------------

void* ref_synth_create(int n_images, int ppi, int band, double sigma, double outlier_fraction,
                       uint64_t seed) {
  Synth* s = new Synth;
  const int rc = guarded([&] {
    SyntheticScene sc;
    sc.n_images = n_images;
    sc.points_per_image = ppi;
    sc.overlap_band = band;
    sc.noise_sigma = sigma;
    sc.outlier_fraction = outlier_fraction;
    sc.seed = seed;
    s->data = generate_synthetic(sc);
  });
  if (rc != 0) {
    delete s;
    return nullptr;
  }
  return s;
}
uint64_t ref_synth_count(void* h, int i) { return static_cast<Synth*>(h)->data.images.at(i).size(); }
void ref_synth_copy(void* h, int i, float* out) {
  const FeatureSet& fs = static_cast<Synth*>(h)->data.images.at(i);
  if (fs.size()) std::memcpy(out, fs.descriptors.data(), fs.size() * sizeof(Descriptor));
}
void ref_synth_copy_keypoints(void* h, int i, float* out) {
  const FeatureSet& fs = static_cast<Synth*>(h)->data.images.at(i);
  for (size_t k = 0; k < fs.size(); ++k) {
    out[4 * k] = fs.keypoints[k].x;
    out[4 * k + 1] = fs.keypoints[k].y;
    out[4 * k + 2] = fs.keypoints[k].scale;
    out[4 * k + 3] = fs.keypoints[k].orientation;
  }
}
uint64_t ref_synth_pair_count(void* h) { return static_cast<Synth*>(h)->data.true_pairs.size(); }
void ref_synth_pairs(void* h, uint64_t* out) {
  const auto& p = static_cast<Synth*>(h)->data.true_pairs;
  for (size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].a;
    out[2 * i + 1] = p[i].b;
  }
}
void ref_synth_free(void* h) { delete static_cast<Synth*>(h); }

// ---- block schedule (mbr.cpp:321-376, 378-419) -----------------------------

int ref_iterate_schedule_to_file(const uint64_t* ids, uint64_t n_ids, const uint64_t* pairs,
                                 uint64_t n_pairs, int size_blk, int size_gpu,
                                 const char* path) {
  return guarded([&] {
    std::vector<IdPair> ps;
    for (uint64_t i = 0; i < n_pairs; ++i) ps.emplace_back(pairs[2 * i], pairs[2 * i + 1]);
    const ViewGraph g = make_view_graph(std::vector<ImageId>(ids, ids + n_ids), ps);
    write_plan(path, iterate_schedule(g, size_blk, size_gpu));
  });
}

// ---- feature table + execute_plan (engine.cpp:411-527) ---------------------

void* ref_features_create() { return new FeatureTable; }
void ref_features_add(void* h, uint64_t id, const float* desc, uint64_t n) {
  static_cast<FeatureTable*>(h)->features[id] = fs_from(id, desc, n);
}
void ref_features_free(void* h) { delete static_cast<FeatureTable*>(h); }

// Runs the reference execute_plan as shipped (verification off, one matcher
// thread) and returns its matches flattened in result order:
// pair_ids[2*p], offsets[p+1], matches[2*m].  Buffers must be large enough.
int ref_execute_plan(const char* plan_path, void* features, uint64_t hash_seed, int tables,
                     int cb, int fb, int k, double ratio, uint64_t capacity_units,
                     uint64_t* pair_ids, uint64_t* offsets, int32_t* matches,
                     uint64_t* n_pairs_out, double* wall_s_out, uint64_t* counters_out) {
  return guarded([&] {
    const SchedulePlan plan = read_plan(plan_path);
    const HashFunctions hf = make_hash_functions(hash_seed, {tables, cb, fb});
    DeviceArena arena(capacity_units);
    ExecuteOptions opts;
    opts.match.k_nearest = k;
    opts.match.ratio = ratio;
    opts.verify.enabled = false;
    const ExecutionResult res =
        execute_plan(plan, static_cast<FeatureTable*>(features)->features, hf, arena, opts);
    uint64_t m = 0;
    offsets[0] = 0;
    for (size_t p = 0; p < res.matches.size(); ++p) {
      pair_ids[2 * p] = res.matches[p].query_image;
      pair_ids[2 * p + 1] = res.matches[p].train_image;
      for (const auto& [qi, ti] : res.matches[p].matches) {
        matches[2 * m] = qi;
        matches[2 * m + 1] = ti;
        ++m;
      }
      offsets[p + 1] = m;
    }
    *n_pairs_out = res.matches.size();
    *wall_s_out = res.metrics.wall_time_s;
    counters_out[0] = res.metrics.pairs_matched;
    counters_out[1] = res.metrics.initial_matches;
    counters_out[2] = res.metrics.uploads;
    counters_out[3] = res.metrics.evictions;
    counters_out[4] = res.metrics.units_uploaded;
    counters_out[5] = res.metrics.peak_occupancy;
  });
}

// Baseline (ii) "host cores": the same reference functions (row mean restated
// from engine.cpp:446-461, compute_codes, match_pair) with the independent
// per-image code computations and per-pair matches of each row spread over
// `threads` std::threads.  Output equals execute_plan's (pairs keyed by
// IdPair, engine.cpp:419, 506-512).  Runs the plan's rows [row_begin, row_end)
// (global row numbers in plan order, iteration by iteration; row_end = 0
// means every row) and returns wall seconds of that work.  When pair_ids is
// non-null the results are returned like ref_execute_plan's (pairs sorted by
// IdPair): pair_ids[2*p], offsets[p+1], matches[2*m] with m <= match_cap.
int ref_execute_plan_rows(const char* plan_path, void* features, uint64_t hash_seed, int tables,
                          int cb, int fb, int k, double ratio, int threads, uint64_t row_begin,
                          uint64_t row_end, uint64_t* pairs_done, uint64_t* total_matches,
                          double* wall_s_out, void** results_out) {
  return guarded([&] {
    const SchedulePlan plan = read_plan(plan_path);
    const HashFunctions hf = make_hash_functions(hash_seed, {tables, cb, fb});
    const auto& feats = static_cast<FeatureTable*>(features)->features;
    MatchParams mp;
    mp.k_nearest = k;
    mp.ratio = ratio;
    const int T = std::max(1, threads);
    const auto t0 = std::chrono::steady_clock::now();
    std::map<IdPair, PairMatches> results;
    uint64_t done = 0, global_row = 0;
    for (const ScheduleIteration& it : plan.iterations) {
      for (const BlockRow& row : it.rows) {
        const uint64_t gr = global_row++;
        if (gr < row_begin || (row_end && gr >= row_end)) continue;
        std::set<ImageId> needed(row.row_images.begin(), row.row_images.end());
        for (const ScheduleBlock& blk : row.blocks)
          needed.insert(blk.col_images.begin(), blk.col_images.end());
        std::array<double, kDescriptorDim> acc{};
        std::size_t total = 0;
        for (ImageId id : needed) {
          const FeatureSet& fs = feats.at(id);
          for (const Descriptor& d : fs.descriptors)
            for (int c = 0; c < kDescriptorDim; ++c) acc[c] += d.v[c];
          total += fs.size();
        }
        std::array<float, kDescriptorDim> mean{};
        if (total > 0)
          for (int c = 0; c < kDescriptorDim; ++c)
            mean[c] = static_cast<float>(acc[c] / static_cast<double>(total));
        std::vector<ImageId> ids(needed.begin(), needed.end());
        std::vector<HashCodeSet> codes(ids.size());
        {
          std::atomic<size_t> next{0};
          std::vector<std::thread> pool;
          for (int w = 0; w < T; ++w)
            pool.emplace_back([&] {
              for (size_t i; (i = next++) < ids.size();)
                codes[i] = compute_codes(feats.at(ids[i]), hf, mean);
            });
          for (auto& th : pool) th.join();
        }
        std::map<ImageId, const HashCodeSet*> by_id;
        for (size_t i = 0; i < ids.size(); ++i) by_id[ids[i]] = &codes[i];
        std::vector<IdPair> pairs;
        for (const ScheduleBlock& blk : row.blocks)
          pairs.insert(pairs.end(), blk.pairs.begin(), blk.pairs.end());
        std::vector<PairMatches> out(pairs.size());
        {
          std::atomic<size_t> next{0};
          std::vector<std::thread> pool;
          for (int w = 0; w < T; ++w)
            pool.emplace_back([&] {
              for (size_t i; (i = next++) < pairs.size();)
                out[i] = match_pair(feats.at(pairs[i].a), *by_id.at(pairs[i].a),
                                    feats.at(pairs[i].b), *by_id.at(pairs[i].b), mp);
            });
          for (auto& th : pool) th.join();
        }
        for (size_t i = 0; i < pairs.size(); ++i) results[pairs[i]] = std::move(out[i]);
        done += pairs.size();
      }
    }
    const std::chrono::duration<double> dt = std::chrono::steady_clock::now() - t0;
    uint64_t m = 0;
    for (const auto& [p, pm] : results) m += pm.matches.size();
    *pairs_done = done;
    *total_matches = m;
    *wall_s_out = dt.count();
    if (results_out) *results_out = new Results{std::move(results)};
  });
}

uint64_t ref_results_pairs(void* h) { return static_cast<Results*>(h)->r.size(); }
uint64_t ref_results_matches(void* h) {
  uint64_t m = 0;
  for (const auto& [p, pm] : static_cast<Results*>(h)->r) m += pm.matches.size();
  return m;
}
// pair_ids[2*p] (IdPair order), offsets[p+1], matches[2*m]
void ref_results_copy(void* h, uint64_t* pair_ids, uint64_t* offsets, int32_t* matches) {
  uint64_t o = 0, p = 0;
  offsets[0] = 0;
  for (const auto& [key, pm] : static_cast<Results*>(h)->r) {
    pair_ids[2 * p] = pm.query_image;
    pair_ids[2 * p + 1] = pm.train_image;
    for (const auto& [qi, ti] : pm.matches) {
      matches[2 * o] = qi;
      matches[2 * o + 1] = ti;
      ++o;
    }
    offsets[++p] = o;
  }
}
void ref_results_free(void* h) { delete static_cast<Results*>(h); }

// The reference's synthetic scene (features.cpp:68-197) straight into a
// feature table, images [drop, n_images) renumbered from 0 (the bench
// workloads drop the short leading images of a band scene).
void* ref_synth_features(int n_images, int ppi, int band, double sigma, double outlier_fraction,
                         uint64_t seed, int drop) {
  FeatureTable* t = new FeatureTable;
  const int rc = guarded([&] {
    SyntheticScene sc;
    sc.n_images = n_images;
    sc.points_per_image = ppi;
    sc.overlap_band = band;
    sc.noise_sigma = sigma;
    sc.outlier_fraction = outlier_fraction;
    sc.seed = seed;
    SyntheticDataset data = generate_synthetic(sc);
    for (int i = drop; i < n_images; ++i) {
      FeatureSet fs = std::move(data.images.at(i));
      fs.image_id = static_cast<ImageId>(i - drop);
      t->features[fs.image_id] = std::move(fs);
    }
  });
  if (rc != 0) {
    delete t;
    return nullptr;
  }
  return t;
}

uint64_t ref_features_count(void* h, uint64_t id) {
  const auto& f = static_cast<FeatureTable*>(h)->features;
  const auto it = f.find(id);
  return it == f.end() ? 0 : it->second.size();
}

// ---- verification stage 1 (verify.cpp:135-341, compiled from the reference) --

// knn_from_delaunay: neighbors_out[n * k] (-1 padded), fallback flag
int ref_knn_from_delaunay(const double* xy, uint64_t n, int k, int32_t* neighbors_out, int* fallback_out) {
  return guarded([&] {
    std::vector<Point2> pts(n);
    for (uint64_t i = 0; i < n; ++i) pts[i] = Point2{xy[2 * i], xy[2 * i + 1]};
    const DelaunayKnn d = knn_from_delaunay(pts, k);
    for (uint64_t i = 0; i < n; ++i)
      for (int j = 0; j < k; ++j)
        neighbors_out[i * k + j] = j < static_cast<int>(d.neighbors[i].size()) ? d.neighbors[i][j] : -1;
    *fallback_out = d.used_fallback ? 1 : 0;
  });
}

// sao_filter: keep_out[m], scores_out[m], flags (1 passthrough, 2 fallback)
int ref_sao_filter(const int32_t* matches, uint64_t m, const float* qkp, uint64_t nq, const float* tkp,
                   uint64_t nt, int n_neighbors, double threshold, uint8_t* keep_out, double* scores_out,
                   uint32_t* flags_out) {
  return guarded([&] {
    PairMatches pm;
    for (uint64_t i = 0; i < m; ++i) pm.matches.emplace_back(matches[2 * i], matches[2 * i + 1]);
    auto kps = [](const float* k, uint64_t n) {
      std::vector<Keypoint> v(n);
      for (uint64_t i = 0; i < n; ++i) v[i] = Keypoint{k[4 * i], k[4 * i + 1], k[4 * i + 2], k[4 * i + 3]};
      return v;
    };
    SaoParams sp;
    sp.n_neighbors = n_neighbors;
    sp.score_threshold = threshold;
    const SaoOutcome o = sao_filter(pm, kps(qkp, nq), kps(tkp, nt), sp);
    // kept matches are the input ones with score <= threshold, in input order
    size_t k = 0;
    for (uint64_t i = 0; i < m; ++i) {
      const bool kept = k < o.kept.matches.size() && o.kept.matches[k] == pm.matches[i] &&
                        (o.passthrough || o.scores[i] <= threshold);
      keep_out[i] = kept ? 1 : 0;
      k += kept ? 1 : 0;
      scores_out[i] = o.scores[i];
    }
    *flags_out = (o.passthrough ? 1u : 0u) | (o.delaunay_fallback ? 2u : 0u);
  });
}

// ---- retrieval (retrieval.cpp:14-205, compiled from the reference) --------

// encode_vlad: values_out[k_words * 128], degenerate_out
int ref_encode_vlad(const float* centroids, int k_words, const float* desc, uint64_t n, float* values_out,
                    uint8_t* degenerate_out) {
  return guarded([&] {
    Codebook cb;
    cb.k_words = k_words;
    cb.centroids.assign(centroids, centroids + static_cast<size_t>(std::max(k_words, 0)) * kDescriptorDim);
    FeatureSet fs;
    fs.descriptors.resize(n);
    fs.keypoints.resize(n);
    if (n) std::memcpy(fs.descriptors.data(), desc, n * kDescriptorDim * sizeof(float));
    const VladVector v = encode_vlad(fs, cb);
    std::memcpy(values_out, v.values.data(), v.values.size() * sizeof(float));
    *degenerate_out = v.degenerate ? 1 : 0;
  });
}

// encode_vlad over many images on `threads` host threads (the select_pairs
// loop, retrieval.cpp:397-398, spread over cores): the CPU baseline
int ref_encode_vlad_batch(const float* centroids, int k_words, const float* const* descs, const uint64_t* counts,
                          uint64_t n_images, int threads, float* values_out, uint8_t* degenerate_out) {
  return guarded([&] {
    Codebook cb;
    cb.k_words = k_words;
    cb.centroids.assign(centroids, centroids + static_cast<size_t>(std::max(k_words, 0)) * kDescriptorDim);
    const size_t dim = static_cast<size_t>(k_words) * kDescriptorDim;
    std::atomic<uint64_t> next{0};
    std::vector<std::string> errs(std::max(threads, 1));
    auto work = [&](int w) {
      try {
        for (uint64_t i; (i = next.fetch_add(1)) < n_images;) {
          FeatureSet fs;
          fs.descriptors.resize(counts[i]);
          fs.keypoints.resize(counts[i]);
          if (counts[i]) std::memcpy(fs.descriptors.data(), descs[i], counts[i] * kDescriptorDim * sizeof(float));
          const VladVector v = encode_vlad(fs, cb);
          std::memcpy(values_out + i * dim, v.values.data(), dim * sizeof(float));
          degenerate_out[i] = v.degenerate ? 1 : 0;
        }
      } catch (const std::exception& e) {
        errs[w] = e.what();
      }
    };
    std::vector<std::thread> pool;
    for (int w = 1; w < threads; ++w) pool.emplace_back(work, w);
    work(0);
    for (auto& t : pool) t.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::runtime_error(e);
  });
}

// train_codebook on descriptors [n][128]: centroids_out[k_words * 128],
// sse_out[max_iters] (entries written: *n_sse)
int ref_train_codebook(const float* desc, uint64_t n, int k_words, int max_iters, uint64_t seed,
                       float* centroids_out, double* sse_out, int* n_sse) {
  return guarded([&] {
    std::vector<Descriptor> d(n);
    if (n) std::memcpy(d.data(), desc, n * kDescriptorDim * sizeof(float));
    std::vector<double> hist;
    const Codebook cb = train_codebook(d, k_words, max_iters, seed, &hist);
    std::memcpy(centroids_out, cb.centroids.data(), cb.centroids.size() * sizeof(float));
    for (size_t i = 0; i < hist.size(); ++i) sse_out[i] = hist[i];
    *n_sse = static_cast<int>(hist.size());
  });
}

// File formats: the reference's own writers and
// reader, for byte-level parity and as the timed CPU baseline of tools/io_bench.py.
int ref_write_features(const char* path, uint64_t id, const float* desc, const float* kp, uint64_t n) {
  return guarded([&] {
    FeatureSet fs = fs_from(id, desc, n);
    for (uint64_t i = 0; i < n; ++i)
      fs.keypoints[i] = Keypoint{kp[4 * i], kp[4 * i + 1], kp[4 * i + 2], kp[4 * i + 3]};
    write_features(path, fs);
  });
}

// read_features; desc_out / kp_out may be null (count only)
int ref_read_features(const char* path, uint64_t capacity, uint64_t* id, uint64_t* n, float* desc_out,
                      float* kp_out) {
  return guarded([&] {
    const FeatureSet fs = read_features(path);
    *id = fs.image_id;
    *n = fs.size();
    if (desc_out && fs.size() <= capacity) {
      std::memcpy(desc_out, fs.descriptors.data(), fs.size() * sizeof(Descriptor));
      for (size_t i = 0; i < fs.size(); ++i) {
        kp_out[4 * i] = fs.keypoints[i].x;
        kp_out[4 * i + 1] = fs.keypoints[i].y;
        kp_out[4 * i + 2] = fs.keypoints[i].scale;
        kp_out[4 * i + 3] = fs.keypoints[i].orientation;
      }
    }
  });
}

// write_matches_binary of pairs[p] = (q, t) with matches[offsets[p]..offsets[p+1])
int ref_write_matches_binary(const char* path, uint64_t n_pairs, const uint64_t* pair_ids,
                             const uint64_t* offsets, const int32_t* matches, const uint8_t* stages) {
  return guarded([&] {
    std::vector<PairMatches> all(n_pairs);
    for (uint64_t p = 0; p < n_pairs; ++p) {
      all[p].query_image = pair_ids[2 * p];
      all[p].train_image = pair_ids[2 * p + 1];
      all[p].stage = stages && stages[p] ? PairMatches::Stage::kVerified : PairMatches::Stage::kInitial;
      for (uint64_t m = offsets[p]; m < offsets[p + 1]; ++m)
        all[p].matches.emplace_back(matches[2 * m], matches[2 * m + 1]);
    }
    write_matches_binary(path, all);
  });
}

}  // extern "C"
