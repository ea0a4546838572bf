// bandmatch_b200.hpp -- reference-side binding of the B200 matcher.
//
// Header-only C++ adapter a bandmatch maintainer adds next to
// include/bandmatch/engine.hpp: the reference's own types (FeatureSet,
// HashFunctions, HashCodeSet, PairMatches, SchedulePlan, DeviceArena,
// ExecuteOptions, ExecutionResult) on top of the C ABI in bandmatch_gpu.h.
// Errors come back as bandmatch::Error with the reference's stable codes.
//
//   reference call                         | drop-in
//   ---------------------------------------+-------------------------------------------
//   compute_codes(fs, hf, mean)            | bandmatch_b200::compute_codes(ctx, fs, hf, mean)
//     hashmatch.cpp:71-100                 |
//   match_pair(qf, qc, tf, tc, mp)         | bandmatch_b200::match_pair(ctx, qf, qc, tf, tc, mp)
//     hashmatch.cpp:102-211                |
//   execute_plan(plan, feats, hf, arena,   | bandmatch_b200::execute_plan(ctx, plan, feats, hf,
//                opts, graph)              |                              arena, opts, graph)
//     engine.cpp:411-527                   |   (call sites: bandmatch_cli.cpp:234, :278)
//   encode_vlad(fs, cb) per image          | bandmatch_b200::encode_vlad_batch(ctx, feats, cb)
//   train_codebook(pool, k, iters, seed)    | bandmatch_b200::train_codebook(ctx, pool, k, iters, seed)
//     retrieval.cpp:160-205                |
//   select_pairs(feats, cb, top_n, hnsw,   | bandmatch_b200::select_pairs(ctx, feats, cb, top_n,
//                seed) retrieval.cpp:386   |                              hnsw, seed)
//
// The caller's DeviceArena is kept in step with the HBM arena through the
// DeviceBackend hooks (engine.hpp:98-104), so its counters, CapacityExceeded
// and NotResident behave exactly as in the reference.  With
// opts.verify.enabled the initial matches are verified on host threads with
// sao_filter (libbmg's native SAO, bit-equal) + the reference's ransac_fundamental, as VerifyPool does
// (engine.cpp:326-377), WHILE the GPU matches later rows: each block row's
// pairs arrive through the executor's on_pair hand-off as soon as that row's
// matches are in host memory and go into a bounded queue (backpressure as in
// VerifyPool::push, engine.cpp:293-299) that opts.threads workers drain.
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <deque>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "bandmatch/engine.hpp"
#include "bandmatch/hashmatch.hpp"
#include "bandmatch/retrieval.hpp"
#include "bandmatch_gpu.h"

namespace bandmatch_b200 {

inline void check(int rc) {
  if (rc != BMG_OK) bandmatch::fail(bmg_status_name(rc), bmg_last_error());
}

// One B200 device context: hash planes resident in HBM, the descriptor arena
// and the kernels' scratch.  Not thread-safe (matching runs on one caller
// thread, engine.hpp:109).
class Context {
 public:
  Context(const bandmatch::HashFunctions& hf, std::uint64_t capacity_units, int device = 0)
      : seed_(hf.seed), params_(hf.params) {
    bmg_config cfg{};
    cfg.device = device;
    cfg.hash = {hf.params.tables, hf.params.coarse_bits, hf.params.fine_bits};
    cfg.coarse_planes = hf.coarse.data();
    cfg.fine_planes = hf.fine.data();
    cfg.function_seed = hf.seed;
    cfg.capacity_units = capacity_units;
    check(bmg_create(&cfg, &ctx_));
  }
  ~Context() { bmg_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bmg_context* get() const { return ctx_; }
  std::uint64_t seed() const { return seed_; }
  const bandmatch::HashParams& params() const { return params_; }

 private:
  bmg_context* ctx_ = nullptr;
  std::uint64_t seed_;
  bandmatch::HashParams params_;
};

inline const float* desc_ptr(const bandmatch::FeatureSet& fs) {
  return fs.descriptors.empty() ? nullptr : fs.descriptors[0].v.data();
}

inline bandmatch::HashCodeSet compute_codes(Context& ctx, const bandmatch::FeatureSet& fs,
                                            const bandmatch::HashFunctions& hf,
                                            const std::array<float, bandmatch::kDescriptorDim>& mean) {
  if (hf.seed != ctx.seed()) bandmatch::fail("HashMismatch", "context built from other hash functions");
  bandmatch::HashCodeSet cs;
  cs.image_id = fs.image_id;
  cs.function_seed = hf.seed;
  cs.params = hf.params;
  cs.count = fs.size();
  cs.fine_words = (hf.params.fine_bits + 63) / 64;
  cs.coarse.assign(cs.count * hf.params.tables, 0);
  cs.fine.assign(cs.count * cs.fine_words, 0);
  check(bmg_compute_codes(ctx.get(), desc_ptr(fs), cs.count, mean.data(), cs.coarse.data(),
                          cs.fine.data()));
  return cs;
}

inline bmg_code_set view_of(const bandmatch::HashCodeSet& cs) {
  bmg_code_set v{};
  v.image_id = cs.image_id;
  v.function_seed = cs.function_seed;
  v.params = {cs.params.tables, cs.params.coarse_bits, cs.params.fine_bits};
  v.count = cs.count;
  v.coarse = cs.coarse.data();
  v.fine = cs.fine.data();
  return v;
}

inline bandmatch::PairMatches match_pair(Context& ctx, const bandmatch::FeatureSet& qf,
                                         const bandmatch::HashCodeSet& qc,
                                         const bandmatch::FeatureSet& tf,
                                         const bandmatch::HashCodeSet& tc,
                                         const bandmatch::MatchParams& mp) {
  if (qc.count != qf.size() || tc.count != tf.size())
    bandmatch::fail("HashMismatch", "code set does not cover its feature set");
  bandmatch::PairMatches pm;
  pm.query_image = qf.image_id;
  pm.train_image = tf.image_id;
  const bmg_code_set qv = view_of(qc), tv = view_of(tc);
  const bmg_match_params p{mp.k_nearest, mp.ratio};
  std::vector<std::int32_t> out(2 * std::max<std::size_t>(qf.size(), 1));
  std::uint64_t n = 0;
  check(bmg_match_pair(ctx.get(), desc_ptr(qf), &qv, desc_ptr(tf), &tv, &p, out.data(), &n));
  pm.matches.reserve(n);
  for (std::uint64_t i = 0; i < n; ++i) pm.matches.emplace_back(out[2 * i], out[2 * i + 1]);
  return pm;
}

// sao_filter (verify.hpp:53-54, verify.cpp:303-341) on libbmg's native SAO
// (bmg_sao_filter: the reference's triangulation and rings, adjacency-driven
// instead of the all-triangle Bowyer-Watson), the reference's outcome type.
inline bandmatch::SaoOutcome sao_filter(const bandmatch::PairMatches& in,
                                        const std::vector<bandmatch::Keypoint>& query_kps,
                                        const std::vector<bandmatch::Keypoint>& train_kps,
                                        const bandmatch::SaoParams& params) {
  static_assert(sizeof(bandmatch::Keypoint) == 4 * sizeof(float), "Keypoint must be float[4]");
  const std::size_t m = in.matches.size();
  std::vector<std::int32_t> flat(2 * std::max<std::size_t>(m, 1));
  for (std::size_t i = 0; i < m; ++i) {
    flat[2 * i] = static_cast<std::int32_t>(in.matches[i].first);
    flat[2 * i + 1] = static_cast<std::int32_t>(in.matches[i].second);
  }
  std::vector<std::uint8_t> keep(std::max<std::size_t>(m, 1));
  bandmatch::SaoOutcome out;
  out.scores.assign(m, 0.0);
  std::uint32_t flags = 0;
  check(bmg_sao_filter(flat.data(), m, query_kps.empty() ? nullptr : &query_kps[0].x, query_kps.size(),
                       train_kps.empty() ? nullptr : &train_kps[0].x, train_kps.size(), params.n_neighbors,
                       params.score_threshold, keep.data(), out.scores.data(), &flags));
  out.passthrough = (flags & BMG_SAO_PASSTHROUGH) != 0;
  out.delaunay_fallback = (flags & BMG_SAO_DELAUNAY_FALLBACK) != 0;
  out.kept.query_image = in.query_image;
  out.kept.train_image = in.train_image;
  out.kept.stage = in.stage;
  for (std::size_t i = 0; i < m; ++i)
    if (keep[i]) out.kept.matches.push_back(in.matches[i]);
  return out;
}

namespace detail {

struct Hooks {
  bandmatch::DeviceArena* arena;
  const bandmatch::DeviceBackend* backend;
  static void on_upload(void* u, std::uint64_t id, std::uint64_t units) {
    auto* h = static_cast<Hooks*>(u);
    h->arena->upload(id, units);
    if (h->backend->on_upload) h->backend->on_upload(id, units);
  }
  static void on_evict(void* u, std::uint64_t id) {
    auto* h = static_cast<Hooks*>(u);
    h->arena->evict(id);
    if (h->backend->on_evict) h->backend->on_evict(id);
  }
};

// Verification overlapped with the GPU: a bounded producer / consumer queue
// fed by bmg_execute_plan's on_pair hand-off (collector thread) and drained
// by `threads` workers running the reference's SAO + RANSAC per pair
// (VerifyPool, engine.cpp:275-390; its per-job body :326-377).  push blocks
// while the queue is full -- backpressure on the collector thread only, the
// GPU keeps matching.  Results are keyed by IdPair (engine.cpp:419).
class Verifier {
 public:
  struct Record {
    bandmatch::PairMatches matches;
    bandmatch::PairOutcome outcome;
  };
  Verifier(const std::map<bandmatch::ImageId, bandmatch::FeatureSet>& features,
           const bandmatch::ExecuteOptions& opts)
      : features_(features), opts_(opts), capacity_(std::max<std::size_t>(1, opts.queue_capacity)) {
    for (int w = 0; w < std::max(1, opts.threads); ++w) workers_.emplace_back([this] { run(); });
  }
  ~Verifier() { close(); }

  // bmg_pair_callback: copy the pair's initial matches out of the pinned
  // log and queue the job
  static void on_pair(void* u, std::uint64_t q, std::uint64_t t, const std::int32_t* m,
                      std::uint64_t n) {
    auto* v = static_cast<Verifier*>(u);
    Job job;
    job.initial.query_image = q;
    job.initial.train_image = t;
    job.initial.matches.reserve(n);
    for (std::uint64_t i = 0; i < n; ++i) job.initial.matches.emplace_back(m[2 * i], m[2 * i + 1]);
    std::unique_lock<std::mutex> lk(v->mu_);
    v->push_cv_.wait(lk, [v] { return v->queue_.size() < v->capacity_; });
    v->queue_.push_back(std::move(job));
    v->pop_cv_.notify_one();
  }

  // every queued job processed, workers joined; rethrows the first error
  void close() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      if (closed_) return;
      closed_ = true;
    }
    pop_cv_.notify_all();
    for (std::thread& t : workers_) t.join();
    if (err_) std::rethrow_exception(err_);
  }

  std::map<bandmatch::IdPair, Record> records;

 private:
  struct Job {
    bandmatch::PairMatches initial;
  };
  void run() {
    for (;;) {
      Job job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        pop_cv_.wait(lk, [this] { return closed_ || !queue_.empty(); });
        if (queue_.empty()) return;
        job = std::move(queue_.front());
        queue_.pop_front();
      }
      push_cv_.notify_one();
      Record rec = process(job.initial);
      std::lock_guard<std::mutex> lk(mu_);
      records[rec.outcome.pair] = std::move(rec);
    }
  }
  Record process(const bandmatch::PairMatches& in) {
    using namespace bandmatch;
    Record r;
    const FeatureSet& qf = features_.at(in.query_image);
    const FeatureSet& tf = features_.at(in.train_image);
    r.matches.query_image = in.query_image;
    r.matches.train_image = in.train_image;
    r.matches.stage = PairMatches::Stage::kVerified;
    PairOutcome& oc = r.outcome;
    oc.pair = IdPair(in.query_image, in.train_image);
    oc.initial = in.matches.size();
    try {
      const SaoOutcome sao = bandmatch_b200::sao_filter(in, qf.keypoints, tf.keypoints, opts_.verify.sao);
      oc.after_sao = sao.kept.matches.size();
      oc.sao_passthrough = sao.passthrough;
      oc.delaunay_fallback = sao.delaunay_fallback;
      const std::uint64_t seed =
          seed_for(opts_.seed, "verify." + std::to_string(oc.pair.a) + "." + std::to_string(oc.pair.b));
      const InlierSet inl = ransac_fundamental(sao.kept, qf.keypoints, tf.keypoints, opts_.verify.ransac, seed);
      for (int idx : inl.kept) r.matches.matches.push_back(sao.kept.matches[idx]);
      oc.inliers = r.matches.matches.size();
      oc.ransac_iterations = inl.iterations;
    } catch (const Error& e) {
      oc.no_model = true;
      r.matches.matches.clear();
      if (e.code() != "TooFewMatches" && e.code() != "NoModel") {
        std::lock_guard<std::mutex> lk(mu_);
        if (!err_) err_ = std::current_exception();
      }
    } catch (...) {
      oc.no_model = true;
      r.matches.matches.clear();
      std::lock_guard<std::mutex> lk(mu_);
      if (!err_) err_ = std::current_exception();
    }
    oc.inlier_ratio = oc.initial == 0 ? 0.0 : static_cast<double>(oc.inliers) / oc.initial;
    return r;
  }

  const std::map<bandmatch::ImageId, bandmatch::FeatureSet>& features_;
  const bandmatch::ExecuteOptions& opts_;
  const std::size_t capacity_;
  std::mutex mu_;
  std::condition_variable push_cv_, pop_cv_;
  std::deque<Job> queue_;
  bool closed_ = false;
  std::exception_ptr err_;
  std::vector<std::thread> workers_;
};

}  // namespace detail

// execute_plan (engine.cpp:411-527): the row body runs on the B200; results,
// metrics and the arena follow the reference's semantics.
inline bandmatch::ExecutionResult execute_plan(
    Context& ctx, const bandmatch::SchedulePlan& plan,
    const std::map<bandmatch::ImageId, bandmatch::FeatureSet>& features,
    const bandmatch::HashFunctions& hf, bandmatch::DeviceArena& arena,
    const bandmatch::ExecuteOptions& opts, bandmatch::ViewGraph* graph = nullptr) {
  using namespace bandmatch;
  if (hf.seed != ctx.seed()) fail("HashMismatch", "context built from other hash functions");
  // flatten the plan (mbr.hpp:26-68)
  std::vector<std::uint64_t> rpi, nd_off{0}, nd, p_off{0}, prs, ev_off{0}, ev;
  for (const ScheduleIteration& it : plan.iterations) {
    rpi.push_back(it.rows.size());
    for (const BlockRow& row : it.rows) {
      std::set<ImageId> needed(row.row_images.begin(), row.row_images.end());
      for (const ScheduleBlock& blk : row.blocks) {
        needed.insert(blk.col_images.begin(), blk.col_images.end());
        for (const IdPair& p : blk.pairs) {
          prs.push_back(p.a);
          prs.push_back(p.b);
        }
      }
      nd.insert(nd.end(), needed.begin(), needed.end());
      nd_off.push_back(nd.size());
      p_off.push_back(prs.size() / 2);
      ev.insert(ev.end(), row.evict_after.begin(), row.evict_after.end());
      ev_off.push_back(ev.size());
    }
  }
  bmg_plan fp{};
  fp.n_iterations = rpi.size();
  fp.rows_per_iteration = rpi.data();
  fp.n_rows = nd_off.size() - 1;
  fp.row_needed_offsets = nd_off.data();
  fp.needed_ids = nd.data();
  fp.row_pair_offsets = p_off.data();
  fp.pairs = prs.data();
  fp.row_evict_offsets = ev_off.data();
  fp.evict_ids = ev.data();
  std::vector<bmg_feature_view> views;
  for (const auto& [id, fs] : features) views.push_back({id, desc_ptr(fs), fs.size()});
  detail::Hooks hooks{&arena, &opts.backend};
  bmg_execute_options eo{};
  eo.match = {opts.match.k_nearest, opts.match.ratio};
  eo.on_upload = &detail::Hooks::on_upload;
  eo.on_evict = &detail::Hooks::on_evict;
  eo.hook_user = &hooks;
  std::unique_ptr<detail::Verifier> verifier;
  if (opts.verify.enabled) {
    verifier = std::make_unique<detail::Verifier>(features, opts);
    eo.on_pair = &detail::Verifier::on_pair;
    eo.on_pair_user = verifier.get();
  }
  bmg_result* r = nullptr;
  const int rc = bmg_execute_plan(ctx.get(), &fp, views.data(), views.size(), &eo, &r);
  if (rc != BMG_OK && verifier) {
    const std::string msg = bmg_last_error();
    try {
      verifier->close();
    } catch (...) {
    }
    bandmatch::fail(bmg_status_name(rc), msg);
  }
  check(rc);
  std::unique_ptr<bmg_result, void (*)(bmg_result*)> guard(r, bmg_result_free);
  const std::uint64_t n_pairs = bmg_result_pair_count(r), n_m = bmg_result_match_count(r);
  std::vector<std::uint64_t> ids(2 * n_pairs), offs(n_pairs + 1);
  std::vector<std::int32_t> m(2 * n_m);
  check(bmg_result_copy(r, ids.data(), offs.data(), m.data()));
  std::uint64_t counters[6];
  double wall = 0.0;
  check(bmg_result_metrics(r, counters, &wall));

  ExecutionResult res;
  res.metrics.strategy = plan.strategy;
  res.metrics.pairs_matched = counters[0];
  res.metrics.initial_matches = counters[1];
  for (std::uint64_t i = 0; i < bmg_result_iteration_count(r); ++i) {
    std::uint64_t o[3];
    check(bmg_result_iteration(r, i, o));
    IterationMetrics im;
    im.dimension = plan.iterations[i].dimension;
    im.pairs = o[0];
    im.uploads = o[1];
    im.units_uploaded = o[2];
    res.metrics.per_iteration.push_back(im);
  }
  std::vector<PairMatches> initial(n_pairs);
  for (std::uint64_t p = 0; p < n_pairs; ++p) {
    initial[p].query_image = ids[2 * p];
    initial[p].train_image = ids[2 * p + 1];
    for (std::uint64_t k = offs[p]; k < offs[p + 1]; ++k)
      initial[p].matches.emplace_back(m[2 * k], m[2 * k + 1]);
    if (graph) graph->set_pair_state(IdPair(ids[2 * p], ids[2 * p + 1]), PairState::kProcessed);
  }
  if (!opts.verify.enabled) {
    res.matches = std::move(initial);
  } else {
    // the workers have been verifying since the first row's hand-off; wait
    // for the rest (the iteration barrier of engine.cpp:497-499 only orders
    // verification against the next iteration's matching, which cannot
    // change any result, so the GPU does not wait for it)
    verifier->close();
    for (auto& [pair, rec] : verifier->records) {
      res.outcomes.push_back(rec.outcome);
      res.matches.push_back(std::move(rec.matches));
      res.metrics.verified_matches += res.matches.back().matches.size();
    }
  }
  res.metrics.uploads = arena.uploads();
  res.metrics.evictions = arena.evictions();
  res.metrics.units_uploaded = arena.units_uploaded();
  res.metrics.peak_occupancy = arena.peak_occupancy();
  res.metrics.utilization_proxy =
      res.metrics.uploads == 0 ? 0.0
                               : static_cast<double>(res.metrics.pairs_matched) / res.metrics.uploads;
  res.metrics.wall_time_s = wall;
  res.metrics.pairs_per_second = wall > 0.0 ? res.metrics.pairs_matched / wall : 0.0;
  return res;
}

// ---- retrieval -----------------------------------------

// encode_vlad (retrieval.cpp:160-205) of every image in one device call
// (bit-exact with the reference's per-image encode_vlad).
inline std::vector<bandmatch::VladVector> encode_vlad_batch(Context& ctx,
                                                            const std::vector<bandmatch::FeatureSet>& features,
                                                            const bandmatch::Codebook& cb) {
  std::vector<bmg_feature_view> views(features.size());
  for (std::size_t i = 0; i < features.size(); ++i)
    views[i] = {features[i].image_id, desc_ptr(features[i]), features[i].size()};
  const std::size_t dim = static_cast<std::size_t>(std::max(cb.k_words, 0)) * bandmatch::kDescriptorDim;
  std::vector<float> vals(std::max<std::size_t>(features.size() * dim, 1));
  std::vector<std::uint8_t> deg(std::max<std::size_t>(features.size(), 1));
  check(bmg_encode_vlad(ctx.get(), cb.centroids.data(), cb.k_words, views.data(), views.size(), vals.data(),
                        deg.data()));
  std::vector<bandmatch::VladVector> out(features.size());
  for (std::size_t i = 0; i < features.size(); ++i) {
    out[i].values.assign(vals.begin() + i * dim, vals.begin() + (i + 1) * dim);
    out[i].degenerate = deg[i] != 0;
  }
  return out;
}

// train_codebook (retrieval.hpp:34-36, retrieval.cpp:56-158) on the device:
// the reference's seeding and Lloyd iterations, bit-exact centroids and SSE
// history; errors as the reference (InvalidArgument, TooFewDescriptors).
inline bandmatch::Codebook train_codebook(Context& ctx, const std::vector<bandmatch::Descriptor>& descriptors,
                                          int k_words, int max_iters, std::uint64_t seed,
                                          std::vector<double>* sse_history = nullptr) {
  static_assert(sizeof(bandmatch::Descriptor) == bandmatch::kDescriptorDim * sizeof(float),
                "Descriptor must be float[128]");
  const std::size_t dim = static_cast<std::size_t>(std::max(k_words, 1)) * bandmatch::kDescriptorDim;
  std::vector<float> cent(dim);
  std::vector<double> sse(static_cast<std::size_t>(std::max(max_iters, 1)));
  int n_sse = 0;
  check(bmg_train_codebook(ctx.get(), descriptors.empty() ? nullptr : descriptors[0].v.data(),
                           descriptors.size(), k_words, max_iters, seed, cent.data(), sse.data(), &n_sse));
  if (sse_history) sse_history->assign(sse.begin(), sse.begin() + n_sse);
  bandmatch::Codebook cb;
  cb.k_words = k_words;
  cb.centroids = std::move(cent);
  return cb;
}

// select_pairs (retrieval.cpp:386-415) with its per-image encode_vlad loop
// (:397-398) replaced by the batched GPU encoder; the HNSW index and the
// neighbour union are the reference's own code.
inline bandmatch::ViewGraph select_pairs(Context& ctx, const std::vector<bandmatch::FeatureSet>& features,
                                         const bandmatch::Codebook& cb, int retrieval_top_n,
                                         const bandmatch::HnswParams& params, std::uint64_t seed) {
  if (retrieval_top_n < 1) bandmatch::fail("InvalidArgument", "retrieval_top_n must be >= 1");
  std::vector<bandmatch::ImageId> ids;
  ids.reserve(features.size());
  for (const bandmatch::FeatureSet& fs : features) ids.push_back(fs.image_id);
  bandmatch::ViewGraph g{std::move(ids)};
  const int n = static_cast<int>(features.size());
  if (n <= 1) return g;
  const std::vector<bandmatch::VladVector> vlads = encode_vlad_batch(ctx, features, cb);
  bandmatch::HnswIndex index(cb.k_words * bandmatch::kDescriptorDim, params,
                             bandmatch::seed_for(seed, "retrieval.hnsw"));
  for (int i = 0; i < n; ++i) index.insert(i, vlads[i].values);
  for (int i = 0; i < n; ++i) {
    const auto found = index.search(vlads[i].values, retrieval_top_n + 1);
    int added = 0;
    for (const auto& [j, d] : found) {
      if (j == i) continue;
      if (added == retrieval_top_n) break;
      g.add_edge(i, j);
      ++added;
    }
  }
  return g;
}

}  // namespace bandmatch_b200
