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
//
// The caller's DeviceArena is kept in step with the HBM arena through the
// DeviceBackend hooks (engine.hpp:98-104), so its counters, CapacityExceeded
// and NotResident behave exactly as in the reference.  With
// opts.verify.enabled the initial matches are verified on host threads with
// the reference's sao_filter + ransac_fundamental, as VerifyPool does
// (engine.cpp:326-377).
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdint>
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
  bmg_result* r = nullptr;
  check(bmg_execute_plan(ctx.get(), &fp, views.data(), views.size(), &eo, &r));
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
    // host verification, as VerifyPool::process (engine.cpp:326-377)
    res.matches.resize(n_pairs);
    res.outcomes.resize(n_pairs);
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex err_mu;
    auto work = [&] {
      for (std::size_t i; (i = next++) < n_pairs;) {
        const PairMatches& in = initial[i];
        const FeatureSet& qf = features.at(in.query_image);
        const FeatureSet& tf = features.at(in.train_image);
        PairMatches& out = res.matches[i];
        PairOutcome& oc = res.outcomes[i];
        out.query_image = in.query_image;
        out.train_image = in.train_image;
        out.stage = PairMatches::Stage::kVerified;
        oc.pair = IdPair(in.query_image, in.train_image);
        oc.initial = in.matches.size();
        try {
          const SaoOutcome sao = sao_filter(in, qf.keypoints, tf.keypoints, opts.verify.sao);
          oc.after_sao = sao.kept.matches.size();
          oc.sao_passthrough = sao.passthrough;
          oc.delaunay_fallback = sao.delaunay_fallback;
          const std::uint64_t seed = seed_for(opts.seed, "verify." + std::to_string(oc.pair.a) +
                                                             "." + std::to_string(oc.pair.b));
          const InlierSet inl =
              ransac_fundamental(sao.kept, qf.keypoints, tf.keypoints, opts.verify.ransac, seed);
          for (int idx : inl.kept) out.matches.push_back(sao.kept.matches[idx]);
          oc.inliers = out.matches.size();
          oc.ransac_iterations = inl.iterations;
        } catch (const Error& e) {
          oc.no_model = true;
          out.matches.clear();
          if (e.code() != "TooFewMatches" && e.code() != "NoModel") {
            std::lock_guard<std::mutex> lk(err_mu);
            if (!err) err = std::current_exception();
          }
        }
        oc.inlier_ratio = oc.initial == 0 ? 0.0 : static_cast<double>(oc.inliers) / oc.initial;
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, opts.threads); ++t) pool.emplace_back(work);
    for (auto& t : pool) t.join();
    if (err) std::rethrow_exception(err);
    for (const PairMatches& pm : res.matches) res.metrics.verified_matches += pm.matches.size();
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

}  // namespace bandmatch_b200
