// test_reference_binding.cpp -- the reference's own C++ API driven through
// the drop-in binding (include/bandmatch_b200.hpp) against the UNMODIFIED
// reference (oracle/_ref objects compiled from /root/reference/proj/src).
// TEST INFRASTRUCTURE: built by tests/cpp/Makefile where the reference
// exists; the binary travels to the GPU box and is run by
// tests/test_gpu_binding.py.  Prints PASS/FAIL lines, exits non-zero on FAIL.
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <vector>

#include "bandmatch/engine.hpp"
#include "bandmatch/features.hpp"
#include "bandmatch/hashmatch.hpp"
#include "bandmatch/mbr.hpp"
#include "bandmatch/view_graph.hpp"
#include "bandmatch_b200.hpp"

using namespace bandmatch;

static int failures = 0;
static void report(bool ok, const char* what) {
  std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
  if (!ok) ++failures;
}

int main() {
  SyntheticScene sc;
  sc.n_images = 14;
  sc.points_per_image = 700;
  sc.overlap_band = 3;
  sc.noise_sigma = 0.02;
  sc.outlier_fraction = 0.2;
  sc.seed = 7;
  const SyntheticDataset data = generate_synthetic(sc);
  std::map<ImageId, FeatureSet> feats;
  std::vector<ImageId> ids;
  for (const FeatureSet& fs : data.images) {
    feats.emplace(fs.image_id, fs);
    ids.push_back(fs.image_id);
  }
  const ViewGraph g = make_view_graph(ids, data.true_pairs);
  const SchedulePlan plan = iterate_schedule(g, 3, 6);
  const HashFunctions hf = make_hash_functions(seed_for(42, "matching"));
  const std::uint64_t cap = arena_units_for(feats, 6);

  ExecuteOptions opts;
  opts.verify.enabled = false;
  DeviceArena ref_arena(cap);
  const ExecutionResult ref = execute_plan(plan, feats, hf, ref_arena, opts);

  bandmatch_b200::Context ctx(hf, cap);
  DeviceArena arena(cap);
  std::vector<ImageId> ups, evs;
  ExecuteOptions gopts = opts;
  gopts.backend.on_upload = [&](ImageId id, std::uint64_t) { ups.push_back(id); };
  gopts.backend.on_evict = [&](ImageId id) { evs.push_back(id); };
  ViewGraph marked = g;
  const ExecutionResult got = bandmatch_b200::execute_plan(ctx, plan, feats, hf, arena, gopts, &marked);

  bool same = got.matches.size() == ref.matches.size();
  for (std::size_t i = 0; same && i < ref.matches.size(); ++i)
    same = got.matches[i].query_image == ref.matches[i].query_image &&
           got.matches[i].train_image == ref.matches[i].train_image &&
           got.matches[i].matches == ref.matches[i].matches &&
           got.matches[i].stage == ref.matches[i].stage;
  report(same, "execute_plan match lists equal the reference, pair by pair");
  const PipelineMetrics &a = got.metrics, &b = ref.metrics;
  report(a.pairs_matched == b.pairs_matched && a.initial_matches == b.initial_matches &&
             a.uploads == b.uploads && a.evictions == b.evictions &&
             a.units_uploaded == b.units_uploaded && a.peak_occupancy == b.peak_occupancy &&
             a.per_iteration.size() == b.per_iteration.size(),
         "execute_plan metrics equal the reference (pairs, matches, uploads, evictions, units, peak)");
  report(ups.size() == b.uploads && evs.size() == b.evictions && arena.occupancy() == 0,
         "DeviceBackend hooks saw every arena transition; arena handed back empty");
  bool processed = true;
  for (const IdPair& p : g.pairs()) processed &= marked.pair_state(p) == PairState::kProcessed;
  report(processed, "view graph pairs marked processed");

  // sao_filter (verify.cpp:303-341) on libbmg's native SAO, every matched
  // pair, against the reference's own
  {
    bool eq = true;
    std::size_t n_checked = 0;
    for (const PairMatches& pm : ref.matches) {
      const FeatureSet& qf = feats.at(pm.query_image);
      const FeatureSet& tf = feats.at(pm.train_image);
      const SaoParams sp;
      const SaoOutcome r = sao_filter(pm, qf.keypoints, tf.keypoints, sp);
      const SaoOutcome gq = bandmatch_b200::sao_filter(pm, qf.keypoints, tf.keypoints, sp);
      eq &= r.kept.matches == gq.kept.matches && r.scores == gq.scores && r.passthrough == gq.passthrough &&
            r.delaunay_fallback == gq.delaunay_fallback && r.kept.query_image == gq.kept.query_image &&
            r.kept.train_image == gq.kept.train_image && r.kept.stage == gq.kept.stage;
      ++n_checked;
    }
    report(eq && n_checked > 0, "sao_filter on the native SAO equals the reference's, every matched pair");
  }

  // compute_codes / match_pair through the binding
  std::array<float, kDescriptorDim> mean{};
  for (int c = 0; c < kDescriptorDim; ++c) mean[c] = 0.001f * static_cast<float>(c % 7);
  const FeatureSet& q = feats.at(4);
  const FeatureSet& t = feats.at(5);
  const HashCodeSet rq = compute_codes(q, hf, mean), rt = compute_codes(t, hf, mean);
  const HashCodeSet gq = bandmatch_b200::compute_codes(ctx, q, hf, mean);
  const HashCodeSet gt = bandmatch_b200::compute_codes(ctx, t, hf, mean);
  report(gq.coarse == rq.coarse && gq.fine == rq.fine && gt.coarse == rt.coarse && gt.fine == rt.fine,
         "compute_codes equals the reference");
  MatchParams mp;
  report(bandmatch_b200::match_pair(ctx, q, gq, t, gt, mp).matches ==
             match_pair(q, rq, t, rt, mp).matches,
         "match_pair equals the reference");
  mp.k_nearest = 3;
  mp.ratio = 0.8;
  report(bandmatch_b200::match_pair(ctx, q, gq, t, gt, mp).matches ==
             match_pair(q, rq, t, rt, mp).matches,
         "match_pair (K=3, ratio=0.8) equals the reference");

  // retrieval: encode_vlad per image and select_pairs (retrieval.cpp:160-205,
  // :386-415) with the GPU encoder, against the reference
  {
    std::vector<FeatureSet> fv;
    for (const auto& [id, fs] : feats) fv.push_back(fs);
    std::vector<Descriptor> pool;
    for (const FeatureSet& fs : fv)
      for (std::size_t i = 0; i < fs.size(); i += 7) pool.push_back(fs.descriptors[i]);
    std::vector<double> rsse, gsse;
    const Codebook cb = train_codebook(pool, 16, 8, 11, &rsse);
    const Codebook gcb = bandmatch_b200::train_codebook(ctx, pool, 16, 8, 11, &gsse);
    report(gcb.k_words == cb.k_words && gcb.centroids.size() == cb.centroids.size() &&
               std::memcmp(gcb.centroids.data(), cb.centroids.data(), cb.centroids.size() * sizeof(float)) == 0 &&
               rsse == gsse,
           "train_codebook on the device equals the reference (centroids and SSE history), bit for bit");
    const std::vector<VladVector> gv = bandmatch_b200::encode_vlad_batch(ctx, fv, cb);
    bool eq = gv.size() == fv.size();
    for (std::size_t i = 0; eq && i < fv.size(); ++i) {
      const VladVector rv = encode_vlad(fv[i], cb);
      eq = rv.degenerate == gv[i].degenerate &&
           std::memcmp(rv.values.data(), gv[i].values.data(), rv.values.size() * sizeof(float)) == 0;
    }
    report(eq, "encode_vlad_batch equals the reference encode_vlad, bit for bit");
    HnswParams hp;
    const ViewGraph rg = select_pairs(fv, cb, 3, hp, 5);
    const ViewGraph gg = bandmatch_b200::select_pairs(ctx, fv, cb, 3, hp, 5);
    report(rg.pairs() == gg.pairs(), "select_pairs with the GPU encoder equals the reference");
  }

  // error semantics
  auto code_of = [](auto&& f) -> std::string {
    try {
      f();
    } catch (const Error& e) {
      return e.code();
    }
    return "";
  };
  const HashFunctions other = make_hash_functions(1);
  const HashCodeSet oq = compute_codes(q, other, mean);
  report(code_of([&] { bandmatch_b200::match_pair(ctx, q, oq, t, gt, MatchParams{}); }) == "HashMismatch",
         "HashMismatch on code sets from different seeds");
  MatchParams bad;
  bad.k_nearest = 0;
  report(code_of([&] { bandmatch_b200::match_pair(ctx, q, gq, t, gt, bad); }) == "InvalidArgument",
         "InvalidArgument on k_nearest < 1");
  {
    bandmatch_b200::Context small_ctx(hf, 10);
    DeviceArena small(10);
    report(code_of([&] { bandmatch_b200::execute_plan(small_ctx, plan, feats, hf, small, opts); }) ==
               "CapacityExceeded",
           "CapacityExceeded when the arena is too small");
  }
  std::printf("%s: %d failure(s)\n", failures ? "FAILED" : "OK", failures);
  return failures ? 1 : 0;
}
