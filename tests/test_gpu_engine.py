"""GPU execute_plan (engine.cpp:411-527, verification off) against the
compiled reference's execute_plan on the same scene and MBR plan: identical
match lists per pair, identical arena counters (test_engine.cpp:265-324)."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import engine

pytestmark = pytest.mark.gpu


def run_both(reference, tmp_path, n_images, ppi, band, size_blk, size_gpu, seed=7, k=8,
             ratio=0.5, mean="exact"):
    imgs, pairs = reference.generate_synthetic(n_images, ppi, band, 0.02, 0.2, seed)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(n_images), pairs, size_blk, size_gpu, plan_path)
    plan = bm.read_plan(plan_path)
    hseed = bm.seed_for(42, "matching")
    hf = bm.make_hash_functions(hseed)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    cap = engine.arena_units_for(feats, size_gpu)
    ref, ref_counters, _ = reference.execute_plan(plan_path, dict(enumerate(imgs)), hseed,
                                                  k=k, ratio=ratio, capacity_units=cap)
    arena = bm.DeviceArena(cap, hf)
    ups, evs = [], []
    opts = bm.ExecuteOptions(bm.MatchParams(k, ratio), on_upload=lambda i, n: ups.append((i, n)),
                             on_evict=lambda i: evs.append(i), mean=mean)
    res = bm.execute_plan(plan, feats, arena, opts)
    return plan, ref, ref_counters, res, arena, ups, evs, feats


def test_band_block_plan_equals_reference(reference, tmp_path):
    plan, ref, rc, res, arena, ups, evs, feats = run_both(reference, tmp_path, 12, 600, 3, 3, 6)
    assert len(plan.iterations) >= 1
    got = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    assert list(got) == sorted(ref)
    for key, m in ref.items():
        assert np.array_equal(got[key], m), key
    met = res.metrics
    assert met.pairs_matched == rc["pairs_matched"]
    assert met.initial_matches == rc["initial_matches"]
    assert met.uploads == rc["uploads"] and met.evictions == rc["evictions"]
    assert met.units_uploaded == rc["units_uploaded"]
    assert met.peak_occupancy == rc["peak_occupancy"]
    assert len(ups) == met.uploads and len(evs) == met.evictions
    assert sum(n for _, n in ups) == met.units_uploaded
    assert arena.occupancy() == 0
    assert sum(it.pairs for it in met.per_iteration) == met.pairs_matched


@pytest.mark.parametrize("mean", ["exact", "chain"])
def test_config2_block_equals_reference(reference, tmp_path, mean):
    # BASELINE config 2 shape at reduced descriptor count: 32 images, band 11,
    # iterate_schedule(16, 32) -> 2 rows, 286 pairs.  Both row-mean paths
    # (parallel F96 reconstruction, literal FP64 chain) must give the
    # reference's lists.
    plan, ref, rc, res, *_ = run_both(reference, tmp_path, 32, 1024, 11, 16, 32,
                                      mean=mean)
    assert rc["pairs_matched"] == 286
    got = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    for key, m in ref.items():
        assert np.array_equal(got[key], m), key


def test_capacity_and_missing_image_errors(reference, tmp_path):
    imgs, pairs = reference.generate_synthetic(6, 50, 1, 0.02, 0.2, 3)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(6), pairs, 2, 4, plan_path)
    plan = bm.read_plan(plan_path)
    hf = bm.make_hash_functions(31)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    with pytest.raises(bm.BandmatchError) as e:
        bm.execute_plan(plan, feats, bm.DeviceArena(60, hf))
    assert e.value.code == "CapacityExceeded"
    del feats[3]
    with pytest.raises(bm.BandmatchError) as e:
        bm.execute_plan(plan, feats, bm.DeviceArena(10 ** 6, hf))
    assert e.value.code == "InvalidArgument"


def test_arena_semantics():
    hf = bm.make_hash_functions(5)
    a = bm.DeviceArena(10, hf)
    d = np.zeros((4, 128), np.float32)
    a.upload(1, d)
    a.upload(1, d)  # resident: no-op (engine.cpp:19)
    assert a.uploads() == 1 and a.occupancy() == 4
    with pytest.raises(bm.BandmatchError) as e:
        a.upload(2, np.zeros((7, 128), np.float32))
    assert e.value.code == "CapacityExceeded"
    a.evict(1)
    with pytest.raises(bm.BandmatchError) as e:
        a.evict(1)
    assert e.value.code == "NotResident"
    assert a.peak_occupancy() == 4 and a.evictions() == 1


def test_empty_plan_executes_to_zeros():
    hf = bm.make_hash_functions(1)
    res = bm.execute_plan(bm.SchedulePlan(), {}, bm.DeviceArena(0, hf))
    assert res.matches == [] and res.metrics.pairs_matched == 0 and res.metrics.uploads == 0


@pytest.mark.parametrize("flags", [dict(serial=True), dict(retain=True), dict(retain=True, reproject=True),
                                   dict(serial=True, reproject=True, retain=True)])
def test_execution_modes_give_identical_results(reference, tmp_path, flags):
    # rows on one stream (serial), images kept resident (retain), projections
    # recomputed in the call (reproject): all must reproduce the reference
    plan, ref, rc, res, arena, *_ = run_both(reference, tmp_path, 14, 700, 3, 3, 6, seed=11)
    feats = {i: bm.FeatureSet(i, d) for i, d in
             enumerate(reference.generate_synthetic(14, 700, 3, 0.02, 0.2, 11)[0])}
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    a2 = bm.DeviceArena(engine.arena_units_for(feats, 6) * 3, hf)
    for _ in range(2):  # the second call runs on whatever the first left resident
        r2 = bm.execute_plan(plan, feats, a2, bm.ExecuteOptions(**flags))
        got = {(pm.query_image, pm.train_image): pm.matches for pm in r2.matches}
        assert list(got) == sorted(ref)
        for key, m in ref.items():
            assert np.array_equal(got[key], m), key


def test_multi_iteration_plan_with_reuploads(reference, tmp_path):
    # a small arena forces several iterations, evictions and re-uploads of
    # images whose projections must be recomputed after each re-upload
    plan, ref, rc, res, arena, ups, evs, _ = run_both(reference, tmp_path, 20, 500, 4, 2, 4, seed=5)
    assert len(plan.iterations) >= 2 and rc["uploads"] > 20
    got = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    for key, m in ref.items():
        assert np.array_equal(got[key], m), key
    assert res.metrics.uploads == rc["uploads"] and arena.occupancy() == 0


def test_result_views_outlive_the_call(reference, tmp_path):
    # match arrays are zero-copy views of the result's pinned buffer; they
    # must stay valid (and unchanged) after later calls reuse the context
    plan, ref, rc, res, arena, *_ = run_both(reference, tmp_path, 12, 600, 3, 3, 6)
    saved = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    copies = {k: v.copy() for k, v in saved.items()}
    feats = {i: bm.FeatureSet(i, d) for i, d in
             enumerate(reference.generate_synthetic(12, 600, 3, 0.02, 0.2, 9)[0])}
    for _ in range(3):
        bm.execute_plan(plan, feats, arena)
    for k in saved:
        assert np.array_equal(saved[k], copies[k]), k


def test_rows_run_out_of_order_but_hooks_follow_the_plan(reference, tmp_path):
    # the device runs each iteration's rows fewest-uploads-first (band plans:
    # last row first); the arena's hooks and counters must still follow the
    # plan's row order (engine.cpp:438-444, 491-494), results unchanged
    plan, ref, rc, res, arena, ups, evs, feats = run_both(reference, tmp_path, 16, 400, 3, 4, 8, seed=13)
    assert any(len(it.rows) > 1 for it in plan.iterations)
    resident, exp_ups, exp_evs = set(), [], []
    for it in plan.iterations:
        for row in it.rows:
            for i in row.needed():
                if i not in resident:
                    resident.add(i)
                    exp_ups.append((i, len(feats[i].descriptors)))
            for i in row.evict_after:
                resident.discard(i)
                exp_evs.append(i)
    assert ups == exp_ups and evs == exp_evs
    got = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    for key, m in ref.items():
        assert np.array_equal(got[key], m), key
    assert res.metrics.peak_occupancy == rc["peak_occupancy"] and arena.occupancy() == 0


def test_result_match_file_byte_identical_to_reference(reference, tmp_path):
    # acceptance gate 10 (acceptance.cpp:718-761): matches.bin of the GPU
    # execute_plan, written natively from the result's pinned log, equals the
    # reference writer's file for the reference execute_plan's matches
    plan, ref, rc, res, *_ = run_both(reference, tmp_path, 14, 700, 3, 3, 6, seed=21)
    ours, theirs = tmp_path / "ours.bin", tmp_path / "theirs.bin"
    bm.write_matches_binary(ours, res.matches)
    reference.write_matches_binary(theirs, [(q, t, m) for (q, t), m in ref.items()])
    assert ours.read_bytes() == theirs.read_bytes()


def test_image_needed_again_after_its_eviction(reference, tmp_path):
    """Row 0 evicts image 0, row 1 of the same iteration needs it again and
    does not evict it: the reference's arena re-uploads it
    (counters and hooks), keeps it resident afterwards, and a second call
    starts from that state."""
    imgs, _ = reference.generate_synthetic(4, 500, 2, 0.02, 0.2, 5)
    B = bm.ScheduleBlock
    rows = [bm.BlockRow(0, [0], [B(0, 1, [0], [1], [(0, 1)])], [0]),
            bm.BlockRow(1, [0], [B(1, 2, [0], [2], [(0, 2)])], [])]
    plan = bm.SchedulePlan("custom", 2, 4, 4, [bm.ScheduleIteration(4, 0, 0, rows)])
    plan_path = tmp_path / "plan.json"
    bm.write_plan(plan_path, plan)
    hseed = bm.seed_for(42, "matching")
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    cap = 10 ** 6
    ref, rc, _ = reference.execute_plan(plan_path, dict(enumerate(imgs)), hseed, capacity_units=cap)
    arena = bm.DeviceArena(cap, bm.make_hash_functions(hseed))
    ups, evs = [], []
    opts = bm.ExecuteOptions(on_upload=lambda i, n: ups.append(i), on_evict=lambda i: evs.append(i))
    res = bm.execute_plan(plan, feats, arena, opts)
    met = res.metrics
    assert (met.uploads, met.evictions, met.units_uploaded, met.peak_occupancy) == (
        rc["uploads"], rc["evictions"], rc["units_uploaded"], rc["peak_occupancy"])
    assert ups == [0, 1, 0, 2] and evs == [0]
    assert all(arena.resident(i) for i in (0, 1, 2))
    assert arena.occupancy() == sum(len(imgs[i]) for i in (0, 1, 2))
    got = {(pm.query_image, pm.train_image): pm.matches for pm in res.matches}
    for key, m in ref.items():
        assert np.array_equal(got[key], m), key
    # second call: 0, 1, 2 resident -> row 0 uploads nothing, evicts 0; row 1
    # re-uploads 0
    ups.clear()
    evs.clear()
    res2 = bm.execute_plan(plan, feats, arena, opts)
    assert ups == [0] and evs == [0]
    assert res2.metrics.uploads == 5 and res2.metrics.evictions == 2
    for pm in res2.matches:
        assert np.array_equal(pm.matches, got[pm.query_image, pm.train_image])
    arena.evict(0)  # still resident in the arena: NotResident would be the bug
    assert not arena.resident(0)
