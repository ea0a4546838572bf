"""GPU matching overlapping host verification (north_star (5); the reference's
VerifyPool hand-off, engine.cpp:275-299, push at :479): execute_plan hands
each block row's pairs to on_pair from a collector thread as soon as that
row's matches are in host memory, while later rows still run on the GPU, and
a blocking consumer (backpressure) does not stall the GPU."""
import threading
import time

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import engine, multigpu

pytestmark = pytest.mark.gpu


def scene(reference, tmp_path, n=40, ppi=8192, band=5, blk=8, gpu=16):
    imgs, pairs = reference.generate_synthetic(n, ppi, band, 0.02, 0.2, 17)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(n), pairs, blk, gpu, plan_path)
    plan = bm.read_plan(plan_path)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    return plan, feats, hf


def test_rows_are_handed_over_while_later_rows_run(reference, tmp_path):
    plan, feats, hf = scene(reference, tmp_path)
    n_rows = sum(len(it.rows) for it in plan.iterations)
    assert n_rows >= 3
    got = []
    lock = threading.Lock()
    main = threading.get_ident()
    threads = set()

    def on_pair(q, t, m):
        with lock:
            got.append((q, t, m))
            threads.add(threading.get_ident())

    arena = bm.DeviceArena(engine.arena_units_for(feats, plan.size_gpu), hf)
    res = bm.execute_plan(plan, feats, arena, bm.ExecuteOptions(on_pair=on_pair))
    # every planned pair handed over exactly once, with the result's matches
    assert sorted((q, t) for q, t, _ in got) == plan.pairs()
    byp = {(q, t): m for q, t, m in got}
    for pm in res.matches:
        assert np.array_equal(byp[pm.query_image, pm.train_image], pm.matches)
    assert main not in threads  # the collector thread, not the caller's
    # the first row handed over before the last row's kernels finished
    timing = [t for t in res.row_timing if t[0] >= 0]
    assert len(timing) == n_rows
    first_handoff = min(h for h, _ in timing)
    last_done = max(d for _, d in timing)
    assert first_handoff < last_done - 0.2, res.row_timing


def test_blocking_consumer_does_not_stall_the_gpu(reference, tmp_path):
    """A consumer that blocks on the first pair (a full verification queue)
    only delays the hand-off: the GPU finishes every row meanwhile."""
    plan, feats, hf = scene(reference, tmp_path)
    state = {"first": True}

    def on_pair(q, t, m):
        if state["first"]:
            state["first"] = False
            time.sleep(0.5)

    arena = bm.DeviceArena(engine.arena_units_for(feats, plan.size_gpu), hf)
    res = bm.execute_plan(plan, feats, arena, bm.ExecuteOptions(on_pair=on_pair))
    first_handoff = min(h for h, _ in res.row_timing)
    last_done = max(d for _, d in res.row_timing)
    # all rows done on the device well before the blocked callback returned
    assert last_done < first_handoff + 400, res.row_timing
    assert res.metrics.wall_time_s >= 0.5


def test_results_unchanged_with_and_without_hand_off(reference, tmp_path):
    plan, feats, hf = scene(reference, tmp_path, n=24, ppi=3000)
    cap = engine.arena_units_for(feats, plan.size_gpu)
    a = bm.execute_plan(plan, feats, bm.DeviceArena(cap, hf))
    b = bm.execute_plan(plan, feats, bm.DeviceArena(cap, hf), bm.ExecuteOptions(on_pair=lambda *x: None))
    for x, y in zip(multigpu.result_flat(a), multigpu.result_flat(b)):
        assert np.array_equal(x, y)
