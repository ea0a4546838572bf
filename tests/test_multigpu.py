"""Sharding one plan across ranks on CPU: world_size-2 gloo groups
run execute_plan_distributed with the C oracle standing in for the GPU row loop
(the GPU branch is covered by tests/test_gpu_parity.py); the merged result --
gathered through shared memory -- must equal the single-process execution of
the whole plan."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import multigpu
from paper_2505_22089_b200.engine import ExecutionResult, IterationMetrics, PipelineMetrics


def oracle_executor(oracle, coarse, fine):
    """Test double for the GPU row loop: the restated reference row body."""
    def run(plan, features):
        out, met = {}, PipelineMetrics(plan.strategy)
        resident = set()
        for it in plan.iterations:
            im = IterationMetrics()
            for row in it.rows:
                needed = row.needed()
                for i in needed:
                    if i not in resident:
                        resident.add(i)
                        met.uploads += 1
                        im.uploads += 1
                mean = oracle.row_mean([features[i].descriptors for i in needed])
                codes = {i: oracle.compute_codes(features[i].descriptors, coarse, fine, mean)
                         for i in needed}
                for b in row.blocks:
                    for a, c in b.pairs:
                        out[(a, c)] = oracle.match_pair(features[a].descriptors, codes[a],
                                                        features[c].descriptors, codes[c],
                                                        (6, 8, 128))
                        im.pairs += 1
                for i in row.evict_after:
                    resident.discard(i)
                    met.evictions += 1
            met.per_iteration.append(im)
        assert not resident, "local plan must leave the arena empty"
        met.pairs_matched = len(out)
        met.initial_matches = sum(len(v) for v in out.values())
        return ExecutionResult([bm.PairMatches(a, c, m) for (a, c), m in sorted(out.items())], met)
    return run


def scene(reference, tmp_path):
    imgs, pairs = reference.generate_synthetic(14, 120, 3, 0.02, 0.2, 5)
    path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(14), pairs, 2, 5, path)
    return {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}, bm.read_plan(path)


def _worker(rank, world, port, feats, plan, queue):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from oracle_lib import Oracle
    o = Oracle()
    coarse, fine = o.make_hash_functions(o.seed_for(42, "matching"))
    sub = multigpu.shard_plan(plan, world)[rank]
    mine = {i: feats[i] for i in multigpu.needed_images(sub)}  # only this rank's images
    res = multigpu.execute_plan_distributed(plan, mine, None, 0,
                                            executor=oracle_executor(o, coarse, fine),
                                            tag=f"test{port}")
    if rank == 0:
        queue.put([(pm.query_image, pm.train_image, np.asarray(pm.matches).tolist())
                   for pm in res.matches])
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shards_cover_every_pair_once_with_rows_unchanged(reference, tmp_path):
    feats, plan = scene(reference, tmp_path)
    row_needed = {}
    for it in plan.iterations:
        for r in it.rows:
            row_needed[r.row_chunk, tuple(r.row_images)] = r.needed()
    for world in (1, 2, 3, 8, 40):
        subs = multigpu.shard_plan(plan, world)
        assert len(subs) == world
        covered = sorted(pr for s in subs for pr in s.pairs())
        assert covered == plan.pairs()  # exactly once
        for s in subs:
            assert len(s.iterations) == len(plan.iterations)  # iterations stay barriers
            for it in s.iterations:
                held = set()
                for r in it.rows:
                    # a (part of a) row keeps its whole needed set: same mean and codes
                    assert r.needed() == row_needed[r.row_chunk, tuple(r.row_images)]
                    held |= set(r.needed())
                    held -= set(r.evict_after)
                assert not held  # every rank's arena ends each iteration empty


def test_shard_balance_on_the_bench_plans():
    from pathlib import Path
    root = Path(__file__).resolve().parents[1] / "bench_data"
    for f in ("plan_strip500.json", "plan_shard16k.json", "plan_block32.json"):
        plan = bm.read_plan(root / f)
        for world in (2, 4, 8):
            subs = multigpu.shard_plan(plan, world)
            cost = [sum(len(b.pairs) for it in s.iterations for r in it.rows for b in r.blocks)
                    + multigpu.PREP_WEIGHT * sum(len(r.needed()) for it in s.iterations for r in it.rows)
                    for s in subs]
            # no rank far above the mean (prep of shared rows is duplicated)
            assert max(cost) <= 1.25 * (sum(cost) / world) + 1, (f, world, cost)
            assert sorted(p for s in subs for p in s.pairs()) == plan.pairs()


def test_weak_scaled_strips_give_every_rank_a_strip500_share():
    """bench.py --gpus N (strip500, --scaling weak): the 500 N-image strip's
    shards each carry about the one-GPU strip500 work (pairs and image-rows)."""
    import importlib.util
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    spec = importlib.util.spec_from_file_location("bench", root / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    one = bm.read_plan(root / "bench_data" / "plan_strip500.json")
    one_pairs = one.pair_count()
    one_rows = sum(len(r.needed()) for it in one.iterations for r in it.rows)
    assert bench.resolve_config("strip500", 1, "weak")[4:] == ("plan_strip500.json", "weak")
    assert bench.resolve_config("strip500", 2, "strong")[4:] == ("plan_strip500.json", "strong")
    assert bench.resolve_config("block32", 4, "weak")[5] == "strong"
    for world in (2, 4, 8):
        n_cfg, _, band, drop, f, lab = bench.resolve_config("strip500", world, "weak")
        assert lab == "weak" and n_cfg == 500 * world + drop and band == 10
        plan = bm.read_plan(root / "bench_data" / f)
        assert len({i for it in plan.iterations for r in it.rows for i in r.needed()}) == 500 * world
        subs = multigpu.shard_plan(plan, world)
        one_cost = one_pairs + multigpu.PREP_WEIGHT * one_rows
        for s in subs:
            img_rows = sum(len(r.needed()) for it in s.iterations for r in it.rows)
            assert 0.9 * one_pairs <= s.pair_count() <= 1.1 * one_pairs
            # a row split between ranks repeats its prep on both (~1.2x the cost model's work)
            assert s.pair_count() + multigpu.PREP_WEIGHT * img_rows <= 1.25 * one_cost
        assert sorted(p for s in subs for p in s.pairs()) == plan.pairs()


def test_shared_memory_gather_merges_by_idpair(tmp_path):
    """gather_results in one process with a fake 3-rank barrier schedule:
    each 'rank' writes its IdPair-sorted result; rank 0's merge is the union
    in IdPair order."""
    rng = np.random.default_rng(1)
    parts = []
    for r in range(3):
        pms = []
        for k in range(4):
            a = int(rng.integers(0, 50))
            m = rng.integers(0, 100, (int(rng.integers(0, 5)), 2)).astype(np.int32)
            pms.append(bm.PairMatches(a, 100 + 10 * k + r, m))
        parts.append(ExecutionResult(sorted(pms, key=lambda p: (p.query_image, p.train_image)),
                                     PipelineMetrics(pairs_matched=4)))
    # ranks 1, 2 write first (their barrier is a no-op here), then rank 0 merges
    import threading
    ev = threading.Barrier(3)
    out = {}

    def run(r):
        out[r] = multigpu.gather_results(parts[r], r, 3, ev.wait, "unit")
    ts = [threading.Thread(target=run, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    gathered, mets = out[0]
    ids, offs, m = gathered.flat()
    assert out[1] is None and out[2] is None
    assert [(pm.query_image, pm.train_image) for pm in gathered] == [tuple(map(int, x)) for x in ids]
    want = sorted((pm.query_image, pm.train_image, pm.matches.tolist()) for p in parts for pm in p.matches)
    got = [(int(ids[i, 0]), int(ids[i, 1]), m[offs[i]:offs[i + 1]].tolist()) for i in range(len(ids))]
    assert got == want
    assert sum(x.pairs_matched for x in mets) == 12


def test_two_rank_gloo_execution_equals_single_process(reference, oracle, tmp_path):
    feats, plan = scene(reference, tmp_path)
    coarse, fine = oracle.make_hash_functions(oracle.seed_for(42, "matching"))
    single = oracle_executor(oracle, coarse, fine)(plan, feats)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, feats, plan, q))
             for port in [free_port()] for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [(a, b) for a, b, _ in got] == [(pm.query_image, pm.train_image) for pm in single.matches]
    assert len(got) == len(plan.pairs())
    for (a, b, m), pm in zip(got, single.matches):
        assert np.array_equal(np.array(m, np.int32).reshape(-1, 2), pm.matches)
