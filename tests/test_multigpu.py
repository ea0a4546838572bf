"""Row sharding across ranks on CPU: world_size-2 gloo groups run
execute_plan_distributed with the C oracle standing in for the GPU row loop;
the merged result must equal the single-process execution of the whole plan."""
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
    res = multigpu.execute_plan_distributed(plan, feats, None, 0,
                                            executor=oracle_executor(o, coarse, fine))
    if rank == 0:
        queue.put([(pm.query_image, pm.train_image, pm.matches.tolist()) for pm in res.matches])
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_is_exact_cover_and_balanced(reference, tmp_path):
    feats, plan = scene(reference, tmp_path)
    n_rows = sum(len(it.rows) for it in plan.iterations)
    for world in (1, 2, 3, 8):
        parts = multigpu.partition_rows(plan, world)
        assert sorted(x for p in parts for x in p) == list(range(n_rows))
        for p in parts:
            sub = multigpu.local_plan(plan, p)
            for it in sub.iterations:
                held = set()
                for r in it.rows:
                    held |= set(r.needed())
                    held -= set(r.evict_after)
                assert not held
        covered = sorted(pr for p in parts for pr in multigpu.local_plan(plan, p).pairs())
        assert covered == plan.pairs()


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
    for (a, b, m), pm in zip(got, single.matches):
        assert np.array_equal(np.array(m, np.int32).reshape(-1, 2), pm.matches)
