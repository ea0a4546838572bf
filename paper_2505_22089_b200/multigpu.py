"""Multi-GPU execution of one SchedulePlan: block rows shard across the GPUs of
one node with no collective on the data path.

Rows are independent given the plan: a row's mean, codes and matches depend
only on its own resident image set (engine.cpp:433-465), so each rank takes a
contiguous, pair-balanced range of every iteration's rows, uploads what its
rows need into its own HBM arena, and its matches go D2H on that rank.  The
only communication is the final gather of match lists to rank 0 (host
objects; the reference keys results by IdPair, engine.cpp:419, so the merge is
order-independent).  Iterations stay barriers, as in the reference
(engine.cpp:497-499), because an iteration's plan covers the pairs the
previous one left.
"""
from __future__ import annotations

from dataclasses import replace

from .engine import (BlockRow, DeviceArena, ExecuteOptions, ExecutionResult, IterationMetrics,
                     PipelineMetrics, ScheduleIteration, SchedulePlan, execute_plan)
from .hashmatch import HashFunctions, PairMatches

__all__ = ["partition_rows", "local_plan", "execute_plan_distributed", "merge_results"]


def partition_rows(plan: SchedulePlan, world: int) -> list[set[int]]:
    """Global row indices per rank: each iteration's rows are cut into `world`
    contiguous ranges with balanced pair counts (MBR order keeps neighbouring
    rows -- which share images -- on the same GPU)."""
    out = [set() for _ in range(world)]
    g = 0
    for it in plan.iterations:
        weights = [sum(len(b.pairs) for b in r.blocks) for r in it.rows]
        total = sum(weights)
        acc, rank = 0, 0
        for w in weights:
            # advance to the next rank once this one holds its share
            while rank < world - 1 and acc >= total * (rank + 1) / world:
                rank += 1
            out[rank].add(g)
            acc += w
            g += 1
    return out


def local_plan(plan: SchedulePlan, rows: set[int]) -> SchedulePlan:
    """The rank's sub-plan: its rows, with eviction directives recomputed the
    way generate_blocks does (mbr.cpp:299-317) so the local arena holds only
    what its later rows still need and ends every iteration empty."""
    lp = SchedulePlan(plan.strategy, plan.size_blk, plan.size_gpu, plan.final_dimension)
    g = 0
    for it in plan.iterations:
        mine = []
        for r in it.rows:
            if g in rows:
                mine.append(r)
            g += 1
        needed = [set(r.needed()) for r in mine]
        resident: set = set()
        new_rows = []
        for t, r in enumerate(mine):
            resident |= needed[t]
            later = set().union(*needed[t + 1:]) if t + 1 < len(mine) else set()
            ev = sorted(x for x in resident if x not in later)
            resident -= set(ev)
            new_rows.append(BlockRow(r.row_chunk, list(r.row_images), list(r.blocks), ev))
        lp.iterations.append(ScheduleIteration(it.dimension, it.bandwidth_before,
                                               it.bandwidth_after, new_rows))
    return lp


def merge_results(parts: list[ExecutionResult], strategy: str = "") -> ExecutionResult:
    """Merge per-rank results: pairs sorted by IdPair, counters summed
    (uploads/evictions/peak are per-device arena figures)."""
    by_pair: dict = {}
    met = PipelineMetrics(strategy)
    n_it = max((len(p.metrics.per_iteration) for p in parts), default=0)
    its = [IterationMetrics() for _ in range(n_it)]
    for p in parts:
        for pm in p.matches:
            by_pair[(pm.query_image, pm.train_image)] = pm
        m = p.metrics
        met.pairs_matched += m.pairs_matched
        met.initial_matches += m.initial_matches
        met.uploads += m.uploads
        met.evictions += m.evictions
        met.units_uploaded += m.units_uploaded
        met.peak_occupancy = max(met.peak_occupancy, m.peak_occupancy)
        met.wall_time_s = max(met.wall_time_s, m.wall_time_s)
        met.device_ms = max(met.device_ms, m.device_ms)
        for i, im in enumerate(m.per_iteration):
            its[i].pairs += im.pairs
            its[i].uploads += im.uploads
            its[i].units_uploaded += im.units_uploaded
    met.per_iteration = its
    met.utilization_proxy = met.pairs_matched / met.uploads if met.uploads else 0.0
    met.pairs_per_second = met.pairs_matched / met.wall_time_s if met.wall_time_s > 0 else 0.0
    return ExecutionResult([by_pair[k] for k in sorted(by_pair)], met)


def execute_plan_distributed(plan: SchedulePlan, features: dict, hf: HashFunctions,
                             capacity_units: int, opts: ExecuteOptions = ExecuteOptions(),
                             device: int | None = None, executor=None):
    """Run `plan` across the ranks of the default torch.distributed group
    (one process per GPU).  Returns the merged ExecutionResult on rank 0 and
    the rank-local one elsewhere.  `executor(sub_plan, features)` replaces the
    GPU row loop (tests inject a CPU stand-in to exercise the sharding)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    sub = local_plan(plan, partition_rows(plan, world)[rank])
    if executor is None:
        if device is None:
            device = rank
        arena = DeviceArena(capacity_units, hf, device)
        res = execute_plan(sub, features, arena, opts)
    else:
        res = executor(sub, features)
    payload = ([(pm.query_image, pm.train_image, pm.matches) for pm in res.matches], res.metrics)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0)
    if rank != 0:
        return res
    parts = [ExecutionResult([PairMatches(q, t, m) for q, t, m in pl], met) for pl, met in gathered]
    return merge_results(parts, plan.strategy)
