"""Multi-GPU execution of ONE SchedulePlan: its work shards across the GPUs of
one node with no collective on the data path.

Block rows are independent given the plan: a row's mean, codes and matches
depend only on its own resident image set (engine.cpp:433-465), and a pair's
matches only on the row's codes of its two images (engine.cpp:467-472).  So
each iteration's pair sequence (rows in plan order, pairs in block order) is
cut into `world` contiguous pieces balanced by a cost model -- one unit per
pair plus `prep_weight` units per needed image of every row a piece touches
(a rank that takes part of a row computes that row's mean, codes and bucket
tables itself: they are bit-identical on every GPU) -- and each rank runs the
sub-plan of its piece through the single-GPU executor.  A row split between
ranks keeps all of its blocks on every rank (blocks outside the rank's range
keep their images and lose their pairs), so its needed set -- and hence its
mean -- is unchanged.  Eviction directives are recomputed per rank the way
generate_blocks derives them (mbr.cpp:299-317): each arena holds what its
later rows still need and ends every iteration empty.  Iterations stay
barriers (engine.cpp:497-499).

The only communication is the final gather of the match lists to rank 0,
through shared memory (one node): each rank writes its result -- already in
IdPair order -- into a /dev/shm segment, rank 0 maps the segments and orders
the pairs by IdPair (results are keyed by pair, engine.cpp:419, 506-512);
match lists are not copied or pickled.
"""
from __future__ import annotations

import os
import tempfile
from collections.abc import Sequence

import numpy as np

from .engine import (BlockRow, DeviceArena, ExecuteOptions, ExecutionResult, IterationMetrics,
                     PipelineMetrics, ScheduleBlock, ScheduleIteration, SchedulePlan, execute_plan)
from .hashmatch import HashFunctions, PairMatches

__all__ = ["shard_plan", "needed_images", "execute_plan_distributed", "gather_results",
           "result_flat", "FlatPairs", "GatheredPairs"]

# cost of one needed image of a row (mean + codes + bucket tables) in units of
# one pair's matching, measured on the B200 (block32: 0.67 ms of row prep for
# 48 image-rows vs 2.03 ms of matching for 286 pairs)
PREP_WEIGHT = 2.0


def _pieces(costs_pairs: list, row_needed: list, world: int, prep_weight: float) -> list:
    """Cut one iteration's pair sequence into <= world contiguous pieces:
    returns [(row, first pair, end pair)] per piece.  costs_pairs[r] = pairs
    of row r.  Binary search on the largest piece cost; a piece is filled
    greedily (a piece's cost only grows as it extends, so greedy filling is
    optimal for a given cap)."""
    total_pairs = sum(costs_pairs)
    if total_pairs == 0:
        return [[] for _ in range(world)]

    def fill(cap):
        pieces, cur, cost, touched = [], [], 0.0, set()
        for r, n in enumerate(costs_pairs):
            p = 0
            while p < n:
                add_row = 0.0 if r in touched else prep_weight * row_needed[r]
                room = cap - cost - add_row
                if room < 1.0:
                    if not cur:
                        return None  # a single pair plus its row does not fit
                    pieces.append(cur)
                    cur, cost, touched = [], 0.0, set()
                    continue
                take = min(n - p, int(room))
                cur.append((r, p, p + take))
                cost += add_row + take
                touched.add(r)
                p += take
        if cur:
            pieces.append(cur)
        return pieces

    lo = max(1.0, prep_weight * max((row_needed[r] for r, n in enumerate(costs_pairs) if n), default=0) + 1)
    hi = float(total_pairs) + prep_weight * sum(row_needed) + 1.0
    best = fill(hi)
    for _ in range(60):
        if hi - lo <= 0.5:
            break
        mid = (lo + hi) / 2
        got = fill(mid)
        if got is not None and len(got) <= world:
            best, hi = got, mid
        else:
            lo = mid
    best = best + [[] for _ in range(world - len(best))]
    return best


def _local_evictions(rows: list) -> list:
    needed = [set(r.needed()) for r in rows]
    resident: set = set()
    out = []
    for t, r in enumerate(rows):
        resident |= needed[t]
        later = set().union(*needed[t + 1:]) if t + 1 < len(rows) else set()
        ev = sorted(x for x in resident if x not in later)
        resident -= set(ev)
        out.append(BlockRow(r.row_chunk, list(r.row_images), r.blocks, ev))
    return out


def shard_plan(plan: SchedulePlan, world: int, prep_weight: float = PREP_WEIGHT) -> list:
    """One sub-plan per rank; together they cover every planned pair exactly
    once, with every row's needed set (so its mean and codes) unchanged."""
    subs = [SchedulePlan(plan.strategy, plan.size_blk, plan.size_gpu, plan.final_dimension)
            for _ in range(world)]
    for it in plan.iterations:
        pairs_of = [[p for b in r.blocks for p in b.pairs] for r in it.rows]
        pieces = _pieces([len(x) for x in pairs_of], [len(r.needed()) for r in it.rows], world,
                         prep_weight)
        for rank in range(world):
            rows = []
            for r, p0, p1 in pieces[rank]:
                row = it.rows[r]
                blocks, k = [], 0
                for b in row.blocks:
                    lo, hi = max(p0 - k, 0), min(p1 - k, len(b.pairs))
                    blocks.append(ScheduleBlock(b.row_chunk, b.col_chunk, b.row_images, b.col_images,
                                                list(b.pairs[lo:hi]) if hi > lo else []))
                    k += len(b.pairs)
                rows.append(BlockRow(row.row_chunk, list(row.row_images), blocks, []))
            subs[rank].iterations.append(ScheduleIteration(it.dimension, it.bandwidth_before,
                                                           it.bandwidth_after, _local_evictions(rows)))
    return subs


def needed_images(plan: SchedulePlan) -> set:
    """Every image any row of the plan needs (what a rank must load)."""
    return {i for it in plan.iterations for r in it.rows for i in r.needed()}


class FlatPairs(Sequence):
    """A result's pairs as flat arrays (IdPair order): pair_ids [P,2] u64,
    offsets [P+1] u64, matches [M,2] i32; PairMatches made on access."""

    def __init__(self, ids, offs, matches):
        self.ids, self.offs, self.m = ids, offs, matches

    def __len__(self):
        return len(self.ids)

    def __getitem__(self, p):
        if isinstance(p, slice):
            return [self[i] for i in range(*p.indices(len(self)))]
        if p < 0:
            p += len(self)
        if not 0 <= p < len(self):
            raise IndexError(p)
        return PairMatches(int(self.ids[p, 0]), int(self.ids[p, 1]),
                           self.m[int(self.offs[p]):int(self.offs[p + 1])])

    def flat(self):
        return self.ids, self.offs, self.m


def result_flat(res: ExecutionResult):
    """(pair_ids, offsets, matches) of a result in IdPair order."""
    if hasattr(res.matches, "flat"):
        return res.matches.flat()
    pms = sorted(res.matches, key=lambda pm: (pm.query_image, pm.train_image))
    ids = np.array([(pm.query_image, pm.train_image) for pm in pms], np.uint64).reshape(-1, 2)
    counts = [len(pm.matches) for pm in pms]
    offs = np.zeros(len(pms) + 1, np.uint64)
    np.cumsum(counts, out=offs[1:])
    m = (np.ascontiguousarray(np.concatenate([np.asarray(pm.matches, np.int32).reshape(-1, 2)
                                              for pm in pms]))
         if pms and sum(counts) else np.zeros((0, 2), np.int32))
    return ids, offs, m


def _shm_dir() -> str:
    return "/dev/shm" if os.path.isdir("/dev/shm") and os.access("/dev/shm", os.W_OK) \
        else tempfile.gettempdir()


class GatheredPairs(Sequence):
    """Rank 0's view of the gathered result: pairs in IdPair order, each
    pair's matches a slice of the shared-memory segment its rank wrote
    (mapped, not copied).  ``flat()`` materialises the canonical arrays."""

    def __init__(self, ids, seg_of, begin, end, segs):
        self.ids, self._seg, self._b, self._e, self._segs = ids, seg_of, begin, end, segs

    def __len__(self):
        return len(self.ids)

    def __getitem__(self, p):
        if isinstance(p, slice):
            return [self[i] for i in range(*p.indices(len(self)))]
        if p < 0:
            p += len(self)
        if not 0 <= p < len(self):
            raise IndexError(p)
        m = self._segs[self._seg[p]][self._b[p]:self._e[p]]
        return PairMatches(int(self.ids[p, 0]), int(self.ids[p, 1]), m)

    def flat(self):
        counts = (self._e - self._b).astype(np.int64)
        offs = np.zeros(len(self.ids) + 1, np.uint64)
        np.cumsum(counts, out=offs[1:])
        parts = [self._segs[s][b:e] for s, b, e in zip(self._seg, self._b, self._e) if e > b]
        m = np.ascontiguousarray(np.concatenate(parts), np.int32) if parts else np.zeros((0, 2), np.int32)
        return self.ids, offs, m


def gather_results(res: ExecutionResult, rank: int, world: int, barrier, tag: str):
    """Gathers every rank's match lists to rank 0 through shared memory (one
    node): each rank writes its result -- pair ids, offsets, matches, in
    IdPair order -- into a /dev/shm segment with one write per array; rank
    0 maps the segments (no copy) and orders the pairs by IdPair.
    `barrier()` synchronises the ranks (torch.distributed).  Returns
    (GatheredPairs, [per-rank metrics]) on rank 0, None elsewhere."""
    import pickle  # metrics only (a few integers per rank)

    ids, offs, m = result_flat(res)
    path = os.path.join(_shm_dir(), f"bmg_gather_{tag}_{rank}")
    met = pickle.dumps(res.metrics)
    hdr = np.array([len(ids), len(m), len(met)], np.uint64)
    with open(path, "wb") as f:
        for arr in (hdr, np.ascontiguousarray(ids, np.uint64), np.ascontiguousarray(offs, np.uint64),
                    np.ascontiguousarray(m, np.int32)):
            f.write(memoryview(arr).cast("B"))
        f.write(met)
    barrier()
    out = None
    if rank == 0:
        all_ids, all_b, all_e, all_seg, segs, mets = [], [], [], [], [], []
        for r in range(world):
            p = os.path.join(_shm_dir(), f"bmg_gather_{tag}_{r}")
            raw = np.memmap(p, np.uint8, mode="r")
            P, M, K = (int(x) for x in raw[:24].view(np.uint64))
            o = 24
            ids_r = raw[o:o + 16 * P].view(np.uint64).reshape(-1, 2)
            o += 16 * P
            offs_r = raw[o:o + 8 * (P + 1)].view(np.uint64).astype(np.int64)
            o += 8 * (P + 1)
            segs.append(raw[o:o + 8 * M].view(np.int32).reshape(-1, 2))
            o += 8 * M
            mets.append(pickle.loads(bytes(raw[o:o + K])))
            all_ids.append(ids_r)
            all_b.append(offs_r[:-1])
            all_e.append(offs_r[1:])
            all_seg.append(np.full(P, r, np.int32))
        ids = np.concatenate(all_ids)
        order = np.lexsort((ids[:, 1], ids[:, 0]))
        out = (GatheredPairs(np.ascontiguousarray(ids[order]), np.concatenate(all_seg)[order],
                             np.concatenate(all_b)[order], np.concatenate(all_e)[order], segs), mets)
    barrier()
    os.unlink(path)  # rank 0's mappings stay valid
    return out


def merge_metrics(mets: list, strategy: str = "") -> PipelineMetrics:
    """Per-rank PipelineMetrics summed (uploads/evictions/peak are per-device
    arena figures; wall and device time are the max over ranks)."""
    met = PipelineMetrics(strategy)
    n_it = max((len(m.per_iteration) for m in mets), default=0)
    its = [IterationMetrics() for _ in range(n_it)]
    for m in mets:
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
    return met


def execute_plan_distributed(plan: SchedulePlan, features: dict, hf: HashFunctions | None = None,
                             capacity_units: int = 0, opts: ExecuteOptions = ExecuteOptions(),
                             device: int | None = None, executor=None, arena: DeviceArena | None = None,
                             tag: str = "plan"):
    """Run `plan` across the ranks of the default torch.distributed group
    (one process per GPU; several ranks may share a device).  `features`
    needs only the images of this rank's shard (needed_images(shard_plan(
    plan, world)[rank])).  Returns the merged ExecutionResult on rank 0 and
    None elsewhere.  `executor(sub_plan, features)` replaces the GPU row loop
    (tests inject a CPU stand-in)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    sub = shard_plan(plan, world)[rank]
    if executor is None:
        if arena is None:
            arena = DeviceArena(capacity_units, hf, rank if device is None else device)
        res = execute_plan(sub, features, arena, opts)
    else:
        res = executor(sub, features)
    got = gather_results(res, rank, world, dist.barrier, tag)
    if rank != 0:
        return None
    pairs, mets = got
    return ExecutionResult(pairs, merge_metrics(mets, plan.strategy))
