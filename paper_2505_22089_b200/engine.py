"""Python mirror of bandmatch's executor surface (include/bandmatch/engine.hpp,
include/bandmatch/mbr.hpp): SchedulePlan + plan JSON (mbr.cpp:378-463),
DeviceArena counters, ``execute_plan`` (engine.cpp:411-527) whose row body runs
on the B200 through the C ABI (``bmg_execute_plan``).

The block scheduler itself stays on the host and is an *input* here: plans are
read from the reference's plan JSON.  Verification (SAO + RANSAC) stays on the
CPU: pass ``on_pair`` to receive every pair's initial matches as soon as they
are in host memory (the reference's VerifyPool hand-off, engine.cpp:478-479).
"""
from __future__ import annotations

import ctypes as C
from collections.abc import Sequence
import json
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import BandmatchError, check, ptr
from .hashmatch import FeatureSet, HashFunctions, Matcher, MatchParams, PairMatches

__all__ = ["ScheduleBlock", "BlockRow", "ScheduleIteration", "SchedulePlan", "read_plan",
           "write_plan", "plan_from_json", "DeviceArena", "ExecuteOptions", "IterationMetrics",
           "PipelineMetrics", "ExecutionResult", "execute_plan", "arena_units_for", "flatten_plan"]


@dataclass
class ScheduleBlock:
    row_chunk: int = 0
    col_chunk: int = 0
    row_images: list = field(default_factory=list)
    col_images: list = field(default_factory=list)
    pairs: list = field(default_factory=list)  # [(a, b)] with a < b


@dataclass
class BlockRow:
    row_chunk: int = 0
    row_images: list = field(default_factory=list)
    blocks: list = field(default_factory=list)
    evict_after: list = field(default_factory=list)

    def needed(self) -> list:
        """engine.cpp:434-436: row_images ∪ every block's col_images, ascending."""
        s = set(self.row_images)
        for b in self.blocks:
            s.update(b.col_images)
        return sorted(s)


@dataclass
class ScheduleIteration:
    dimension: int = 0
    bandwidth_before: int = 0
    bandwidth_after: int = 0
    rows: list = field(default_factory=list)

    def pair_count(self) -> int:
        return sum(len(b.pairs) for r in self.rows for b in r.blocks)


@dataclass
class SchedulePlan:
    strategy: str = ""
    size_blk: int = 0
    size_gpu: int = 0
    final_dimension: int = 0
    iterations: list = field(default_factory=list)

    def pair_count(self) -> int:
        return sum(it.pair_count() for it in self.iterations)

    def pairs(self) -> list:
        return sorted(tuple(p) for it in self.iterations for r in it.rows for b in r.blocks
                      for p in b.pairs)


def plan_from_json(j: dict) -> SchedulePlan:
    try:
        plan = SchedulePlan(j["strategy"], j["budget"]["size_blk"], j["budget"]["size_gpu"],
                            j["final_dimension"])
        for ji in j["iterations"]:
            it = ScheduleIteration(ji["dimension"], ji["bandwidth_before"], ji["bandwidth_after"])
            for jr in ji["rows"]:
                row = BlockRow(jr["row_chunk"], list(jr["row_images"]), [], list(jr["evict_after"]))
                for jb in jr["blocks"]:
                    row.blocks.append(ScheduleBlock(
                        jb["row_chunk"], jb["col_chunk"], list(jb["row_images"]),
                        list(jb["col_images"]),
                        [(min(a, b), max(a, b)) for a, b in jb["pairs"]]))
                it.rows.append(row)
            plan.iterations.append(it)
    except (KeyError, TypeError) as e:
        raise BandmatchError("FormatError", f"plan JSON missing fields: {e}")
    return plan


def read_plan(path) -> SchedulePlan:
    """read_plan, mbr.cpp:421-463."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for reading")
    except json.JSONDecodeError as e:
        raise BandmatchError("FormatError", f"invalid plan JSON in {path}: {e}")
    return plan_from_json(j)


def write_plan(path, plan: SchedulePlan, config_echo: str | None = None) -> None:
    """write_plan, mbr.cpp:378-419."""
    j = {}
    if config_echo is not None:
        j["config"] = json.loads(config_echo)
    j.update({"strategy": plan.strategy,
              "budget": {"size_blk": plan.size_blk, "size_gpu": plan.size_gpu},
              "final_dimension": plan.final_dimension, "iterations": []})
    for it in plan.iterations:
        ji = {"dimension": it.dimension, "bandwidth_before": it.bandwidth_before,
              "bandwidth_after": it.bandwidth_after, "rows": []}
        for r in it.rows:
            ji["rows"].append({"row_chunk": r.row_chunk, "row_images": r.row_images,
                               "evict_after": r.evict_after,
                               "blocks": [{"row_chunk": b.row_chunk, "col_chunk": b.col_chunk,
                                           "row_images": b.row_images, "col_images": b.col_images,
                                           "pairs": [list(p) for p in b.pairs]}
                                          for b in r.blocks]})
        j["iterations"].append(ji)
    with open(path, "w") as f:
        f.write(json.dumps(j, indent=2) + "\n")


@dataclass
class FlatPlan:
    """SchedulePlan flattened into the bmg_plan arrays (include/bandmatch_gpu.h)."""
    rows_per_iteration: np.ndarray
    row_needed_offsets: np.ndarray
    needed_ids: np.ndarray
    row_pair_offsets: np.ndarray
    pairs: np.ndarray
    row_evict_offsets: np.ndarray
    evict_ids: np.ndarray

    def c(self):
        return _lib.PlanC(len(self.rows_per_iteration), ptr(self.rows_per_iteration),
                          len(self.row_needed_offsets) - 1, ptr(self.row_needed_offsets),
                          ptr(self.needed_ids), ptr(self.row_pair_offsets), ptr(self.pairs),
                          ptr(self.row_evict_offsets), ptr(self.evict_ids))


def flatten_plan(plan: SchedulePlan, rows=None) -> FlatPlan:
    """Flatten (optionally only the rows with the given global indices, which
    keeps their iteration grouping -- used to shard rows across GPUs)."""
    rpi, nd_off, nd, p_off, prs, ev_off, ev = [], [0], [], [0], [], [0], []
    g = 0
    for it in plan.iterations:
        cnt = 0
        for r in it.rows:
            take = rows is None or g in rows
            g += 1
            if not take:
                continue
            cnt += 1
            nd.extend(r.needed())
            nd_off.append(len(nd))
            for b in r.blocks:
                for a, bb in b.pairs:
                    prs.extend((a, bb))
            p_off.append(len(prs) // 2)
            ev.extend(r.evict_after)
            ev_off.append(len(ev))
        rpi.append(cnt)
    u = lambda x: np.ascontiguousarray(x if len(x) else [0], np.uint64)
    return FlatPlan(u(rpi) if rpi else np.zeros(1, np.uint64)[:0].copy(), u(nd_off), u(nd),
                    u(p_off), u(prs), u(ev_off), u(ev))


class DeviceArena:
    """DeviceArena (engine.hpp:20-44) backed by a B200 context: capacity in
    descriptor units, uploads are real H2D copies into HBM."""

    def __init__(self, capacity_units: int, hf: HashFunctions, device: int = 0):
        self.matcher = Matcher(hf, capacity_units, device)

    def _s(self):
        return self.matcher.arena_stats()

    def capacity(self): return self._s()["capacity"]
    def occupancy(self): return self._s()["occupancy"]
    def peak_occupancy(self): return self._s()["peak_occupancy"]
    def uploads(self): return self._s()["uploads"]
    def evictions(self): return self._s()["evictions"]
    def units_uploaded(self): return self._s()["units_uploaded"]
    def resident_count(self): return self._s()["resident_count"]
    def resident(self, image_id): return self.matcher.resident(image_id)
    def upload(self, image_id, desc): self.matcher.upload(image_id, desc)
    def evict(self, image_id): self.matcher.evict(image_id)


@dataclass
class ExecuteOptions:
    match: MatchParams = field(default_factory=MatchParams)
    on_pair: object = None    # callable(query_image, train_image, matches (n,2) int32)
    on_upload: object = None  # DeviceBackend::on_upload(image_id, units)
    on_evict: object = None   # DeviceBackend::on_evict(image_id)
    retain: bool = False      # keep images resident (skip eviction directives)
    serial: bool = False      # all rows on one stream (kernel timing; same results)
    reproject: bool = False   # recompute resident images' projections in the call (timing)
    # row means: "exact" (parallel F96 reconstruction, the default) or
    # "chain" (the literal sequential FP64 chain; a test hook, same results)
    mean: str = "exact"

    def flags(self) -> int:
        modes = {"exact": 0, "chain": _lib.EXEC_MEAN_CHAIN}
        if self.mean not in modes:
            raise BandmatchError("InvalidArgument", f"unknown mean mode {self.mean!r}")
        return ((_lib.EXEC_RETAIN if self.retain else 0) | (_lib.EXEC_SERIAL if self.serial else 0)
                | (_lib.EXEC_REPROJECT if self.reproject else 0) | modes[self.mean])


@dataclass
class IterationMetrics:
    pairs: int = 0
    uploads: int = 0
    units_uploaded: int = 0


@dataclass
class PipelineMetrics:
    strategy: str = ""
    pairs_matched: int = 0
    initial_matches: int = 0
    verified_matches: int = 0
    uploads: int = 0
    evictions: int = 0
    units_uploaded: int = 0
    peak_occupancy: int = 0
    utilization_proxy: float = 0.0
    per_iteration: list = field(default_factory=list)
    wall_time_s: float = 0.0
    pairs_per_second: float = 0.0
    device_ms: float = 0.0  # CUDA-event span of the row loop on the compute stream


@dataclass
class ExecutionResult:
    matches: list
    metrics: PipelineMetrics
    outcomes: list = field(default_factory=list)
    # per plan row: (host ms when its pairs went to on_pair or -1, device ms
    # when its last kernel finished) -- the GPU / host-verification overlap
    row_timing: list = field(default_factory=list)


def arena_units_for(features: dict, gpu_images: int) -> int:
    """arena_units_for, engine.cpp:403-409."""
    largest = max((fs.size() for fs in features.values()), default=0)
    return largest * max(0, gpu_images)


def _is_path(x) -> bool:
    return isinstance(x, (str, bytes, os.PathLike))


def _feature_files(features: dict):
    """bmg_feature_file array for {id: path to a .feat file}."""
    L = _lib.load()
    files = (_lib.FeatureFileC * max(1, len(features)))()
    keep = []
    for i, (iid, path) in enumerate(features.items()):
        b = os.fsencode(path)
        keep.append(b)
        fid, n = C.c_uint64(0), C.c_uint64(0)
        check(L.bmg_read_features_header(b, C.byref(fid), C.byref(n)))
        files[i] = _lib.FeatureFileC(int(iid), b, n.value)
    return files, keep


def _feature_views(features: dict):
    if features and all(_is_path(v) for v in features.values()):
        return _feature_files(features)
    views = (_lib.FeatureViewC * max(1, len(features)))()
    keep = []
    for i, (iid, fs) in enumerate(features.items()):
        d = fs.descriptors if isinstance(fs, FeatureSet) else np.ascontiguousarray(fs, np.float32)
        keep.append(d)
        views[i] = _lib.FeatureViewC(int(iid), ptr(d) if d.size else None, d.shape[0])
    return views, keep


class _ResultBuffer:
    """Owns a bmg_result; numpy views of its pinned log keep it alive (the
    result is freed when the last view is garbage collected)."""

    def __init__(self, L, h):
        self.L, self.h = L, h

    def wrap(self, arr: np.ndarray) -> np.ndarray:
        # a base object that carries the owner: slices of `out` keep it alive
        out = np.ndarray(arr.shape, arr.dtype, buffer=_Owned(arr, self))
        out.flags.writeable = False
        return out

    def close(self):
        if self.h:
            self.L.bmg_result_free(self.h)
            self.h = None

    def __del__(self):
        self.close()


class _PairList(Sequence):
    """ExecutionResult.matches: PairMatches (sorted by IdPair) built on access
    from the result's pair ids, ranges and pinned match log."""

    _EMPTY = np.zeros((0, 2), np.int32)

    def __init__(self, ids, rng, log, holder=None):
        self._ids, self._rng, self._log, self._holder = ids, rng, log, holder

    def _write_bmmt(self, bpath: bytes):
        """write_matches_binary of the whole result from its pinned log."""
        if self._holder is None or not self._holder.h:
            raise BandmatchError("InvalidArgument", "result buffer already released")
        check(self._holder.L.bmg_result_write_matches(self._holder.h, bpath))

    def __len__(self):
        return len(self._ids) // 2

    def __getitem__(self, p):
        if isinstance(p, slice):
            return [self[i] for i in range(*p.indices(len(self)))]
        if p < 0:
            p += len(self)
        if not 0 <= p < len(self):
            raise IndexError(p)
        b, e = int(self._rng[2 * p]), int(self._rng[2 * p + 1])
        return PairMatches(int(self._ids[2 * p]), int(self._ids[2 * p + 1]),
                           self._log[b:e] if e > b else self._EMPTY)

    def __eq__(self, other):
        return list(self) == list(other)

    def flat(self):
        """(pair_ids [P,2] u64, offsets [P+1] u64, matches [M,2] i32): the
        result in IdPair order, matches concatenated (the layout of
        bmg_result_copy)."""
        ids = np.asarray(self._ids, np.uint64).reshape(-1, 2)
        rng = np.asarray(self._rng, np.int64).reshape(-1, 2)
        counts = rng[:, 1] - rng[:, 0]
        offs = np.zeros(len(counts) + 1, np.uint64)
        np.cumsum(counts, out=offs[1:])
        if self._log is None or not counts.sum():
            return ids, offs, np.zeros((0, 2), np.int32)
        parts = [self._log[b:e] for b, e in rng if e > b]
        return ids, offs, np.ascontiguousarray(np.concatenate(parts), np.int32)

    def __reduce__(self):
        return (list, (list(self),))


class _Owned:
    """Buffer-protocol wrapper around a ctypes-backed array + its owner."""

    def __init__(self, arr, owner):
        self.arr, self.owner = arr, owner

    def __buffer__(self, flags):
        return memoryview(self.arr)


def execute_plan(plan: SchedulePlan, features: dict, arena: DeviceArena,
                 opts: ExecuteOptions = ExecuteOptions(), rows=None, flat: FlatPlan | None = None,
                 views=None) -> ExecutionResult:
    """execute_plan (engine.cpp:411-527) with verification off: the row body
    (uploads, mean, codes, bucket tables, cascade matching) runs on the B200.
    Results are sorted by IdPair.  ``rows`` restricts execution to a subset of
    global row indices (multi-GPU sharding).  ``features`` maps image ids to
    FeatureSets / descriptor arrays (pinned or pageable host memory), or to
    paths of .feat files, which are then read as their images upload
    (bmg_execute_plan_files) instead of being loaded up front."""
    L = _lib.load()
    flat = flat or flatten_plan(plan, rows)
    views, keep = views or _feature_views(features)
    pc = flat.c()
    cbs = []

    def wrap(fn, ctype, conv):
        if fn is None:
            return ctype()
        cb = ctype(conv)
        cbs.append(cb)
        return cb

    on_pair = wrap(opts.on_pair, _lib.PAIR_CB,
                   lambda u, q, t, m, n: opts.on_pair(
                       q, t, np.ctypeslib.as_array(m, (2 * n,)).reshape(-1, 2).copy() if n else
                       np.zeros((0, 2), np.int32)))
    on_up = wrap(opts.on_upload, _lib.UPLOAD_HOOK, lambda u, i, n: opts.on_upload(i, n))
    on_ev = wrap(opts.on_evict, _lib.EVICT_HOOK, lambda u, i: opts.on_evict(i))
    oc = _lib.ExecOptionsC(opts.match.c(), on_pair, None, on_up, on_ev, None, opts.flags())
    h = C.c_void_p()
    run = L.bmg_execute_plan_files if isinstance(views, C.Array) and views._type_ is _lib.FeatureFileC \
        else L.bmg_execute_plan
    check(run(arena.matcher.handle, C.byref(pc), views, len(features), C.byref(oc), C.byref(h)))
    holder = _ResultBuffer(L, h)
    npairs = L.bmg_result_pair_count(h)
    nm = L.bmg_result_match_count(h)
    counters = np.zeros(6, np.uint64)
    wall = C.c_double(0)
    check(L.bmg_result_metrics(h, ptr(counters), C.byref(wall)))
    dev_ms = C.c_double(0)
    check(L.bmg_result_device_ms(h, C.byref(dev_ms)))
    its = []
    for i in range(L.bmg_result_iteration_count(h)):
        o = np.zeros(3, np.uint64)
        check(L.bmg_result_iteration(h, i, ptr(o)))
        its.append(IterationMetrics(int(o[0]), int(o[1]), int(o[2])))
    row_timing = []
    for r in range(len(flat.row_needed_offsets) - 1):
        o = np.zeros(2, np.float64)
        check(L.bmg_result_row_timing(h, r, ptr(o)))
        row_timing.append((float(o[0]), float(o[1])))
    matches = []
    if npairs:
        # zero-copy: every pair's (query_idx, train_idx) array is a view into
        # the result's pinned log, kept alive by the views themselves; the
        # PairMatches objects are made on access
        pid_p, rng_p, log_p = C.POINTER(C.c_uint64)(), C.POINTER(C.c_uint64)(), C.POINTER(C.c_int32)()
        check(L.bmg_result_view(h, C.byref(pid_p), C.byref(rng_p), C.byref(log_p)))
        ids = np.ctypeslib.as_array(pid_p, (2 * npairs,)).copy()
        rng = np.ctypeslib.as_array(rng_p, (2 * npairs,)).copy()
        top = int(rng[1::2].max()) if nm else 0
        log = holder.wrap(np.ctypeslib.as_array(log_p, (max(2 * top, 1),))).reshape(-1, 2) if top else None
        matches = _PairList(ids, rng, log, holder)
    else:
        holder.close()
    c = [int(x) for x in counters]
    met = PipelineMetrics(plan.strategy, c[0], c[1], 0, c[2], c[3], c[4], c[5],
                          c[0] / c[2] if c[2] else 0.0, its, wall.value,
                          c[0] / wall.value if wall.value > 0 else 0.0)
    met.device_ms = dev_ms.value
    del keep
    return ExecutionResult(matches, met, row_timing=row_timing)
