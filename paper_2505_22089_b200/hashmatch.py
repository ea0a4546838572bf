"""Python mirror of bandmatch's hashmatch API (include/bandmatch/hashmatch.hpp),
running on the B200 through the C ABI.

Same names, argument meaning and error behaviour as the reference:
``make_hash_functions`` (hashmatch.cpp:53-69), ``compute_codes`` (:71-100),
``match_pair`` (:102-211), the BMMT/text match files (:254-363).  Errors raise
``BandmatchError`` carrying the reference's stable code ("HashMismatch",
"InvalidArgument", ...).
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import DIM, BandmatchError, check, ptr

__all__ = [
    "HashParams", "HashFunctions", "HashCodeSet", "MatchParams", "PairMatches", "Matcher",
    "make_hash_functions", "compute_codes", "match_pair", "seed_for", "FeatureSet",
    "write_matches_binary", "read_matches_binary", "write_matches_text", "read_matches_text",
]


@dataclass(frozen=True)
class HashParams:
    """HashParams, hashmatch.hpp:11-15."""
    tables: int = 6
    coarse_bits: int = 8
    fine_bits: int = 128

    @property
    def fine_words(self) -> int:
        return (self.fine_bits + 63) // 64

    def c(self):
        return _lib.HashParamsC(self.tables, self.coarse_bits, self.fine_bits)


@dataclass
class HashFunctions:
    """HashFunctions, hashmatch.hpp:19-34: coarse [tables][bits][128], fine [bits][128]."""
    params: HashParams
    seed: int
    coarse: np.ndarray
    fine: np.ndarray


@dataclass
class FeatureSet:
    """FeatureSet, features.hpp:47-53 (descriptors float32 [n][128]; keypoints
    [n][4] = x, y, scale, orientation, used only by host-side verification)."""
    image_id: int
    descriptors: np.ndarray
    keypoints: np.ndarray | None = None

    def __post_init__(self):
        self.descriptors = np.ascontiguousarray(self.descriptors, dtype=np.float32).reshape(-1, DIM)

    def size(self) -> int:
        return int(self.descriptors.shape[0])

    __len__ = size


@dataclass
class HashCodeSet:
    """HashCodeSet, hashmatch.hpp:36-56."""
    image_id: int
    function_seed: int
    params: HashParams
    count: int
    coarse: np.ndarray  # uint32 [count][tables]
    fine: np.ndarray    # uint64 [count][fine_words]

    @property
    def fine_words(self) -> int:
        return self.params.fine_words

    def bucket(self, feature: int, table: int) -> int:
        return int(self.coarse[feature, table])

    def fine_code(self, feature: int) -> np.ndarray:
        return self.fine[feature]

    def size_bytes(self) -> int:
        return self.coarse.size * 4 + self.fine.size * 8

    def c(self):
        return _lib.CodeSetC(self.image_id, self.function_seed, self.params.c(), self.count,
                             ptr(self.coarse) if self.count else None,
                             ptr(self.fine) if self.count else None)


@dataclass(frozen=True)
class MatchParams:
    """MatchParams, hashmatch.hpp:77-80."""
    k_nearest: int = 8
    ratio: float = 0.5

    def c(self):
        return _lib.MatchParamsC(self.k_nearest, self.ratio)


@dataclass
class PairMatches:
    """PairMatches, hashmatch.hpp:70-75: (query_idx, train_idx), unique query_idx."""
    query_image: int = 0
    train_image: int = 0
    matches: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.int32))
    stage: str = "initial"  # "initial" | "verified"

    def as_list(self):
        return [tuple(map(int, m)) for m in self.matches]


def seed_for(root: int, stage: str) -> int:
    """seed_for, common.hpp:38-45."""
    return int(_lib.load().bmg_seed_for(root, stage.encode()))


def make_hash_functions(seed: int, params: HashParams = HashParams()) -> HashFunctions:
    """make_hash_functions, hashmatch.cpp:53-69 (host-side, libstdc++ <random>)."""
    L = _lib.load()
    if params.tables < 1 or params.coarse_bits < 1 or params.coarse_bits > 32 or params.fine_bits < 1:
        raise BandmatchError("InvalidArgument", "hash params out of range")
    coarse = np.zeros(params.tables * params.coarse_bits * DIM, np.float32)
    fine = np.zeros(params.fine_bits * DIM, np.float32)
    hp = params.c()
    check(L.bmg_make_hash_functions(seed, C.byref(hp), ptr(coarse), ptr(fine)))
    return HashFunctions(params, seed, coarse.reshape(params.tables, params.coarse_bits, DIM),
                         fine.reshape(params.fine_bits, DIM))


class Matcher:
    """One device context: hash planes resident in HBM, the descriptor arena
    (DeviceArena capacity in descriptor units) and the kernels' scratch."""

    def __init__(self, hf: HashFunctions, capacity_units: int = 1 << 40, device: int = 0):
        L = _lib.load()
        self.hf = hf
        self._coarse = np.ascontiguousarray(hf.coarse, np.float32)
        self._fine = np.ascontiguousarray(hf.fine, np.float32)
        cfg = _lib.ConfigC(device, hf.params.c(), ptr(self._coarse), ptr(self._fine), hf.seed,
                           capacity_units)
        h = C.c_void_p()
        check(L.bmg_create(C.byref(cfg), C.byref(h)))
        self.handle = h
        self._L = L

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self._L.bmg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- arena --
    def upload(self, image_id: int, desc: np.ndarray) -> None:
        desc = np.ascontiguousarray(desc, np.float32).reshape(-1, DIM)
        check(self._L.bmg_upload(self.handle, image_id, ptr(desc), desc.shape[0]))
        self._keep = getattr(self, "_keep", {})
        self._keep[image_id] = desc  # must stay alive until the copy completes

    def evict(self, image_id: int) -> None:
        check(self._L.bmg_evict(self.handle, image_id))
        getattr(self, "_keep", {}).pop(image_id, None)

    def resident(self, image_id: int) -> bool:
        return bool(self._L.bmg_is_resident(self.handle, image_id))

    def arena_stats(self) -> dict:
        s = _lib.ArenaStatsC()
        check(self._L.bmg_arena_stats_get(self.handle, C.byref(s)))
        return {n: getattr(s, n) for n, _ in s._fields_}

    def synchronize(self):
        check(self._L.bmg_synchronize(self.handle))

    # -- row body --
    def row(self, needed, mean: np.ndarray | None = None) -> None:
        ids = np.ascontiguousarray(sorted(int(i) for i in needed), np.uint64)
        m = None if mean is None else np.ascontiguousarray(mean, np.float32)
        check(self._L.bmg_row(self.handle, ptr(ids), len(ids), ptr(m)))

    def row_mean(self) -> np.ndarray:
        out = np.zeros(DIM, np.float32)
        check(self._L.bmg_row_mean(self.handle, ptr(out)))
        return out

    def codes(self, image_id: int, count: int) -> HashCodeSet:
        p = self.hf.params
        coarse = np.zeros((max(count, 1), p.tables), np.uint32)
        fine = np.zeros((max(count, 1), p.fine_words), np.uint64)
        check(self._L.bmg_codes(self.handle, image_id, ptr(coarse), ptr(fine)))
        return HashCodeSet(image_id, self.hf.seed, p, count, coarse[:count], fine[:count])

    def match(self, pairs, mp: MatchParams = MatchParams(), max_matches: int | None = None):
        """Match (query, train) image pairs of the current row; returns a list of
        (n,2) int32 arrays in pair order."""
        pairs = list(pairs)
        q = np.ascontiguousarray([a for a, _ in pairs], np.uint64)
        t = np.ascontiguousarray([b for _, b in pairs], np.uint64)
        counts = getattr(self, "_keep", {})
        cap = max_matches if max_matches is not None else max(
            1, sum(len(counts[a]) if a in counts else 1 << 20 for a, _ in pairs))
        offs = np.zeros(len(pairs) + 1, np.uint64)
        out = np.zeros(2 * cap, np.int32)
        mpc = mp.c()
        check(self._L.bmg_match(self.handle, ptr(q), ptr(t), len(pairs), C.byref(mpc), ptr(offs),
                                ptr(out), cap))
        return [out[2 * int(offs[i]): 2 * int(offs[i + 1])].reshape(-1, 2).copy()
                for i in range(len(pairs))]

    # -- stateless mirrors --
    def compute_codes(self, fs: FeatureSet, mean) -> HashCodeSet:
        p = self.hf.params
        n = fs.size()
        m = np.ascontiguousarray(mean, np.float32).reshape(DIM)
        coarse = np.zeros((max(n, 1), p.tables), np.uint32)
        fine = np.zeros((max(n, 1), p.fine_words), np.uint64)
        check(self._L.bmg_compute_codes(self.handle, ptr(fs.descriptors) if n else None, n, ptr(m),
                                        ptr(coarse), ptr(fine)))
        return HashCodeSet(fs.image_id, self.hf.seed, p, n, coarse[:n].copy(), fine[:n].copy())

    def match_pair(self, qf: FeatureSet, qc: HashCodeSet, tf: FeatureSet, tc: HashCodeSet,
                   mp: MatchParams = MatchParams()) -> PairMatches:
        if qc.count != qf.size() or tc.count != tf.size():
            raise BandmatchError("HashMismatch", "code set does not cover its feature set")
        qcs, tcs = _codeset_c(qc), _codeset_c(tc)
        out = np.zeros(2 * max(qf.size(), 1), np.int32)
        n = C.c_uint64(0)
        mpc = mp.c()
        check(self._L.bmg_match_pair(self.handle, ptr(qf.descriptors) if qf.size() else None,
                                     C.byref(qcs[0]), ptr(tf.descriptors) if tf.size() else None,
                                     C.byref(tcs[0]), C.byref(mpc), ptr(out), C.byref(n)))
        return PairMatches(qf.image_id, tf.image_id, out[: 2 * n.value].reshape(-1, 2).copy())

    # -- instrumentation --
    def launch_count(self) -> int:
        return int(self._L.bmg_launch_count(self.handle))

    def set_profiling(self, on: bool):
        check(self._L.bmg_set_profiling(self.handle, 1 if on else 0))

    def kernel_time(self, cls: str):
        ms, n = C.c_double(0), C.c_uint64(0)
        check(self._L.bmg_kernel_time(self.handle, cls.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def fixup_counts(self):
        a, b = C.c_uint64(0), C.c_uint64(0)
        check(self._L.bmg_fixup_counts(self.handle, C.byref(a), C.byref(b)))
        return a.value, b.value

    def exact_walk_count(self):
        """Queries of the last row / match redone on the exact top-K path."""
        a = C.c_uint64(0)
        check(self._L.bmg_exact_walk_count(self.handle, C.byref(a)))
        return a.value

    def set_test_flags(self, force_exact_walk: bool = False, force_fp64_rerank: bool = False):
        """Test hooks (bmg_set_test_flags): send every query through the exact
        top-K walk and / or every ratio decision through the FP64 re-rank."""
        check(self._L.bmg_set_test_flags(self.handle, (1 if force_exact_walk else 0)
                                         | (2 if force_fp64_rerank else 0)))

    def row_mean_info(self):
        """(rounds, used_chain) of the last computed row mean (diagnostics)."""
        r, u = C.c_uint32(0), C.c_int(0)
        check(self._L.bmg_row_mean_info(self.handle, C.byref(r), C.byref(u)))
        return r.value, bool(u.value)


def _codeset_c(cs: HashCodeSet):
    coarse = np.ascontiguousarray(cs.coarse, np.uint32)
    fine = np.ascontiguousarray(cs.fine, np.uint64)
    keep = (coarse, fine)
    c = _lib.CodeSetC(cs.image_id, cs.function_seed, cs.params.c(), cs.count,
                      ptr(coarse) if cs.count else None, ptr(fine) if cs.count else None)
    return c, keep


_default_matchers: dict = {}


def _matcher_for(hf: HashFunctions) -> Matcher:
    key = (hf.seed, hf.params, id(hf))
    m = _default_matchers.get(key)
    if m is None:
        m = _default_matchers[key] = Matcher(hf)
    return m


def compute_codes(fs: FeatureSet, hf: HashFunctions, centering_mean) -> HashCodeSet:
    """compute_codes(fs, hf, mean), hashmatch.cpp:71-100, on the B200."""
    return _matcher_for(hf).compute_codes(fs, centering_mean)


def match_pair(qf: FeatureSet, qc: HashCodeSet, tf: FeatureSet, tc: HashCodeSet,
               mp: MatchParams = MatchParams(), hf: HashFunctions | None = None) -> PairMatches:
    """match_pair, hashmatch.cpp:102-211, on the B200.  ``hf`` selects the
    device context (defaults to the context of the functions that built qc)."""
    if qc.function_seed != tc.function_seed:
        raise BandmatchError("HashMismatch", "code sets built from different hash function seeds")
    if qc.params != tc.params:
        raise BandmatchError("HashMismatch", "code sets built with different hash parameters")
    if qc.count != qf.size() or tc.count != tf.size():
        raise BandmatchError("HashMismatch", "code set does not cover its feature set")
    if mp.k_nearest < 1:
        raise BandmatchError("InvalidArgument", "k_nearest must be >= 1")
    if qc.count == 0 or tc.count == 0:
        return PairMatches(qf.image_id, tf.image_id)
    if hf is None:
        hf = next((m.hf for (s, p, _), m in _default_matchers.items()
                   if s == qc.function_seed and p == qc.params), None)
        if hf is None:
            hf = HashFunctions(qc.params, qc.function_seed,
                               np.zeros((qc.params.tables, qc.params.coarse_bits, DIM), np.float32),
                               np.zeros((qc.params.fine_bits, DIM), np.float32))
    return _matcher_for(hf).match_pair(qf, qc, tf, tc, mp)


# ---- match files (hashmatch.cpp:243-363) ----------------------------------

def _sorted_by_pair(all_pm):
    out = sorted(all_pm, key=lambda pm: (pm.query_image, pm.train_image))
    res = []
    for pm in out:
        m = np.asarray(pm.matches, np.int32).reshape(-1, 2)
        if len(m) > 1 and not (m[1:, 0] > m[:-1, 0]).all():  # matcher output: ascending qi already
            m = m[np.lexsort((m[:, 1], m[:, 0]))]
        res.append(PairMatches(pm.query_image, pm.train_image, m, pm.stage))
    return res


def write_matches_binary(path, all_pm) -> None:
    """BMMT writer, hashmatch.cpp:311-332, natively (libbmg).  The matches of
    an ``execute_plan`` result are written straight from its pinned log;
    other lists are put in ``sorted_by_pair`` order first (:243-250)."""
    L = _lib.load()
    writer = getattr(all_pm, "_write_bmmt", None)
    if writer is not None:
        writer(str(path).encode())
        return
    ordered = _sorted_by_pair(all_pm)
    n = len(ordered)
    ids = np.array([(pm.query_image, pm.train_image) for pm in ordered], np.uint64).reshape(-1)
    counts = np.array([len(pm.matches) for pm in ordered], np.uint64)
    ends = np.cumsum(counts, dtype=np.uint64)
    ranges = np.stack([ends - counts, ends], 1).reshape(-1) if n else np.zeros(0, np.uint64)
    log = (np.concatenate([np.asarray(pm.matches, np.int32).reshape(-1, 2) for pm in ordered])
           if n else np.zeros((0, 2), np.int32))
    log = np.ascontiguousarray(log, np.int32)
    stages = np.array([1 if pm.stage == "verified" else 0 for pm in ordered], np.uint8)
    check(L.bmg_write_matches_binary(str(path).encode(), n, ptr(ids), ptr(ranges), ptr(log), ptr(stages)))


def read_matches_binary(path):
    """BMMT reader, hashmatch.cpp:334-363 (FormatError / TruncatedFile)."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for reading")
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(data):
            raise BandmatchError("TruncatedFile", f"unexpected end of file while reading {what}")
        b = data[pos: pos + n]
        pos += n
        return b

    if take(4, "match file magic") != b"BMMT":
        raise BandmatchError("FormatError", 'match file: bad magic, expected "BMMT"')
    (version,) = struct.unpack("<I", take(4, "match file version"))
    if version != 1:
        raise BandmatchError("FormatError", f"unsupported match file version {version}")
    (n_pairs,) = struct.unpack("<Q", take(8, "pair count"))
    out = []
    for _ in range(n_pairs):
        q, t = struct.unpack("<QQ", take(16, "image ids"))
        stage = take(1, "match stage")[0]
        if stage > 1:
            raise BandmatchError("FormatError", f"unknown match stage {stage}")
        (count,) = struct.unpack("<I", take(4, "match count"))
        m = np.frombuffer(take(8 * count, "match"), "<u4").astype(np.int32).reshape(-1, 2)
        out.append(PairMatches(q, t, m, "verified" if stage == 1 else "initial"))
    return out


def write_matches_text(path, all_pm) -> None:
    """Text writer, hashmatch.cpp:254-268 (empty pairs omitted)."""
    ordered = _sorted_by_pair(all_pm)
    nonempty = sum(1 for pm in ordered if len(pm.matches))
    with open(path, "w") as f:
        f.write(f"pairs {nonempty}\n")
        for pm in ordered:
            for qi, ti in pm.matches:
                f.write(f"{pm.query_image} {pm.train_image} {int(qi)} {int(ti)}\n")


def read_matches_text(path):
    """Text reader, hashmatch.cpp:270-309."""
    try:
        lines = Path(path).read_text().splitlines()
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for reading")
    if not lines:
        raise BandmatchError("TruncatedFile", "missing match header")
    hdr = lines[0].split()
    if len(hdr) < 2 or hdr[0] != "pairs" or not hdr[1].isdigit():
        raise BandmatchError("FormatError", f"malformed match header '{lines[0]}'")
    declared = int(hdr[1])
    grouped: dict = {}
    for line in lines[1:]:
        if not line:
            continue
        parts = line.split()
        try:
            q, t, qi, ti = (int(x) for x in parts[:4])
            if len(parts) < 4:
                raise ValueError
        except ValueError:
            raise BandmatchError("FormatError", f"malformed match line '{line}'")
        grouped.setdefault((q, t), []).append((qi, ti))
    if len(grouped) < declared:
        raise BandmatchError("TruncatedFile", f"match file lists {len(grouped)} pairs, header declares {declared}")
    if len(grouped) > declared:
        raise BandmatchError("FormatError", f"match file lists {len(grouped)} pairs, header declares {declared}")
    return [PairMatches(q, t, np.array(sorted(v), np.int32).reshape(-1, 2))
            for (q, t), v in sorted(grouped.items())]
