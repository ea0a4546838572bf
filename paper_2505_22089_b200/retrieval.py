"""Retrieval side of the pipeline (include/bandmatch/retrieval.hpp), SURVEY
§8f row f4: VLAD image encoding -- the per-image work select_pairs does
before its HNSW search (retrieval.cpp:386-399) -- on the B200 (vlad.cu,
``bmg_encode_vlad``), bit-exact with ``encode_vlad`` (retrieval.cpp:160-205);
plus the codebook file format (``write_codebook`` / ``read_codebook``,
retrieval.cpp:407-450) and codebook training (``train_codebook``, k-means,
retrieval.cpp:56-158, ``bmg_train_codebook``).  The HNSW index stays on the
host (reference code)."""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import BandmatchError, DIM, check, ptr
from .hashmatch import FeatureSet, HashFunctions, Matcher, _matcher_for, make_hash_functions

__all__ = ["Codebook", "VladVector", "encode_vlad", "encode_vlad_batch", "read_codebook",
           "train_codebook", "write_codebook"]


@dataclass
class Codebook:
    """Codebook, retrieval.hpp:14-21: k_words x 128 centroids, row-major."""
    k_words: int = 0
    centroids: np.ndarray = field(default_factory=lambda: np.zeros((0, DIM), np.float32))

    def centroid(self, k: int) -> np.ndarray:
        return self.centroids[k]


@dataclass
class VladVector:
    """VladVector, retrieval.hpp:36-39."""
    values: np.ndarray
    degenerate: bool = False


def _descs(x) -> np.ndarray:
    d = x.descriptors if isinstance(x, FeatureSet) else x
    return np.ascontiguousarray(np.asarray(d, np.float32).reshape(-1, DIM))


_vlad_ctx: list = []


def _context(matcher: Matcher | None) -> Matcher:
    if matcher is not None:
        return matcher
    if not _vlad_ctx:  # a device session; its hash planes are not used here
        _vlad_ctx.append(_matcher_for(make_hash_functions(0)))
    return _vlad_ctx[0]


def encode_vlad_batch(images, cb: Codebook, matcher: Matcher | None = None) -> list:
    """encode_vlad (retrieval.cpp:160-205) for every image of ``images``
    (FeatureSets or float[n][128] arrays) in one call on the B200: batches of
    images stream to HBM while earlier batches encode."""
    if cb.k_words < 1:
        raise BandmatchError("InvalidArgument", "codebook has no words")
    cent = np.ascontiguousarray(np.asarray(cb.centroids, np.float32).reshape(cb.k_words, DIM))
    arrs = [_descs(x) for x in images]
    n = len(arrs)
    views = (_lib.FeatureViewC * max(n, 1))()
    for i, a in enumerate(arrs):
        views[i].image_id = i
        views[i].descriptors = ptr(a) if len(a) else None
        views[i].count = len(a)
    dim = cb.k_words * DIM
    vals = np.zeros((max(n, 1), dim), np.float32)
    deg = np.zeros(max(n, 1), np.uint8)
    m = _context(matcher)
    check(_lib.load().bmg_encode_vlad(m.handle, ptr(cent), cb.k_words, views, n, ptr(vals), ptr(deg)))
    return [VladVector(vals[i], bool(deg[i])) for i in range(n)]


def encode_vlad(fs, cb: Codebook, matcher: Matcher | None = None) -> VladVector:
    """encode_vlad(fs, cb), retrieval.cpp:160-205, on the B200."""
    return encode_vlad_batch([fs], cb, matcher)[0]


def train_codebook(descriptors, k_words: int, max_iters: int, seed: int, sse_history: list | None = None,
                   matcher: Matcher | None = None) -> Codebook:
    """train_codebook (retrieval.cpp:56-158) on the B200, bit-exact: the
    reference's seeding, Lloyd iterations with FP64 assignments and sums,
    empty clusters reseeded from the farthest point.  ``sse_history`` (a
    list) receives the SSE of every assignment step."""
    d = _descs(descriptors)
    n = len(d)
    cent = np.zeros((max(k_words, 1), DIM), np.float32)
    sse = np.zeros(max(max_iters, 1), np.float64)
    n_sse = C.c_int(0)
    m = _context(matcher)
    check(_lib.load().bmg_train_codebook(m.handle, ptr(d) if n else None, n, k_words, max_iters, seed,
                                         ptr(cent), ptr(sse), C.byref(n_sse)))
    if sse_history is not None:
        sse_history.clear()
        sse_history.extend(float(x) for x in sse[: n_sse.value])
    return Codebook(k_words, cent[:k_words])


_MAGIC = b"BMCB"


def write_codebook(path, cb: Codebook) -> None:
    """write_codebook, retrieval.cpp:411-425: "BMCB", u32 words, u32 dim, f32 centroids."""
    cent = np.asarray(cb.centroids, np.float32)
    if cb.k_words < 1 or cent.size != cb.k_words * DIM:
        raise BandmatchError("FormatError", "codebook shape is inconsistent")
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC + struct.pack("<II", cb.k_words, DIM))
            f.write(np.ascontiguousarray(cent, "<f4").tobytes())
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for writing") from None


def read_codebook(path) -> Codebook:
    """read_codebook, retrieval.cpp:427-448, with its checks and messages."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for reading") from None

    def need(n, what, at):
        if len(data) < at + n:
            raise BandmatchError("TruncatedFile", f"unexpected end of file while reading {what}")

    need(4, "codebook magic", 0)
    if data[:4] != _MAGIC:
        raise BandmatchError("FormatError", 'codebook: bad magic, expected "BMCB"')
    need(4, "word count", 4)
    k = struct.unpack_from("<I", data, 4)[0]
    if k < 1:
        raise BandmatchError("FormatError", "codebook word count must be >= 1")
    need(4, "descriptor dim", 8)
    dim = struct.unpack_from("<I", data, 8)[0]
    if dim != DIM:
        raise BandmatchError("FormatError", f"codebook dim {dim} != 128")
    body = k * DIM * 4
    if len(data) < 12 + body:
        raise BandmatchError("TruncatedFile", "unexpected end of file while reading centroid")
    cent = np.frombuffer(data, "<f4", k * DIM, 12).astype(np.float32).reshape(k, DIM)
    return Codebook(k, cent)
