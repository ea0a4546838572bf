"""Host verification surface (include/bandmatch/verify.hpp), stage 1: the
spatial-angular-order filter ``sao_filter`` (verify.cpp:303-341), native in
libbmg (``bmg_sao_filter``) with the reference's results and an adjacency-
driven Bowyer-Watson instead of the reference's quadratic one (SURVEY §8f
row f1).  RANSAC (verify.cpp:345-527) needs Eigen's JacobiSVD for parity and
is not rebuilt here."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check, ptr
from .hashmatch import PairMatches

__all__ = ["SaoParams", "SaoOutcome", "sao_filter", "knn_from_delaunay"]


def knn_from_delaunay(pts, n_neighbors: int):
    """knn_from_delaunay (verify.cpp:135-196): (neighbors [n][k] padded with
    -1, used_fallback)."""
    L = _lib.load()
    xy = np.ascontiguousarray(np.asarray(pts, np.float64).reshape(-1, 2))
    n = len(xy)
    out = np.full(max(n * n_neighbors, 1), -1, np.int32)
    fb = C.c_int(0)
    check(L.bmg_delaunay_knn(ptr(xy) if n else None, n, n_neighbors, ptr(out), C.byref(fb)))
    return out[: n * n_neighbors].reshape(n, n_neighbors), bool(fb.value)


@dataclass
class SaoParams:
    """SaoParams, verify.hpp:40-43."""
    n_neighbors: int = 6
    score_threshold: float = 0.5


@dataclass
class SaoOutcome:
    """SaoOutcome, verify.hpp:45-53."""
    kept: PairMatches
    scores: np.ndarray = field(default_factory=lambda: np.zeros(0))
    passthrough: bool = False
    delaunay_fallback: bool = False


def sao_filter(matches: PairMatches, query_kps, train_kps, params: SaoParams = SaoParams()) -> SaoOutcome:
    """sao_filter(matches, query_kps, train_kps, params); keypoints [n][4]
    (x, y, scale, orientation) float32."""
    L = _lib.load()
    m = np.ascontiguousarray(np.asarray(matches.matches, np.int32).reshape(-1, 2))
    qk = np.ascontiguousarray(np.asarray(query_kps, np.float32).reshape(-1, 4))
    tk = np.ascontiguousarray(np.asarray(train_kps, np.float32).reshape(-1, 4))
    n = len(m)
    keep = np.zeros(max(n, 1), np.uint8)
    scores = np.zeros(max(n, 1), np.float64)
    flags = C.c_uint32(0)
    check(L.bmg_sao_filter(ptr(m) if n else None, n, ptr(qk), len(qk), ptr(tk), len(tk),
                           params.n_neighbors, params.score_threshold, ptr(keep), ptr(scores),
                           C.byref(flags)))
    kept = PairMatches(matches.query_image, matches.train_image, m[keep[:n] != 0], matches.stage)
    return SaoOutcome(kept, scores[:n], bool(flags.value & 1), bool(flags.value & 2))
