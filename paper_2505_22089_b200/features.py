"""Feature-input surface (include/bandmatch/features.hpp): synthetic band
scenes (features.cpp:68-197, generated host-side by libbmg) and the binary
``.feat`` file format (features.cpp:199-249) read in bulk rather than
float-by-float."""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from ._lib import DIM, BandmatchError, check, ptr
from .hashmatch import FeatureSet

__all__ = ["SyntheticScene", "generate_synthetic", "synthetic_counts", "write_features",
           "read_features", "load_features_dir"]


@dataclass(frozen=True)
class SyntheticScene:
    """SyntheticScene, features.hpp:56-64."""
    n_images: int = 0
    points_per_image: int = 0
    overlap_band: int = 0
    noise_sigma: float = 0.0
    outlier_fraction: float = 0.0
    seed: int = 0


def synthetic_counts(scene: SyntheticScene) -> np.ndarray:
    L = _lib.load()
    counts = np.zeros(max(scene.n_images, 1), np.uint64)
    check(L.bmg_synthetic_counts(scene.n_images, scene.points_per_image, scene.overlap_band,
                                 scene.noise_sigma, scene.outlier_fraction, ptr(counts)))
    return counts[: scene.n_images]


def generate_synthetic(scene: SyntheticScene, keypoints: bool = False, pinned=None, keep=None):
    """generate_synthetic (features.cpp:68-197): returns (images, true_pairs);
    images[i] is a FeatureSet with image_id i.  ``pinned``: optional callable
    (nbytes) -> writable uint8 buffer (e.g. page-locked memory) to generate into.
    ``keep``: optional set of image indices to store (the others are None in
    ``images``; their random draws are still made)."""
    L = _lib.load()
    counts = synthetic_counts(scene)
    if keep is not None:
        mask = np.zeros(max(scene.n_images, 1), np.uint8)
        for i in keep:
            if 0 <= i < scene.n_images:
                mask[i] = 1
        counts = np.where(mask[: scene.n_images] != 0, counts, 0).astype(np.uint64)
    total = int(counts.sum())
    if pinned is not None:
        buf = np.frombuffer(pinned(max(total, 1) * DIM * 4), np.float32, max(total, 1) * DIM)
    else:
        buf = np.zeros(max(total, 1) * DIM, np.float32)
    kps = np.zeros(max(total, 1) * 4, np.float32) if keypoints else None
    if keep is None:
        check(L.bmg_generate_synthetic(scene.n_images, scene.points_per_image, scene.overlap_band,
                                       scene.noise_sigma, scene.outlier_fraction, scene.seed,
                                       ptr(buf), ptr(kps)))
    else:
        check(L.bmg_generate_synthetic_subset(scene.n_images, scene.points_per_image,
                                              scene.overlap_band, scene.noise_sigma,
                                              scene.outlier_fraction, scene.seed, ptr(mask),
                                              ptr(buf), ptr(kps)))
    images, off = [], 0
    for i, n in enumerate(counts.tolist()):
        if keep is not None and not mask[i]:
            images.append(None)
            continue
        d = buf[off * DIM:(off + n) * DIM].reshape(n, DIM)
        k = kps[off * 4:(off + n) * 4].reshape(n, 4) if keypoints else None
        fs = FeatureSet.__new__(FeatureSet)
        fs.image_id, fs.descriptors, fs.keypoints = i, d, k
        images.append(fs)
        off += n
    band = scene.overlap_band
    pairs = [(i, j) for i in range(scene.n_images)
             for j in range(i + 1, min(scene.n_images, i + band + 1))]
    return images, np.array(pairs, np.uint64).reshape(-1, 2)


_MAGIC = b"BMF1"


def write_features(path, fs: FeatureSet) -> None:
    """Binary feature file, features.hpp:88-92 (magic BMF1, version 1)."""
    n = fs.size()
    kp = fs.keypoints if fs.keypoints is not None else np.zeros((n, 4), np.float32)
    rec = np.concatenate([np.asarray(kp, "<f4").reshape(n, 4),
                          np.asarray(fs.descriptors, "<f4").reshape(n, DIM)], axis=1)
    with open(path, "wb") as f:
        f.write(_MAGIC + struct.pack("<IQII", 1, fs.image_id, n, DIM))
        f.write(np.ascontiguousarray(rec, "<f4").tobytes())


def read_features(path, pinned=None, threads: int = 8) -> FeatureSet:
    """read_features, features.cpp:222-249 (same checks, FormatError /
    TruncatedFile), natively: libbmg reads the 528-byte records in large
    blocks on ``threads`` threads straight into the arrays.  ``pinned``:
    optional callable nbytes -> buffer (e.g. pinned host memory) that backs
    the descriptors, so the arena's H2D reads them directly."""
    L = _lib.load()
    bpath = str(path).encode()
    iid, n = C.c_uint64(0), C.c_uint64(0)
    check(L.bmg_read_features_header(bpath, C.byref(iid), C.byref(n)))
    count = n.value
    if pinned is not None:
        desc = np.frombuffer(pinned(max(count, 1) * DIM * 4), np.float32, max(count, 1) * DIM)
        desc = desc[: count * DIM].reshape(count, DIM)
    else:
        desc = np.empty((count, DIM), np.float32)
    kps = np.empty((count, 4), np.float32)
    check(L.bmg_read_features(bpath, count, ptr(desc), ptr(kps), threads, C.byref(iid), C.byref(n)))
    fs = FeatureSet(iid.value, desc)
    fs.keypoints = kps
    return fs


def load_features_dir(path) -> dict:
    """load_features_dir (bandmatch_cli.cpp:56-74): every *.feat, keyed by id."""
    out = {}
    for p in sorted(Path(path).glob("*.feat")):
        fs = read_features(p)
        if fs.image_id in out:
            raise BandmatchError("FormatError", f"duplicate image id {fs.image_id} in {path}")
        out[fs.image_id] = fs
    return out
