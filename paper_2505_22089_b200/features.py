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


def generate_synthetic(scene: SyntheticScene, keypoints: bool = False, pinned=None):
    """generate_synthetic (features.cpp:68-197): returns (images, true_pairs);
    images[i] is a FeatureSet with image_id i.  ``pinned``: optional callable
    (nbytes) -> writable uint8 buffer (e.g. page-locked memory) to generate into."""
    L = _lib.load()
    counts = synthetic_counts(scene)
    total = int(counts.sum())
    if pinned is not None:
        buf = np.frombuffer(pinned(max(total, 1) * DIM * 4), np.float32, max(total, 1) * DIM)
    else:
        buf = np.zeros(max(total, 1) * DIM, np.float32)
    kps = np.zeros(max(total, 1) * 4, np.float32) if keypoints else None
    check(L.bmg_generate_synthetic(scene.n_images, scene.points_per_image, scene.overlap_band,
                                   scene.noise_sigma, scene.outlier_fraction, scene.seed,
                                   ptr(buf), ptr(kps)))
    images, off = [], 0
    for i, n in enumerate(counts.tolist()):
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


def read_features(path) -> FeatureSet:
    """read_features, features.cpp:222-249, as one bulk read."""
    try:
        data = Path(path).read_bytes()
    except OSError:
        raise BandmatchError("FormatError", f"cannot open {path} for reading")
    if len(data) < 4:
        raise BandmatchError("TruncatedFile", "unexpected end of file while reading feature file magic")
    if data[:4] != _MAGIC:
        raise BandmatchError("FormatError", 'feature file: bad magic, expected "BMF1"')
    if len(data) < 24:
        raise BandmatchError("TruncatedFile", "unexpected end of file while reading header")
    version, image_id, count, dim = struct.unpack("<IQII", data[4:24])
    if version != 1:
        raise BandmatchError("FormatError", f"unsupported feature file version {version}")
    if dim != DIM:
        raise BandmatchError("FormatError", f"descriptor dim {dim} != 128")
    need = count * (4 + DIM) * 4
    if len(data) - 24 < need:
        raise BandmatchError("TruncatedFile", "unexpected end of file while reading descriptor")
    rec = np.frombuffer(data, "<f4", count * (4 + DIM), 24).reshape(count, 4 + DIM)
    fs = FeatureSet(image_id, np.ascontiguousarray(rec[:, 4:], np.float32))
    fs.keypoints = np.ascontiguousarray(rec[:, :4], np.float32)
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
