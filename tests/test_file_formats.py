"""the data formats either side of the path --
natively in libbmg (csrc/host_io.cpp) against the compiled reference:
feature files written by the reference's write_features read back bit for
bit (features.cpp:199-249), every truncation / damage failing with the
reference's code and message, and BMMT match files (hashmatch.cpp:311-332)
byte-identical to the reference writer's (acceptance gate 10)."""
import struct

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import features as F


def ref_error(reference, fn):
    with pytest.raises(Exception) as e:
        fn()
    return str(e.value)


@pytest.mark.parametrize("n", [0, 1, 7, 4096, 4097, 20000])
def test_reference_feature_files_read_bit_exact(reference, tmp_path, n):
    rng = np.random.default_rng(n)
    desc = rng.standard_normal((n, 128)).astype(np.float32)
    kp = rng.standard_normal((n, 4)).astype(np.float32)
    if n:
        desc[0, :3] = [np.nan, -0.0, np.float32(1e-45)]  # bit patterns, not values
    p = tmp_path / f"{n}.feat"
    reference.write_features(p, 900 + n, desc, kp)
    for threads in (1, 3, 16):
        fs = F.read_features(p, threads=threads)
        assert fs.image_id == 900 + n
        assert np.array_equal(fs.descriptors.view(np.uint32), desc.view(np.uint32))
        assert np.array_equal(fs.keypoints.view(np.uint32), kp.view(np.uint32))
    rid, rdesc, rkp = reference.read_features(p)
    assert rid == 900 + n and np.array_equal(rdesc.view(np.uint32), desc.view(np.uint32))


def test_feature_file_damage_matches_reference_errors(reference, tmp_path):
    rng = np.random.default_rng(1)
    desc = rng.standard_normal((5, 128)).astype(np.float32)
    kp = rng.standard_normal((5, 4)).astype(np.float32)
    p = tmp_path / "a.feat"
    reference.write_features(p, 3, desc, kp)
    data = p.read_bytes()
    cases = {"magic": b"BMFX" + data[4:], "version": data[:4] + struct.pack("<I", 2) + data[8:],
             "dim": data[:20] + struct.pack("<I", 64) + data[24:]}
    # every cut inside the header, inside a keypoint and inside a descriptor
    for cut in [0, 2, 4, 6, 8, 15, 16, 19, 20, 23, 24, 30, 24 + 16, 24 + 100, 24 + 528 * 3 + 17,
                len(data) - 1]:
        cases[f"cut{cut}"] = data[:cut]
    for name, blob in cases.items():
        q = tmp_path / f"{name}.feat"
        q.write_bytes(blob)
        with pytest.raises(bm.BandmatchError) as ours:
            F.read_features(q)
        theirs = ref_error(reference, lambda: reference.read_features(q))
        assert str(ours.value) == theirs, name
    missing = tmp_path / "nope.feat"
    with pytest.raises(bm.BandmatchError) as ours:
        F.read_features(missing)
    assert str(ours.value) == ref_error(reference, lambda: reference.read_features(missing))


def test_feature_file_into_pinned_style_buffer(reference, tmp_path):
    desc = np.random.default_rng(2).standard_normal((300, 128)).astype(np.float32)
    p = tmp_path / "b.feat"
    reference.write_features(p, 5, desc, np.zeros((300, 4), np.float32))
    keep = []

    def alloc(nbytes):
        b = bytearray(nbytes)
        keep.append(b)
        return b

    fs = F.read_features(p, pinned=alloc)
    assert np.array_equal(fs.descriptors, desc)
    assert np.shares_memory(fs.descriptors, np.frombuffer(keep[0], np.uint8))


def random_pairs(rng, n_pairs):
    out = []
    for _ in range(n_pairs):
        q, t = sorted(rng.choice(50, 2, replace=False).tolist())
        m = int(rng.integers(0, 40))
        qi = np.sort(rng.choice(1000, m, replace=False)).astype(np.int32)
        out.append((q, t, np.stack([qi, rng.integers(0, 1000, m).astype(np.int32)], 1)))
    # unique pairs (a PairMatches list from execute_plan has one entry per pair)
    seen, uniq = set(), []
    for q, t, m in out:
        if (q, t) not in seen:
            seen.add((q, t))
            uniq.append((q, t, m))
    return uniq


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_match_files_byte_identical_to_reference(reference, tmp_path, seed):
    rng = np.random.default_rng(seed)
    pairs = random_pairs(rng, 60)
    stages = rng.integers(0, 2, len(pairs)).tolist()
    ours, theirs = tmp_path / "ours.bin", tmp_path / "theirs.bin"
    bm.write_matches_binary(ours, [bm.PairMatches(q, t, m, "verified" if s else "initial")
                                   for (q, t, m), s in zip(pairs, stages)])
    reference.write_matches_binary(theirs, pairs, stages)
    assert ours.read_bytes() == theirs.read_bytes()
    back = bm.read_matches_binary(ours)
    assert [(p.query_image, p.train_image) for p in back] == sorted((q, t) for q, t, _ in pairs)


def test_empty_match_file_byte_identical(reference, tmp_path):
    ours, theirs = tmp_path / "o.bin", tmp_path / "t.bin"
    bm.write_matches_binary(ours, [])
    reference.write_matches_binary(theirs, [])
    assert ours.read_bytes() == theirs.read_bytes() == b"BMMT" + struct.pack("<IQ", 1, 0)
