"""CPU tests of the host-side surface: the synthetic scene generator
(features.cpp:68-197) against the compiled reference, feature / match / plan
file formats (test_hashmatch.cpp:327-434, test_features.cpp:249-287), plan
flattening and the reference's execute_plan inputs."""
import json
import struct

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import features as F


@pytest.mark.parametrize("scene", [(5, 200, 2, 0.02, 0.2, 7), (13, 8192, 11, 0.02, 0.2, 7),
                                   (8, 50, 2, 0.01, 0.0, 99), (3, 10, 0, 0.0, 1.0, 5),
                                   (4, 0, 1, 0.02, 0.2, 1), (1, 7, 0, 0.5, 0.5, 2 ** 63)])
def test_generator_equals_reference(reference, scene):
    imgs, pairs = F.generate_synthetic(F.SyntheticScene(*scene), keypoints=True)
    ri, rp, rk = reference.generate_synthetic(*scene, keypoints=True)
    assert np.array_equal(pairs, rp)
    for a, b, k in zip(imgs, ri, rk):
        assert np.array_equal(a.descriptors.view(np.uint32), b.view(np.uint32))
        assert np.array_equal(a.keypoints.view(np.uint32), k.view(np.uint32))


@pytest.mark.parametrize("bad", [(0, 10, 0, 0.0, 0.0), (3, 10, 3, 0.0, 0.0), (3, -1, 1, 0.0, 0.0),
                                 (3, 10, 1, 0.0, 1.5), (3, 10, 1, -0.1, 0.0)])
def test_generator_rejects_invalid_scenes(bad):
    with pytest.raises(bm.BandmatchError) as e:
        F.generate_synthetic(F.SyntheticScene(*bad, seed=1))
    assert e.value.code == "InvalidScene"


def test_synthetic_counts_follow_band_structure():
    c = F.synthetic_counts(F.SyntheticScene(32, 8192, 11, 0.02, 0.2, 7))
    ppa = round(8192 * 0.8 / 12)
    assert c[0] == ppa + round(8192 * 0.2)
    assert c[11] == c[31] == 12 * ppa + round(8192 * 0.2) == 8190


def test_feature_file_round_trip_and_damage(tmp_path):
    rng = np.random.default_rng(0)
    fs = bm.FeatureSet(77, rng.standard_normal((9, 128)).astype(np.float32))
    fs.keypoints = rng.standard_normal((9, 4)).astype(np.float32)
    p = tmp_path / "a.feat"
    F.write_features(p, fs)
    back = F.read_features(p)
    assert back.image_id == 77 and np.array_equal(back.descriptors, fs.descriptors)
    assert np.array_equal(back.keypoints, fs.keypoints)
    data = p.read_bytes()
    (tmp_path / "magic.feat").write_bytes(b"X" + data[1:])
    (tmp_path / "ver.feat").write_bytes(data[:4] + struct.pack("<I", 9) + data[8:])
    (tmp_path / "dim.feat").write_bytes(data[:20] + struct.pack("<I", 64) + data[24:])
    (tmp_path / "cut.feat").write_bytes(data[: len(data) // 2])
    for name, code in [("magic", "FormatError"), ("ver", "FormatError"), ("dim", "FormatError"),
                       ("cut", "TruncatedFile"), ("missing", "FormatError")]:
        with pytest.raises(bm.BandmatchError) as e:
            F.read_features(tmp_path / f"{name}.feat")
        assert e.value.code == code


def test_match_binary_round_trip_keeps_empty_pairs_and_stages(tmp_path):
    a = bm.PairMatches(7, 8, np.array([[1, 5], [0, 2]], np.int32), "verified")
    b = bm.PairMatches(3, 4)
    p = tmp_path / "m.bin"
    bm.write_matches_binary(p, [a, b])
    back = bm.read_matches_binary(p)
    assert [(x.query_image, x.train_image, x.stage) for x in back] == [(3, 4, "initial"),
                                                                         (7, 8, "verified")]
    assert back[0].matches.shape == (0, 2)
    assert back[1].as_list() == [(0, 2), (1, 5)]


def test_match_binary_is_byte_identical_to_reference_layout(tmp_path):
    # hashmatch.cpp:311-332: "BMMT", u32 1, u64 n, then per pair u64 q, u64 t,
    # u8 stage, u32 count, count x (u32 qi, u32 ti)
    p = tmp_path / "m.bin"
    bm.write_matches_binary(p, [bm.PairMatches(1, 2, np.array([[0, 0]], np.int32))])
    expect = (b"BMMT" + struct.pack("<IQ", 1, 1) + struct.pack("<QQBI", 1, 2, 0, 1) +
              struct.pack("<II", 0, 0))
    assert p.read_bytes() == expect


def test_damaged_match_binary_files(tmp_path):
    p = tmp_path / "m.bin"
    bm.write_matches_binary(p, [bm.PairMatches(1, 2, np.array([[0, 0]], np.int32))])
    data = bytearray(p.read_bytes())

    def patched(off, val):
        d = bytearray(data)
        d[off] = val
        q = tmp_path / f"p{off}.bin"
        q.write_bytes(bytes(d))
        return q

    for off, val in [(0, ord("X")), (4, 9), (32, 7)]:
        with pytest.raises(bm.BandmatchError) as e:
            bm.read_matches_binary(patched(off, val))
        assert e.value.code == "FormatError"
    cut = tmp_path / "cut.bin"
    cut.write_bytes(bytes(data[: len(data) // 2]))
    with pytest.raises(bm.BandmatchError) as e:
        bm.read_matches_binary(cut)
    assert e.value.code == "TruncatedFile"


def test_match_text_files(tmp_path):
    a = bm.PairMatches(2, 5, np.array([[3, 1], [0, 7]], np.int32))
    b = bm.PairMatches(1, 4, np.array([[2, 2]], np.int32))
    c = bm.PairMatches(9, 10)
    p = tmp_path / "m.txt"
    bm.write_matches_text(p, [a, b, c])
    back = bm.read_matches_text(p)
    assert [(x.query_image, x.train_image) for x in back] == [(1, 4), (2, 5)]
    assert back[1].as_list() == [(0, 7), (3, 1)]
    cases = {"empty": ("", "TruncatedFile"), "hdr": ("pears 3\n", "FormatError"),
             "line": ("pairs 1\n1 2 three 4\n", "FormatError"),
             "short": ("pairs 2\n1 2 0 0\n", "TruncatedFile"),
             "extra": ("pairs 1\n1 2 0 0\n3 4 0 0\n", "FormatError")}
    for name, (text, code) in cases.items():
        q = tmp_path / f"{name}.txt"
        q.write_text(text)
        with pytest.raises(bm.BandmatchError) as e:
            bm.read_matches_text(q)
        assert e.value.code == code


def test_plan_json_round_trip_and_flatten(tmp_path, reference):
    pairs = np.array([(i, j) for i in range(12) for j in range(i + 1, min(12, i + 4))], np.uint64)
    path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(12), pairs, 3, 6, path)
    plan = bm.read_plan(path)
    assert plan.pairs() == sorted(map(tuple, pairs.tolist()))
    out = tmp_path / "again.json"
    bm.write_plan(out, plan)
    assert json.loads(out.read_text()) == json.loads(path.read_text())
    flat = bm.flatten_plan(plan)
    n_rows = sum(len(it.rows) for it in plan.iterations)
    assert len(flat.row_needed_offsets) == n_rows + 1
    assert int(flat.row_pair_offsets[-1]) == len(pairs)
    rows = [r for it in plan.iterations for r in it.rows]
    for k, r in enumerate(rows):
        nd = flat.needed_ids[flat.row_needed_offsets[k]:flat.row_needed_offsets[k + 1]].tolist()
        assert nd == r.needed() and nd == sorted(set(nd))


def test_read_plan_errors(tmp_path):
    (tmp_path / "bad.json").write_text("{")
    (tmp_path / "missing.json").write_text('{"strategy": "mbr"}')
    for name in ["bad", "missing", "absent"]:
        with pytest.raises(bm.BandmatchError) as e:
            bm.read_plan(tmp_path / f"{name}.json")
        assert e.value.code == "FormatError"


def test_bench_plans_are_the_reference_schedules():
    from pathlib import Path
    root = Path(__file__).resolve().parents[1] / "bench_data"
    p = bm.read_plan(root / "plan_block32.json")
    assert p.pair_count() == 286 and sum(len(i.rows) for i in p.iterations) == 2
    s = bm.read_plan(root / "plan_strip500.json")
    assert s.pair_count() == 4945
