"""GPU parity of match_pair (hashmatch.cpp:102-211): the reference's own
known-answer cases (test_hashmatch.cpp:133-325, acceptance gate 4) plus
oracle-checked random and full-size pairs."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import BandmatchError, FeatureSet, MatchParams

pytestmark = pytest.mark.gpu
ZERO = np.zeros(128, np.float32)


def unit_rows(rng, n):
    d = rng.standard_normal((n, 128)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.ascontiguousarray(d, np.float32)


def axis_set(image_id, xs):
    # test_hashmatch.cpp:27-40: (10 + x, 0, ..., 0) -> one bucket per table
    d = np.zeros((len(xs), 128), np.float32)
    d[:, 0] = 10.0 + np.asarray(xs, np.float32)
    return FeatureSet(image_id, d)


def gpu_match(hf, qf, tf, mean=ZERO, mp=MatchParams()):
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    return bm.match_pair(qf, qc, tf, tc, mp, hf=hf), qc, tc


def oracle_match(oracle, hf, qf, tf, qc, tc, mp=MatchParams()):
    return oracle.match_pair(qf.descriptors, (qc.coarse, qc.fine), tf.descriptors,
                             (tc.coarse, tc.fine), (hf.params.tables, hf.params.coarse_bits,
                                                     hf.params.fine_bits), mp.k_nearest, mp.ratio)


def test_exact_copy_beats_distractors(oracle):
    hf = bm.make_hash_functions(9)
    rng = np.random.default_rng(42)
    qf = FeatureSet(1, unit_rows(rng, 1))
    t = unit_rows(rng, 6)
    t[3] = qf.descriptors[0]
    pm, _, _ = gpu_match(hf, qf, FeatureSet(2, t))
    assert pm.as_list() == [(0, 3)]
    assert (pm.query_image, pm.train_image) == (1, 2)


@pytest.mark.parametrize("near,far,expect", [(0.3, 0.7, True), (0.4, 0.7, False),
                                             (0.35, 0.7, False)])
def test_ratio_rule_is_strict(oracle, near, far, expect):
    hf = bm.make_hash_functions(10)
    qf = axis_set(1, [0.0])
    tf = axis_set(2, [near, far])
    pm, _, _ = gpu_match(hf, qf, tf)
    bf = oracle.brute_force_match(qf.descriptors, tf.descriptors, 0.5)
    assert np.array_equal(pm.matches, bf)
    assert bool(len(pm.matches)) == expect


def test_lone_candidate_is_kept():
    hf = bm.make_hash_functions(11)
    pm, _, _ = gpu_match(hf, axis_set(1, [0.0]), axis_set(2, [0.9]))
    assert pm.as_list() == [(0, 0)]


@pytest.mark.parametrize("seed,count", [(2024, 120), (404, 500)])
def test_bucket_covered_instances_equal_brute_force(oracle, seed, count):
    # test_hashmatch.cpp:177-195 and acceptance gate 4 (acceptance.cpp:308-339)
    hf = bm.make_hash_functions(12)
    rng = np.random.default_rng(seed)
    for _ in range(count):
        nq, nt = 1 + int(rng.integers(12)), 1 + int(rng.integers(8))
        qf = axis_set(10, rng.uniform(-1, 1, nq))
        tf = axis_set(20, rng.uniform(-1, 1, nt))
        pm, _, _ = gpu_match(hf, qf, tf)
        assert np.array_equal(pm.matches, oracle.brute_force_match(qf.descriptors, tf.descriptors, 0.5))


def test_empty_and_disjoint_inputs():
    hf = bm.make_hash_functions(16)
    qf = axis_set(1, [0.0, 0.5])
    empty = axis_set(2, [])
    assert len(gpu_match(hf, qf, empty)[0].matches) == 0
    assert len(gpu_match(hf, empty, qf)[0].matches) == 0
    far = np.zeros((2, 128), np.float32)
    far[:, 0] = [-10.0 + 0.2, -10.0 - 0.4]
    assert len(gpu_match(hf, qf, FeatureSet(3, far))[0].matches) == 0


def test_error_codes():
    rng = np.random.default_rng(91)
    qf, tf = FeatureSet(1, unit_rows(rng, 4)), FeatureSet(2, unit_rows(rng, 4))
    h1, h2 = bm.make_hash_functions(1), bm.make_hash_functions(2)
    qc = bm.compute_codes(qf, h1, ZERO)
    with pytest.raises(BandmatchError) as e:
        bm.match_pair(qf, qc, tf, bm.compute_codes(tf, h2, ZERO), hf=h1)
    assert e.value.code == "HashMismatch"
    h3 = bm.make_hash_functions(1, bm.HashParams(5, 8, 128))
    with pytest.raises(BandmatchError) as e:
        bm.match_pair(qf, qc, tf, bm.compute_codes(tf, h3, ZERO), hf=h1)
    assert e.value.code == "HashMismatch"
    tc = bm.compute_codes(tf, h1, ZERO)
    shrunk = FeatureSet(2, tf.descriptors[:3])
    with pytest.raises(BandmatchError) as e:
        bm.match_pair(qf, qc, shrunk, tc, hf=h1)
    assert e.value.code == "HashMismatch"
    with pytest.raises(BandmatchError) as e:
        bm.match_pair(qf, qc, tf, tc, MatchParams(0, 0.5), hf=h1)
    assert e.value.code == "InvalidArgument"
    with pytest.raises(BandmatchError) as e:
        bm.match_pair(qf, qc, tf, tc, MatchParams(33, 0.5), hf=h1)
    assert e.value.code == "Unsupported"


@pytest.mark.parametrize("k,ratio", [(8, 0.5), (1, 0.5), (2, 0.5), (3, 0.8), (9, 0.5), (32, 0.5),
                                     (8, 1.0), (8, 0.2), (16, 0.9)])
def test_random_pairs_match_oracle(oracle, k, ratio):
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(k * 100 + int(ratio * 10))
    base = unit_rows(rng, 3000)
    q = base[:2500] + 0.03 * rng.standard_normal((2500, 128)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qf = FeatureSet(1, q)
    tf = FeatureSet(2, base)
    mean = np.mean(np.concatenate([q, base]), axis=0).astype(np.float32)
    mp = MatchParams(k, ratio)
    pm, qc, tc = gpu_match(hf, qf, tf, mean, mp)
    ref = oracle_match(oracle, hf, qf, tf, qc, tc, mp)
    assert np.array_equal(pm.matches, ref)
    assert len(ref) > (100 if ratio >= 0.5 else 0)


@pytest.mark.parametrize("nq,nt", [(3000, 16384), (16384, 5000), (1, 20000)])
def test_large_train_images_use_the_global_code_path(oracle, nq, nt):
    # > 12,800 train descriptors do not fit the shared-memory code stage, so
    # the kernel reads fine codes through L1/L2 (BASELINE configs 4 and 5)
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(nq + nt)
    base = unit_rows(rng, max(nq, nt))
    t = base[:nt]
    q = base[:nq] + 0.04 * rng.standard_normal((nq, 128)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qf, tf = FeatureSet(1, q), FeatureSet(2, t)
    mean = np.mean(np.concatenate([q, t]), axis=0).astype(np.float32)
    pm, qc, tc = gpu_match(hf, qf, tf, mean)
    oc = oracle.compute_codes(t, hf.coarse, hf.fine, mean)
    assert np.array_equal(tc.coarse, oc[0]) and np.array_equal(tc.fine, oc[1])
    assert np.array_equal(pm.matches, oracle_match(oracle, hf, qf, tf, qc, tc))


def test_full_size_synthetic_pair_matches_reference(reference, oracle):
    # BASELINE config 1: images (band, band+1) of generate_synthetic(ppi=8192)
    band = 11
    imgs, _ = reference.generate_synthetic(band + 2, 8192, band, 0.02, 0.2, 7)
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    qd, td = imgs[band], imgs[band + 1]
    mean = oracle.row_mean([qd, td])
    pm, qc, tc = gpu_match(hf, FeatureSet(band, qd), FeatureSet(band + 1, td), mean)
    rc = reference.compute_codes(qd, hf.coarse, hf.fine, mean)
    assert np.array_equal(qc.coarse, rc[0]) and np.array_equal(qc.fine, rc[1])
    ref = reference.match_pair(qd, rc, td, (tc.coarse, tc.fine), (6, 8, 128))
    assert np.array_equal(pm.matches, ref)
    assert len(ref) > 5000
