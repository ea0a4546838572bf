"""GPU parity of the row body: centering mean (engine.cpp:446-461) and
compute_codes (hashmatch.cpp:71-100) against the C oracle, bit-exact."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm

pytestmark = pytest.mark.gpu


def unit_rows(rng, n, dim=128):
    d = rng.standard_normal((n, dim)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.ascontiguousarray(d, np.float32)


def same_bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.fixture(scope="module")
def hf():
    return bm.make_hash_functions(bm.seed_for(42, "matching"))


def test_row_mean_and_codes_match_oracle(hf, oracle):
    rng = np.random.default_rng(1)
    imgs = [unit_rows(rng, n) for n in (700, 1, 3000, 129)]
    with bm.Matcher(hf) as m:
        for i, d in enumerate(imgs):
            m.upload(10 + i, d)
        m.row([10 + i for i in range(len(imgs))])
        mean = m.row_mean()
        assert same_bits(mean, oracle.row_mean(imgs))
        for i, d in enumerate(imgs):
            cs = m.codes(10 + i, len(d))
            oc = oracle.compute_codes(d, hf.coarse, hf.fine, mean)
            assert np.array_equal(cs.coarse, oc[0])
            assert np.array_equal(cs.fine, oc[1])


@pytest.mark.parametrize("n", [1, 2, 31, 127, 128, 129, 1000, 8192])
def test_compute_codes_sizes(hf, oracle, n):
    rng = np.random.default_rng(n)
    d = unit_rows(rng, n)
    mean = (0.01 * rng.standard_normal(128)).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(1, d), hf, mean)
    oc = oracle.compute_codes(d, hf.coarse, hf.fine, mean)
    assert np.array_equal(cs.coarse, oc[0])
    assert np.array_equal(cs.fine, oc[1])
    assert cs.count == n and cs.coarse.shape == (n, 6) and cs.fine.shape == (n, 2)


def test_descriptor_equal_to_mean_codes_to_zero(hf):
    # test_hashmatch.cpp:77-91: every projection is exactly 0 -> all bits 0
    mean = (0.01 * np.arange(128)).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(1, mean[None, :]), hf, mean)
    assert not cs.coarse.any() and not cs.fine.any()


def test_fixup_overflow_path(hf, oracle):
    # 70k descriptors equal to the mean: 12M uncertifiable signs overflow the
    # fixup list and force the full FP64 recompute; mix in random rows too
    rng = np.random.default_rng(7)
    mean = (0.01 * rng.standard_normal(128)).astype(np.float32)
    d = np.repeat(mean[None, :], 70000, axis=0)
    d[::97] = unit_rows(rng, len(d[::97]))
    cs = bm.compute_codes(bm.FeatureSet(1, d), hf, mean)
    oc = oracle.compute_codes(d[:3000], hf.coarse, hf.fine, mean)
    assert np.array_equal(cs.coarse[:3000], oc[0]) and np.array_equal(cs.fine[:3000], oc[1])
    assert not cs.coarse[1:97].any() and not cs.fine[1:97].any()


def test_copy_and_negation(hf):
    # test_hashmatch.cpp:93-107
    rng = np.random.default_rng(77)
    d = unit_rows(rng, 1)
    d = np.concatenate([d, d, -d]).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(1, d), hf, np.zeros(128, np.float32))
    assert np.array_equal(cs.coarse[0], cs.coarse[1])
    ham = lambda a, b: sum(bin(int(x) ^ int(y)).count("1") for x, y in zip(cs.fine[a], cs.fine[b]))
    assert ham(0, 1) == 0
    assert ham(0, 2) == 128


@pytest.mark.parametrize("params", [(5, 8, 128), (3, 7, 65), (2, 4, 200), (1, 12, 64),
                                    (4, 8, 300), (6, 16, 128), (1, 1, 1), (8, 2, 1024)])
def test_non_default_hash_shapes(oracle, params):
    p = bm.HashParams(*params)
    hf = bm.make_hash_functions(99, p)
    oc_c, oc_f = oracle.make_hash_functions(99, *params)
    assert same_bits(hf.coarse, oc_c) and same_bits(hf.fine, oc_f)
    rng = np.random.default_rng(sum(params))
    d = unit_rows(rng, 777)
    mean = (0.02 * rng.standard_normal(128)).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(1, d), hf, mean)
    oc = oracle.compute_codes(d, hf.coarse, hf.fine, mean)
    assert np.array_equal(cs.coarse, oc[0])
    assert np.array_equal(cs.fine, oc[1])


def test_sift_like_nonnegative_inputs(hf, oracle):
    # SIFT-like: non-negative, 0.2-clipped, renormalised, then quantised
    rng = np.random.default_rng(3)
    d = np.abs(rng.standard_normal((4096, 128))).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = np.minimum(d, 0.2)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = (np.round(d * 512) / 512).astype(np.float32)
    with bm.Matcher(hf) as m:
        m.upload(0, d[:2048])
        m.upload(1, d[2048:])
        m.row([0, 1])
        mean = m.row_mean()
        assert same_bits(mean, oracle.row_mean([d[:2048], d[2048:]]))
        cs = m.codes(1, 2048)
        oc = oracle.compute_codes(d[2048:], hf.coarse, hf.fine, mean)
        assert np.array_equal(cs.coarse, oc[0]) and np.array_equal(cs.fine, oc[1])


def test_extreme_rows_codes_match_oracle(hf, oracle):
    # the tensor-core projection quantises every row on its own power-of-two
    # scale: huge, tiny, mixed-magnitude, subnormal, zero and non-finite rows
    # must still give the reference's bits (non-finite rows take the FP64 path)
    rng = np.random.default_rng(11)
    d = unit_rows(rng, 1024)
    d[0:8] *= np.float32(1e30)
    d[8:16] *= np.float32(1e-30)
    d[16:24, :64] *= np.float32(1e12)
    d[24:32, 1::2] *= np.float32(1e-12)
    d[32:36] = 0.0
    d[36:40, :4] = np.float32(1e-44)
    d[40, 7] = np.nan
    d[41, 100] = np.inf
    d[42, 3] = -np.inf
    d[43:45] = np.float32(3e38) * np.sign(d[43:45])
    mean = (0.01 * rng.standard_normal(128)).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(4, d), hf, mean)
    oc = oracle.compute_codes(d, hf.coarse, hf.fine, mean)
    assert np.array_equal(cs.coarse, oc[0])
    assert np.array_equal(cs.fine, oc[1])


@pytest.mark.parametrize("scale", [1.0, 1e-20, 1e20])
def test_row_scale_invariance_of_codes(hf, oracle, scale):
    # signs of d.p - m.p for rows and mean scaled together
    rng = np.random.default_rng(12)
    d = (unit_rows(rng, 600) * np.float32(scale)).astype(np.float32)
    mean = (0.05 * scale * rng.standard_normal(128)).astype(np.float32)
    cs = bm.compute_codes(bm.FeatureSet(5, d), hf, mean)
    oc = oracle.compute_codes(d, hf.coarse, hf.fine, mean)
    assert np.array_equal(cs.coarse, oc[0]) and np.array_equal(cs.fine, oc[1])
