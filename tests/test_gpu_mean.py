"""GPU row centering mean (engine.cpp:446-461) through the C ABI against the C
oracle's literal sequential FP64 chain, bit for bit: the parallel F96
reconstruction on ordinary rows, its rounding-step replay on adversarial
rows, and the sequential-chain fallback on rows outside its range."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic

pytestmark = pytest.mark.gpu


def same_bits(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


@pytest.fixture(scope="module")
def hf():
    return bm.make_hash_functions(bm.seed_for(42, "matching"))


def row_mean(hf, imgs):
    with bm.Matcher(hf) as m:
        for i, d in enumerate(imgs):
            m.upload(i, np.ascontiguousarray(d, np.float32))
        m.row(range(len(imgs)))
        return m.row_mean(), m.row_mean_info()


def unit_rows(rng, n):
    d = rng.standard_normal((n, 128)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return d


def test_bench_scale_row(hf, oracle):
    # BASELINE config 2 row 0: 32 images x 8190 descriptors (262,080 rows)
    imgs, _ = generate_synthetic(SyntheticScene(43, 8192, 11, 0.02, 0.2, 7))
    descs = [f.descriptors for f in imgs[11:]]
    mean, (rounds, chained) = row_mean(hf, descs)
    assert same_bits(mean, oracle.row_mean(descs))
    # a few uncertified tiles per channel are walked; no fallback
    assert not chained and 1 <= rounds <= 8


@pytest.mark.parametrize("sizes", [(1,), (127, 1, 129), (0, 5, 0, 300), (4096, 4096, 17)])
def test_random_rows(hf, oracle, sizes):
    rng = np.random.default_rng(sum(sizes))
    imgs = [unit_rows(rng, n) for n in sizes]
    mean, (_, chained) = row_mean(hf, imgs)
    assert same_bits(mean, oracle.row_mean(imgs))
    assert not chained


def test_rounding_steps_replayed(hf, oracle):
    # channel 0: 1.0 then 2^-54 x 3 (each add rounds back); channel 1: ties
    # to even; channel 2: a large cancellation after a rounded step
    d = np.zeros((64, 128), np.float32)
    d[:, 3:] = np.random.default_rng(0).standard_normal((64, 125)).astype(np.float32) * 0.1
    d[0, 0] = 1.0
    d[1:4, 0] = 2.0 ** -54
    d[0, 1], d[1, 1], d[2, 1] = 1.0, 2.0 ** -52, 2.0 ** -53
    d[0, 2], d[1, 2], d[2, 2] = 100.0, 2.0 ** -50, -100.0
    mean, (rounds, chained) = row_mean(hf, [d])
    assert same_bits(mean, oracle.row_mean([d]))
    assert not chained and rounds >= 2  # the tile was walked


def test_many_rounding_steps_replayed(hf, oracle):
    # 39 rounding steps in one tile of channel 5, one step in every tile of
    # channel 7: all replayed exactly, no fallback
    rng = np.random.default_rng(2)
    d = unit_rows(rng, 3000)
    d[0, 5] = 1.0
    d[1:40, 5] = 2.0 ** -54
    d[:, 7] = 0.0
    d[0, 7] = 1.0
    d[1::128, 7] = 2.0 ** -54
    mean, (rounds, chained) = row_mean(hf, [d[:1000], d[1000:]])
    assert same_bits(mean, oracle.row_mean([d[:1000], d[1000:]]))
    assert not chained and rounds >= 20


@pytest.mark.parametrize("case", ["large_value", "subnormal", "tiny"])
def test_chain_fallback(hf, oracle, case):
    rng = np.random.default_rng(2)
    d = unit_rows(rng, 3000)
    if case == "large_value":
        d[17, 9] = 300.0
    elif case == "subnormal":
        d[2999, 0] = np.float32(1e-40)
    else:
        d[100, 127] = np.float32(1e-30)
    mean, (_, chained) = row_mean(hf, [d[:1000], d[1000:]])
    assert same_bits(mean, oracle.row_mean([d[:1000], d[1000:]]))
    assert chained


def test_sift_like_quantised_row(hf, oracle):
    rng = np.random.default_rng(3)
    d = np.abs(rng.standard_normal((20000, 128))).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = np.minimum(d, 0.2)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    d = (np.round(d * 512) / 512).astype(np.float32)
    parts = [d[:7000], d[7000:13000], d[13000:]]
    mean, (_, chained) = row_mean(hf, parts)
    assert same_bits(mean, oracle.row_mean(parts))
    assert not chained
