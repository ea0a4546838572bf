"""VLAD encoding on the B200 (vlad.cu, bmg_encode_vlad)
against the compiled reference encode_vlad (retrieval.cpp:160-205): values
and degenerate flags bit-for-bit, on a synthetic scene with a codebook the
reference trains, and on the adversarial cases of test_retrieval.py (FP64
ties, zero / underflowing / overflowing distances, NaN, empty images,
codebooks of 1 and 100 words, several upload batches)."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from test_retrieval import same, vlad_cases

pytestmark = pytest.mark.gpu


def check(reference, imgs, cent):
    got = bm.encode_vlad_batch(imgs, bm.Codebook(len(cent), cent))
    vals, degs = reference.encode_vlad_batch(imgs, cent, threads=8)
    for i in range(len(imgs)):
        assert got[i].degenerate == degs[i], i
        assert same(got[i].values, vals[i]), i


def test_adversarial_cases_equal_reference(reference):
    rng = np.random.default_rng(160)
    for name, d, c in vlad_cases(rng):
        g = bm.encode_vlad(d, bm.Codebook(len(c), c))
        v, dg = reference.encode_vlad(d, c)
        assert g.degenerate == dg, name
        assert same(g.values, v), name


def test_nan_descriptor_follows_reference(reference):
    rng = np.random.default_rng(5)
    c = rng.standard_normal((64, 128)).astype(np.float32)
    d = rng.standard_normal((200, 128)).astype(np.float32)
    d[17, 3] = np.nan  # never < best: the reference assigns it to centroid 0
    g = bm.encode_vlad(d, bm.Codebook(64, c))
    v, dg = reference.encode_vlad(d, c)
    assert g.degenerate == dg
    assert np.array_equal(np.isnan(g.values), np.isnan(v))
    assert same(np.nan_to_num(g.values), np.nan_to_num(v))


def test_scene_with_trained_codebook_equals_reference(reference):
    imgs, _ = reference.generate_synthetic(14, 8192, 11, 0.02, 0.2, 7)
    imgs = imgs[11:] + imgs[:3]  # full-size images and the short first ones
    sample = np.concatenate([im[::16] for im in imgs])
    cent, sse = reference.train_codebook(sample, 64, max_iters=10, seed=3)
    assert len(sse) >= 1
    check(reference, imgs, cent)


def test_batches_and_empty_images_equal_reference(reference, monkeypatch):
    rng = np.random.default_rng(9)
    cent = rng.standard_normal((64, 128)).astype(np.float32)
    imgs = [rng.standard_normal((n, 128)).astype(np.float32) for n in (300, 0, 1, 129, 1000, 0, 77)]
    monkeypatch.setenv("BMG_VLAD_BATCH_BYTES", str(400 * 512))  # several batches, both slots reused
    check(reference, imgs, cent)
    monkeypatch.delenv("BMG_VLAD_BATCH_BYTES")
    check(reference, imgs, cent)


def test_errors():
    with pytest.raises(bm.BandmatchError) as e:
        bm.encode_vlad(np.zeros((3, 128), np.float32), bm.Codebook(0, np.zeros((0, 128), np.float32)))
    assert e.value.code == "InvalidArgument" and "codebook has no words" in str(e.value)
    assert bm.encode_vlad_batch([], bm.Codebook(2, np.ones((2, 128), np.float32))) == []


# ---- train_codebook (retrieval.cpp:56-158) ------------------------------------
@pytest.mark.parametrize("n,k,iters,seed", [(2000, 16, 25, 3), (40, 16, 25, 7), (300, 64, 5, 11),
                                            (69, 64, 3, 1), (5000, 64, 25, 42)])
# (69, 64): 5 duplicates leave exactly k = 64 distinct values (the seeding's boundary)
def test_train_codebook_equals_reference(reference, n, k, iters, seed):
    rng = np.random.default_rng(n + k)
    d = rng.standard_normal((n, 128)).astype(np.float32)
    d[n // 3: n // 3 + 5] = d[0]  # duplicates: skipped by the seeding's distinct check
    hist = []
    got = bm.train_codebook(d, k, iters, seed, sse_history=hist)
    cent, sse = reference.train_codebook(d, k, iters, seed)
    assert same(got.centroids, cent)
    assert np.array_equal(np.asarray(hist), sse)


def test_train_codebook_on_scene_sample_equals_reference(reference):
    imgs, _ = reference.generate_synthetic(14, 8192, 11, 0.02, 0.2, 7)
    sample = np.concatenate([im[::13] for im in imgs[11:]])
    hist = []
    got = bm.train_codebook(sample, 64, 10, 3, sse_history=hist)
    cent, sse = reference.train_codebook(sample, 64, 10, 3)
    assert same(got.centroids, cent) and np.array_equal(np.asarray(hist), sse)
    assert all(a >= b for a, b in zip(sse, sse[1:]))  # Lloyd's SSE is non-increasing


def test_train_codebook_errors(reference):
    d = np.random.default_rng(0).standard_normal((10, 128)).astype(np.float32)
    for args, code in [((d, 0, 5, 1), "InvalidArgument"), ((d, 4, 0, 1), "InvalidArgument"),
                       ((d, 11, 5, 1), "TooFewDescriptors"),
                       ((np.repeat(d[:1], 10, 0), 2, 5, 1), "TooFewDescriptors")]:
        with pytest.raises(bm.BandmatchError) as e:
            bm.train_codebook(*args)
        assert e.value.code == code
        with pytest.raises(Exception) as r:
            reference.train_codebook(*args)
        assert code in str(r.value)
