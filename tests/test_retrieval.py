"""Retrieval, host side: the C restatement of
encode_vlad (oracle.c) against the compiled reference (retrieval.cpp:160-205)
on random and adversarial inputs, and the codebook file format
(retrieval.cpp:407-450).  The GPU encoder is checked in test_gpu_retrieval.py."""
import numpy as np
import pytest

from oracle_lib import Oracle, Reference, RefError
from paper_2505_22089_b200 import BandmatchError, Codebook, read_codebook, write_codebook


@pytest.fixture(scope="module")
def orc():
    return Oracle()


@pytest.fixture(scope="module")
def ref():
    try:
        return Reference()
    except FileNotFoundError as e:
        pytest.skip(str(e))


def vlad_cases(rng):
    """(name, descriptors, centroids) covering the ties and edge cases."""
    unit = lambda a: (a / np.linalg.norm(a, axis=1, keepdims=True)).astype(np.float32)
    c64 = unit(rng.standard_normal((64, 128)))
    d = unit(rng.standard_normal((700, 128)))
    cases = [("random", d, c64), ("k1", d[:50], c64[:1]), ("k100", d, unit(rng.standard_normal((100, 128)))),
             ("empty", np.zeros((0, 128), np.float32), c64)]
    dup = c64.copy()
    dup[7] = dup[3]                       # duplicate centroid: exact FP64 tie, first index wins
    cases.append(("dup_centroid", np.concatenate([d[:100], dup[[3, 7, 3]]]), dup))
    eq = np.concatenate([c64[:20], c64[:20]])  # descriptors equal to centroids: distance 0
    cases.append(("on_centroid", eq, c64))
    mid = ((c64[:10] + c64[10:20]) * 0.5).astype(np.float32)  # near-equidistant points
    cases.append(("midpoints", mid, c64))
    cases.append(("single_cluster_zero", np.repeat(c64[:1], 5, 0), c64))  # residuals 0 -> degenerate
    tiny = (c64 * np.float32(1e-21)).astype(np.float32)  # squared distances underflow in FP32
    cases.append(("tiny", (d[:64] * np.float32(1e-21)).astype(np.float32), tiny))
    big = (c64 * np.float32(1e19)).astype(np.float32)   # squared distances overflow in FP32
    cases.append(("huge", (d[:64] * np.float32(1e19)).astype(np.float32), big))
    sift = np.maximum(rng.standard_normal((300, 128)), 0).astype(np.float32)
    sift = np.minimum(unit(sift + 1e-6), 0.2)
    cases.append(("sift_like", unit(sift), unit(np.abs(rng.standard_normal((64, 128))))))
    return cases


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint32), np.asarray(b).view(np.uint32))


def test_oracle_encode_vlad_equals_reference(orc, ref):
    rng = np.random.default_rng(160)
    for name, d, c in vlad_cases(rng):
        ov, od = orc.encode_vlad(d, c)
        rv, rd = ref.encode_vlad(d, c)
        assert od == rd, name
        assert same(ov, rv), name


def test_oracle_encode_vlad_degenerate_flags(orc):
    rng = np.random.default_rng(1)
    c = rng.standard_normal((4, 128)).astype(np.float32)
    v, dg = orc.encode_vlad(np.zeros((0, 128), np.float32), c)
    assert dg and not v.any()
    v, dg = orc.encode_vlad(np.repeat(c[:1], 3, 0), c)
    assert dg and not v.any()
    v, dg = orc.encode_vlad(rng.standard_normal((9, 128)).astype(np.float32), c)
    assert not dg and abs(float(np.dot(v.astype(np.float64), v)) - 1.0) < 1e-5


def test_reference_batch_equals_single(ref):
    rng = np.random.default_rng(2)
    c = rng.standard_normal((16, 128)).astype(np.float32)
    imgs = [rng.standard_normal((n, 128)).astype(np.float32) for n in (0, 5, 300, 17)]
    vals, degs = ref.encode_vlad_batch(imgs, c, threads=3)
    for i, d in enumerate(imgs):
        v, dg = ref.encode_vlad(d, c)
        assert dg == degs[i] and same(v, vals[i])


def test_encode_vlad_rejects_empty_codebook(orc, ref):
    with pytest.raises(ValueError):
        orc.encode_vlad(np.zeros((1, 128), np.float32), np.zeros((0, 128), np.float32))
    with pytest.raises(RefError) as e:
        ref.encode_vlad(np.zeros((1, 128), np.float32), np.zeros((0, 128), np.float32))
    assert "codebook has no words" in str(e.value)


def test_codebook_file_roundtrip_and_errors(tmp_path):
    rng = np.random.default_rng(3)
    cb = Codebook(5, rng.standard_normal((5, 128)).astype(np.float32))
    p = tmp_path / "cb.bmcb"
    write_codebook(p, cb)
    raw = p.read_bytes()
    assert raw[:4] == b"BMCB" and len(raw) == 12 + 5 * 128 * 4
    back = read_codebook(p)
    assert back.k_words == 5 and same(back.centroids, cb.centroids)
    (tmp_path / "bad").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(BandmatchError) as e:
        read_codebook(tmp_path / "bad")
    assert e.value.code == "FormatError"
    (tmp_path / "short").write_bytes(raw[:100])
    with pytest.raises(BandmatchError) as e:
        read_codebook(tmp_path / "short")
    assert e.value.code == "TruncatedFile"
    with pytest.raises(BandmatchError) as e:
        write_codebook(tmp_path / "x", Codebook(0, np.zeros((0, 128), np.float32)))
    assert e.value.code == "FormatError"
