"""Host verification stage 1: libbmg's sao_filter and its
adjacency-driven Bowyer-Watson Delaunay against the reference's own code
(verify.cpp:1-341, compiled from the reference source by oracle/Makefile) on
random, clustered, lattice (cocircular / collinear), duplicated and real
synthetic-scene keypoints.  CPU only."""
import time

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200.verify import SaoParams, knn_from_delaunay, sao_filter


def point_sets():
    rng = np.random.default_rng(7)
    yield "uniform", rng.uniform(0, 1000, (3000, 2))
    yield "clustered", np.concatenate([c + rng.normal(0, 3, (200, 2)) for c in rng.uniform(0, 500, (10, 2))])
    g = np.stack(np.meshgrid(np.arange(30.0), np.arange(30.0)), -1).reshape(-1, 2)
    yield "lattice", g  # every unit square is cocircular
    yield "lattice_permuted", g[rng.permutation(len(g))]
    yield "collinear", np.stack([np.arange(50.0), 2 * np.arange(50.0)], 1)
    yield "duplicates", np.concatenate([rng.uniform(0, 50, (100, 2)), rng.uniform(0, 50, (1, 2)).repeat(2, 0)])
    yield "tiny", rng.uniform(0, 1, (3, 2))
    yield "float32_grid", rng.integers(0, 40, (1500, 2)).astype(np.float32).astype(np.float64) + 0.5 * rng.integers(0, 2, (1500, 2))
    yield "wide_range", np.concatenate([rng.uniform(0, 1e-3, (300, 2)), rng.uniform(0, 1e5, (300, 2))])


@pytest.mark.parametrize("k", [1, 6, 12])
def test_delaunay_knn_equals_reference(reference, k):
    for name, pts in point_sets():
        got, gfb = knn_from_delaunay(pts, k)
        ref, rfb = reference.knn_from_delaunay(pts, k)
        assert gfb == rfb, name
        assert np.array_equal(got, ref), name


def random_sets(rng, count):
    for trial in range(count):
        kind, n = trial % 6, int(rng.integers(4, 800))
        if kind == 0:
            pts = rng.uniform(0, 10 ** rng.uniform(-3, 6), (n, 2))
        elif kind == 1:  # tight clusters
            c = rng.uniform(0, 1000, (max(1, n // 50), 2))
            pts = c[rng.integers(0, len(c), n)] + rng.normal(0, 10 ** rng.uniform(-3, 1), (n, 2))
        elif kind == 2:  # jittered, shuffled lattice: near-cocircular quads
            g = int(np.sqrt(n)) + 1
            pts = np.stack(np.meshgrid(np.arange(g), np.arange(g)), -1).reshape(-1, 2)[:n].astype(float)
            pts = pts[rng.permutation(len(pts))] + rng.normal(0, 10 ** rng.uniform(-8, -1), pts.shape)
        elif kind == 3:  # float32 pixel coordinates, as keypoints are
            pts = rng.uniform(0, 1000, (n, 2)).astype(np.float32).astype(np.float64)
        elif kind == 4:  # near a circle
            t = rng.uniform(0, 2 * np.pi, n)
            pts = np.stack([np.cos(t), np.sin(t)], 1) * 100 + rng.normal(0, 1e-6, (n, 2))
        else:  # two scales (ill-conditioned: the reference's scan runs)
            pts = np.concatenate([rng.uniform(0, 10 ** rng.uniform(-4, 0), (n // 2, 2)),
                                  rng.uniform(0, 1000, (n - n // 2, 2))])
        yield trial, pts, int(rng.integers(1, 10))


def test_delaunay_knn_equals_reference_randomised(reference):
    for trial, pts, k in random_sets(np.random.default_rng(2025), 120):
        got, gfb = knn_from_delaunay(pts, k)
        ref, rfb = reference.knn_from_delaunay(pts, k)
        assert gfb == rfb and np.array_equal(got, ref), trial


def scene_pair(reference, oracle, ppi, band=3, seed=11):
    imgs, _, kps = reference.generate_synthetic(band + 2, ppi, band, 0.02, 0.2, seed, keypoints=True)
    a, b = band, band + 1
    hf = oracle.make_hash_functions(oracle.seed_for(42, "matching"))
    mean = oracle.row_mean([imgs[a], imgs[b]])
    qa = oracle.compute_codes(imgs[a], hf[0], hf[1], mean)
    qb = oracle.compute_codes(imgs[b], hf[0], hf[1], mean)
    m = oracle.match_pair(imgs[a], qa, imgs[b], qb, (6, 8, 128))
    return m, kps[a], kps[b]


@pytest.mark.parametrize("params", [(6, 0.5), (4, 0.3), (8, 1.0), (1, 0.0)])
def test_sao_filter_equals_reference_on_scene_matches(reference, oracle, params):
    m, qk, tk = scene_pair(reference, oracle, 1200)
    assert len(m) > 300
    out = sao_filter(bm.PairMatches(1, 2, m), qk, tk, SaoParams(*params))
    keep, scores, pt, fb = reference.sao_filter(m, qk, tk, *params)
    assert np.array_equal(out.scores, scores)
    assert np.array_equal(out.kept.matches, m[keep])
    assert (out.passthrough, out.delaunay_fallback) == (pt, fb)


def test_sao_filter_edges(reference):
    rng = np.random.default_rng(3)
    qk = np.zeros((50, 4), np.float32)
    qk[:, :2] = rng.uniform(0, 100, (50, 2))
    tk = qk.copy()
    tk[:, :2] = rng.uniform(0, 100, (50, 2))
    m = np.stack([np.arange(50), rng.permutation(50)], 1).astype(np.int32)
    # short input: passthrough
    out = sao_filter(bm.PairMatches(0, 1, m[:5]), qk, tk, SaoParams(6, 0.5))
    assert out.passthrough and len(out.kept.matches) == 5
    # duplicate positions on one side (several matches at one keypoint position)
    qk2 = qk.copy()
    qk2[10:20, :2] = qk2[0, :2]
    for mm, a, b in ((m, qk, tk), (m, qk2, tk), (m, tk, qk2)):
        out = sao_filter(bm.PairMatches(0, 1, mm), a, b, SaoParams(6, 0.4))
        keep, scores, pt, fb = reference.sao_filter(mm, a, b, 6, 0.4)
        assert np.array_equal(out.scores, scores) and np.array_equal(out.kept.matches, mm[keep])
    # errors as the reference raises them
    with pytest.raises(bm.BandmatchError) as e:
        sao_filter(bm.PairMatches(0, 1, m), qk, tk, SaoParams(0, 0.5))
    assert e.value.code == "InvalidArgument"
    with pytest.raises(bm.BandmatchError) as e:
        sao_filter(bm.PairMatches(0, 1, m), qk, tk, SaoParams(6, float("nan")))
    assert e.value.code == "InvalidArgument"
    bad = m.copy()
    bad[3, 1] = 50
    with pytest.raises(bm.BandmatchError) as e:
        sao_filter(bm.PairMatches(0, 1, bad), qk, tk, SaoParams(6, 0.5))
    assert e.value.code == "InvalidArgument"


def test_sao_filter_is_fast_at_scene_scale(reference, oracle):
    """~2,900 matches (an 8k-descriptor pair at ratio 0.5 keeps ~3k): the
    reference's all-triangle Bowyer-Watson vs the adjacency-driven one."""
    m, qk, tk = scene_pair(reference, oracle, 4000)
    t0 = time.perf_counter()
    out = sao_filter(bm.PairMatches(1, 2, m), qk, tk)
    t_fast = time.perf_counter() - t0
    t0 = time.perf_counter()
    keep, scores, _, _ = reference.sao_filter(m, qk, tk)
    t_ref = time.perf_counter() - t0
    assert np.array_equal(out.scores, scores)
    print(f"\nsao_filter {len(m)} matches: {t_fast * 1e3:.1f} ms vs reference {t_ref * 1e3:.1f} ms")
    assert t_fast < t_ref
