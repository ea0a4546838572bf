"""Parity at the sizes the bench reports and on the edges the fast paths
certify, against the compiled reference (oracle/_ref) or the C restatement:

(a) BASELINE config 2 at full size (32 x 8,190 descriptors, 286 pairs, the
    committed iterate_schedule(16, 32) plan) through the public execute_plan;
(b) a 16,384-descriptor multi-row, multi-iteration MBR plan;
(c) ratio > 1 with near-tied top-2 distances (hashmatch.cpp:47-49 accepts any
    ratio; the FP32 certificate must not pick a different argmin);
(d) fine_bits != 128 and coarse_bits > 12 through match_pair;
(e) crafted inputs that force the exact top-K walk and the FP64 re-rank band,
    asserting that those paths ran;
plus the GPU branch of execute_plan_distributed (one process per rank, here
two ranks sharing the one GPU) against the reference.
"""
import os
import socket
from pathlib import Path

import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import FeatureSet, HashCodeSet, HashParams, MatchParams, engine
from paper_2505_22089_b200 import hashmatch, multigpu

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def unit_rows(rng, n):
    d = rng.standard_normal((n, 128)).astype(np.float32)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return np.ascontiguousarray(d, np.float32)


def flat_of(res):
    return multigpu.result_flat(res)


def assert_same(gpu, ref):
    gi, go, gm = gpu
    ri, ro, rm = ref
    assert np.array_equal(gi, ri)
    for p in range(len(ri)):
        assert np.array_equal(gm[go[p]:go[p + 1]], rm[ro[p]:ro[p + 1]]), tuple(ri[p])
    assert np.array_equal(go, ro)


# ---- (a) config 2 at full size ---------------------------------------------
def test_config2_full_size_equals_reference(reference):
    table = reference.synth_features(43, 8192, 11, 0.02, 0.2, 7, drop=11)
    images, _ = reference.generate_synthetic(43, 8192, 11, 0.02, 0.2, 7)
    images = images[11:]
    plan_path = ROOT / "bench_data" / "plan_block32.json"
    hseed = bm.seed_for(42, "matching")
    _, _, _, ref = reference.execute_plan_rows(plan_path, table, hseed, want_matches=True)
    table.free()
    plan = bm.read_plan(plan_path)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(images)}
    assert min(len(d) for d in images) == 8190
    arena = bm.DeviceArena(engine.arena_units_for(feats, plan.size_gpu), bm.make_hash_functions(hseed))
    res = bm.execute_plan(plan, feats, arena)
    assert res.metrics.pairs_matched == 286
    assert_same(flat_of(res), ref)
    assert len(ref[2]) > 500_000


# ---- (b) 16k descriptors, several rows and iterations ----------------------
def test_16k_multi_row_multi_iteration_plan_equals_reference(reference, tmp_path):
    n, band = 14, 4
    imgs, pairs = reference.generate_synthetic(n, 16384, band, 0.02, 0.2, 21)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(n), pairs, 3, 6, plan_path)
    plan = bm.read_plan(plan_path)
    assert sum(len(it.rows) for it in plan.iterations) >= 3
    assert len(plan.iterations) >= 2
    hseed = bm.seed_for(42, "matching")
    _, _, _, ref = reference.execute_plan_rows(plan_path, dict(enumerate(imgs)), hseed,
                                               want_matches=True)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    arena = bm.DeviceArena(engine.arena_units_for(feats, plan.size_gpu), bm.make_hash_functions(hseed))
    res = bm.execute_plan(plan, feats, arena)
    assert res.metrics.pairs_matched == plan.pair_count()
    assert_same(flat_of(res), ref)


@pytest.mark.parametrize("n", [1024, 4096, 32768])
def test_descriptor_count_sweep_sizes_equal_reference(reference, tmp_path, n):
    """BASELINE config 5's descriptor counts (tools/sweep.py, 1k..32k per
    image): a band-2 scene of 8 images scheduled by the reference, through
    execute_plan, against the reference row body."""
    imgs, pairs = reference.generate_synthetic(8, n, 2, 0.02, 0.2, 5 + n)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(8), pairs, 4, 8, plan_path)
    hseed = bm.seed_for(42, "matching")
    _, _, _, ref = reference.execute_plan_rows(plan_path, dict(enumerate(imgs)), hseed, threads=8,
                                               want_matches=True)
    plan = bm.read_plan(plan_path)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    arena = bm.DeviceArena(engine.arena_units_for(feats, plan.size_gpu), bm.make_hash_functions(hseed))
    res = bm.execute_plan(plan, feats, arena)
    assert res.metrics.pairs_matched == plan.pair_count() > 0
    assert_same(flat_of(res), ref)


def test_row_body_equals_single_thread_execute_plan(reference, tmp_path):
    """The threaded reference row body (the bench's CPU leg and the checker
    above) against the reference execute_plan as shipped."""
    imgs, pairs = reference.generate_synthetic(10, 700, 3, 0.02, 0.2, 4)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(10), pairs, 2, 4, plan_path)
    hseed = bm.seed_for(42, "matching")
    one, _, _ = reference.execute_plan(plan_path, dict(enumerate(imgs)), hseed)
    _, _, _, (ids, offs, m) = reference.execute_plan_rows(plan_path, dict(enumerate(imgs)), hseed,
                                                          threads=3, want_matches=True)
    assert [tuple(map(int, x)) for x in ids] == sorted(one)
    for p, key in enumerate(sorted(one)):
        assert np.array_equal(m[offs[p]:offs[p + 1]], one[key])


# ---- (c) ratio > 1 with near ties --------------------------------------------
def near_tie_pair(rng, n_q, copies, scale=1e-3):
    """Each query q gets `copies` train points q + scale * P_k(v): the same
    offset vector with its coordinates permuted, so all are at the same real
    distance from q and differ only by float rounding -- ties or near ties
    in FP64, ordered arbitrarily in FP32."""
    q = unit_rows(rng, n_q)
    t = []
    for i in range(n_q):
        v = rng.standard_normal(128)
        v /= np.linalg.norm(v)
        for _ in range(copies):
            t.append(q[i] + scale * rng.permutation(v))
    t = np.asarray(t, np.float32)
    perm = rng.permutation(len(t))
    return q, np.ascontiguousarray(t[perm], np.float32)


@pytest.mark.parametrize("ratio", [1.5, 2.0, 1.0, 0.999999])
def test_ratio_above_one_with_near_ties(oracle, ratio):
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(int(ratio * 1000))
    q, t = near_tie_pair(rng, 1500, 3)
    mean = oracle.row_mean([q, t])
    qf, tf = FeatureSet(1, q), FeatureSet(2, t)
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    mp = MatchParams(8, ratio)
    got = bm.match_pair(qf, qc, tf, tc, mp, hf=hf)
    ref = oracle.match_pair(q, (qc.coarse, qc.fine), t, (tc.coarse, tc.fine), (6, 8, 128), 8, ratio)
    assert np.array_equal(got.matches, ref)
    if ratio > 1:
        assert len(ref) > 1000  # near ties are accepted, so the argmin identity matters
        _, rerank = hashmatch._matcher_for(hf).fixup_counts()
        assert rerank > 0  # uncertified argmins went to the FP64 path


@pytest.mark.parametrize("ratio", [0.0, -0.5, float("nan"), float("inf")])
def test_degenerate_ratios_keep_only_what_the_reference_keeps(oracle, ratio):
    # d1 < d2 * ratio (hashmatch.cpp:47-49): never true for ratio <= 0 or
    # NaN, so only lone candidates survive; inf accepts unless d2 = 0
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(5)
    base = unit_rows(rng, 2000)
    q = base[:1500] + 0.02 * rng.standard_normal((1500, 128)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qf, tf = FeatureSet(1, q), FeatureSet(2, base)
    mean = oracle.row_mean([q, base])
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    got = bm.match_pair(qf, qc, tf, tc, MatchParams(8, ratio), hf=hf)
    ref = oracle.match_pair(q, (qc.coarse, qc.fine), base, (tc.coarse, tc.fine), (6, 8, 128), 8, ratio)
    assert np.array_equal(got.matches, ref)


# ---- (d) other hash shapes through matching ----------------------------------
@pytest.mark.parametrize("params", [(6, 8, 64), (6, 8, 200), (6, 8, 300), (3, 8, 1024), (6, 13, 128),
                                    (4, 16, 64), (2, 12, 1), (12, 6, 128)])
def test_match_with_other_hash_shapes(oracle, params):
    p = HashParams(*params)
    hf = bm.make_hash_functions(77, p)
    rng = np.random.default_rng(sum(params))
    base = unit_rows(rng, 4000)
    q = base[:3000] + 0.03 * rng.standard_normal((3000, 128)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    qf, tf = FeatureSet(1, q), FeatureSet(2, base)
    mean = oracle.row_mean([q, base])
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    oq = oracle.compute_codes(q, hf.coarse, hf.fine, mean)
    assert np.array_equal(qc.coarse, oq[0]) and np.array_equal(qc.fine, oq[1])
    for k in (8, 3, 1):
        got = bm.match_pair(qf, qc, tf, tc, MatchParams(k, 0.7), hf=hf)
        ref = oracle.match_pair(q, (qc.coarse, qc.fine), base, (tc.coarse, tc.fine), params, k, 0.7)
        assert np.array_equal(got.matches, ref), k


def test_fine_bits_above_1024_is_unsupported():
    with pytest.raises(bm.BandmatchError) as e:
        bm.Matcher(bm.make_hash_functions(3, HashParams(2, 8, 1025)))
    assert e.value.code == "Unsupported"


# ---- (e) the rare paths, forced --------------------------------------------
@pytest.mark.parametrize("force", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("k", [8, 3, 16])
def test_forced_exact_paths_equal_oracle(oracle, force, k):
    """Every query through the exact top-K walk (the path a lane's dropped
    key triggers) and / or every ratio decision through the FP64 re-rank (the
    path near ties take): those rare paths, exercised on every query, must
    give the reference's lists and report that they ran."""
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(k)
    base = unit_rows(rng, 3000)
    q = base[:2000] + 0.03 * rng.standard_normal((2000, 128)).astype(np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    # 300 exact copies: Hamming-0 candidates reached from every table
    q[:300] = base[:300]
    qf, tf = FeatureSet(1, q), FeatureSet(2, base)
    mean = oracle.row_mean([q, base])
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    m = hashmatch._matcher_for(hf)
    m.set_test_flags(*force)
    try:
        got = bm.match_pair(qf, qc, tf, tc, MatchParams(k, 0.8), hf=hf)
        walks = m.exact_walk_count()
        _, reranks = m.fixup_counts()
    finally:
        m.set_test_flags(False, False)
    ref = oracle.match_pair(q, (qc.coarse, qc.fine), base, (tc.coarse, tc.fine), (6, 8, 128), k, 0.8)
    assert np.array_equal(got.matches, ref)
    if force[0] and k <= 8:  # k > 8 always takes the exact walk
        assert walks == 2000
    if force[1]:
        assert reranks > 1500  # every query with >= 2 kept candidates


def test_fp64_rerank_band_runs_and_matches(oracle):
    """d1 = ratio * d2 to within float rounding: the FP32 certificate cannot
    decide, the FP64 reference path must."""
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    rng = np.random.default_rng(11)
    n = 1200
    q = unit_rows(rng, n)
    t = []
    for i in range(n):
        v = rng.standard_normal(128)
        v /= np.linalg.norm(v)
        t.append(q[i] + 1e-3 * v)
        t.append(q[i] + 2e-3 * rng.permutation(v))  # exactly twice as far in real arithmetic
    t = np.asarray(t, np.float32)
    mean = oracle.row_mean([q, t])
    qf, tf = FeatureSet(1, q), FeatureSet(2, t)
    qc = bm.compute_codes(qf, hf, mean)
    tc = bm.compute_codes(tf, hf, mean)
    got = bm.match_pair(qf, qc, tf, tc, MatchParams(2, 0.5), hf=hf)
    ref = oracle.match_pair(q, (qc.coarse, qc.fine), t, (tc.coarse, tc.fine), (6, 8, 128), 2, 0.5)
    assert np.array_equal(got.matches, ref)
    _, rerank = hashmatch._matcher_for(hf).fixup_counts()
    assert rerank > 100


# ---- the sharded executor's GPU branch -----------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dist_worker(rank, world, port, plan_path, n_img, seed, queue):
    import sys

    import torch.distributed as dist
    sys.path.insert(0, str(ROOT))
    import paper_2505_22089_b200 as bmw
    from paper_2505_22089_b200 import multigpu as mg
    from paper_2505_22089_b200.features import SyntheticScene, generate_synthetic
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = bmw.read_plan(plan_path)
    sub = mg.shard_plan(plan, world)[rank]
    imgs, _ = generate_synthetic(SyntheticScene(n_img, 2000, 5, 0.02, 0.2, seed),
                                 keep=mg.needed_images(sub))  # only this rank's images
    feats = {i: fs for i, fs in enumerate(imgs) if fs is not None}
    hf = bmw.make_hash_functions(bmw.seed_for(42, "matching"))
    res = mg.execute_plan_distributed(plan, feats, hf, 10 ** 9, device=0, tag=f"gpu{port}")
    if rank == 0:
        ids, offs, m = res.matches.flat()
        queue.put((ids.copy(), offs.copy(), m.copy(), res.metrics.pairs_matched))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_distributed_gpu_branch_equals_reference(reference, tmp_path, world):
    import torch.multiprocessing as mp
    n_img, seed = 30, 13
    imgs, pairs = reference.generate_synthetic(n_img, 2000, 5, 0.02, 0.2, seed)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(n_img), pairs, 6, 12, plan_path)
    _, _, _, ref = reference.execute_plan_rows(plan_path, dict(enumerate(imgs)),
                                               bm.seed_for(42, "matching"), want_matches=True)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dist_worker, args=(r, world, port, plan_path, n_img, seed, q))
             for r in range(world)]
    for p in procs:
        p.start()
    ids, offs, m, n_pairs = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert n_pairs == len(pairs)
    assert_same((ids, offs, m), ref)
