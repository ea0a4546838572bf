"""Feature ingestion on the execute_plan path: images
streamed from .feat files as they upload (bmg_execute_plan_files) and from
pageable host arrays through the threaded pinned staging slots must give the
same matches and arena counters as pinned in-memory features -- and the
reference's."""
import numpy as np
import pytest

import paper_2505_22089_b200 as bm
from paper_2505_22089_b200 import engine, multigpu
from paper_2505_22089_b200.features import write_features

pytestmark = pytest.mark.gpu


def scene(reference, tmp_path, n=18, ppi=4000, band=4):
    imgs, pairs, kps = reference.generate_synthetic(n, ppi, band, 0.02, 0.2, 31, keypoints=True)
    plan_path = tmp_path / "plan.json"
    reference.iterate_schedule(np.arange(n), pairs, 4, 8, plan_path)
    return imgs, kps, bm.read_plan(plan_path), plan_path


def test_files_equal_memory_and_reference(reference, tmp_path):
    imgs, kps, plan, plan_path = scene(reference, tmp_path)
    files = {}
    for i, (d, k) in enumerate(zip(imgs, kps)):
        fs = bm.FeatureSet(i, d, k)
        files[i] = tmp_path / f"img{i:04d}.feat"
        write_features(files[i], fs)
    hseed = bm.seed_for(42, "matching")
    hf = bm.make_hash_functions(hseed)
    feats = {i: bm.FeatureSet(i, d) for i, d in enumerate(imgs)}
    cap = engine.arena_units_for(feats, plan.size_gpu)
    mem = bm.execute_plan(plan, feats, bm.DeviceArena(cap, hf))
    ups = []
    fil = bm.execute_plan(plan, {i: str(p) for i, p in files.items()}, bm.DeviceArena(cap, hf),
                          bm.ExecuteOptions(on_upload=lambda i, n: ups.append((i, n))))
    for a, b in zip(multigpu.result_flat(mem), multigpu.result_flat(fil)):
        assert np.array_equal(a, b)
    assert fil.metrics.uploads == mem.metrics.uploads == len(ups)
    assert fil.metrics.units_uploaded == mem.metrics.units_uploaded
    _, _, _, ref = reference.execute_plan_rows(plan_path, dict(enumerate(imgs)), hseed, want_matches=True)
    for a, b in zip(multigpu.result_flat(fil), ref):
        assert np.array_equal(a, b)


def test_damaged_files_fail_like_the_reference_reader(reference, tmp_path):
    imgs, kps, plan, _ = scene(reference, tmp_path, n=8, ppi=600, band=2)
    files = {}
    for i, (d, k) in enumerate(zip(imgs, kps)):
        files[i] = tmp_path / f"img{i}.feat"
        write_features(files[i], bm.FeatureSet(i, d, k))
    hf = bm.make_hash_functions(5)
    paths = {i: str(p) for i, p in files.items()}
    views = engine._feature_views(paths)  # headers read (and counts taken) here
    # truncate one file after its header was read: the upload must fail
    raw = files[3].read_bytes()
    files[3].write_bytes(raw[: len(raw) - 700])
    with pytest.raises(bm.BandmatchError) as e:
        bm.execute_plan(plan, paths, bm.DeviceArena(10 ** 9, hf), views=views)
    assert e.value.code == "TruncatedFile"
    files[3].write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(bm.BandmatchError) as e:
        bm.execute_plan(plan, paths, bm.DeviceArena(10 ** 9, hf), views=views)
    assert e.value.code == "FormatError"
    # a file whose count disagrees with the planned one
    files[3].write_bytes(raw)
    write_features(files[3], bm.FeatureSet(3, imgs[3][:100], kps[3][:100]))
    with pytest.raises(bm.BandmatchError) as e:
        bm.execute_plan(plan, paths, bm.DeviceArena(10 ** 9, hf), views=views)
    assert e.value.code == "InvalidArgument"


def test_pageable_staging_equals_pinned(reference, tmp_path):
    import torch
    imgs, _, plan, _ = scene(reference, tmp_path, n=16, ppi=9000, band=5)
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    pinned = {}
    for i, d in enumerate(imgs):
        t = torch.empty(d.shape, dtype=torch.float32, pin_memory=True)
        t.numpy()[...] = d
        pinned[i] = bm.FeatureSet(i, t.numpy())
    page = {i: bm.FeatureSet(i, np.array(d)) for i, d in enumerate(imgs)}
    cap = engine.arena_units_for(page, plan.size_gpu)
    a = bm.execute_plan(plan, pinned, bm.DeviceArena(cap, hf))
    b = bm.execute_plan(plan, page, bm.DeviceArena(cap, hf))
    for x, y in zip(multigpu.result_flat(a), multigpu.result_flat(b)):
        assert np.array_equal(x, y)


def test_mixed_pinned_pageable_unaligned_and_oversized_sources(reference, tmp_path):
    """The staging packs consecutive pageable images into one pinned slot per
    fork-join and sends pinned ones straight to the copy engine: a plan whose
    images alternate between the two, with pageable arrays at odd (4-byte,
    not 16-byte) addresses, odd counts and one image larger than a staging
    slot (16 MiB), gives the pinned-only result."""
    import torch
    imgs, _, plan, _ = scene(reference, tmp_path, n=12, ppi=3001, band=4)
    big = np.concatenate([imgs[5]] * 12)  # ~36k descriptors: 18 MB > one slot
    big = big[: (16 << 20) // 512 + 777]
    imgs = [big if i == 5 else d for i, d in enumerate(imgs)]
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    pinned = {}
    for i, d in enumerate(imgs):
        t = torch.empty(d.shape, dtype=torch.float32, pin_memory=True)
        t.numpy()[...] = d
        pinned[i] = bm.FeatureSet(i, t.numpy())
    mixed = {}
    for i, d in enumerate(imgs):
        if i % 3 == 1:
            mixed[i] = pinned[i]
        else:
            buf = np.empty(d.size + 1, np.float32)  # one float of offset: 4-byte aligned source
            view = buf[1:].reshape(d.shape)
            view[...] = d
            assert view.ctypes.data % 16 != 0
            mixed[i] = bm.FeatureSet(i, view)
    cap = engine.arena_units_for(pinned, plan.size_gpu)
    a = bm.execute_plan(plan, pinned, bm.DeviceArena(cap, hf))
    b = bm.execute_plan(plan, mixed, bm.DeviceArena(cap, hf))
    for x, y in zip(multigpu.result_flat(a), multigpu.result_flat(b)):
        assert np.array_equal(x, y)
    assert a.metrics.uploads == b.metrics.uploads
