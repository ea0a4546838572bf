"""SURVEY §8f rows f2 / f3 measured: feature-file ingestion (read_features,
features.cpp:222-249) and match-file output (write_matches_binary,
hashmatch.cpp:311-332), native libbmg vs the compiled reference, on the
host of the GPU box.  Files live in a scratch dir (page cache warm after the
first pass: the numbers are the parsing / copy cost, not the disk's).

usage: python tests/probes/io_bench.py [n_files] [ppi] [out.json]"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_2505_22089_b200 as bm  # noqa: E402
from paper_2505_22089_b200 import features as F  # noqa: E402
from oracle_lib import Reference  # noqa: E402  (checker / CPU baseline only)

n_files = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ppi = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
out_json = sys.argv[3] if len(sys.argv) > 3 else None
ref = Reference()
rng = np.random.default_rng(0)
tmp = Path(tempfile.mkdtemp(prefix="bmg_io_"))
files = []
for i in range(n_files):
    d = rng.standard_normal((ppi, 128)).astype(np.float32)
    k = rng.standard_normal((ppi, 4)).astype(np.float32)
    p = tmp / f"img{i:05d}.feat"
    ref.write_features(p, i, d, k)
    files.append(p)
total = sum(p.stat().st_size for p in files)
keep = []


def pinned(nbytes):
    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    keep.append(t)
    return t.numpy()


def timed(fn, reps=3):
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


res = {"files": n_files, "ppi": ppi, "bytes": total, "cores": os.cpu_count(), "page_cache": "warm"}
for th in (1, 8, 16):
    s = timed(lambda: [F.read_features(p, threads=th) for p in files])
    res[f"native_read_t{th}_gbs"] = total / s / 1e9
if torch.cuda.is_available():
    # straight into pinned staging buffers allocated once (the H2D source)
    bufs = [pinned(ppi * 128 * 4) for _ in files]
    s = timed(lambda: [F.read_features(p, pinned=lambda n, b=b: b, threads=16) for p, b in zip(files, bufs)])
    res["native_read_into_pinned_t16_gbs"] = total / s / 1e9
    # files -> HBM: read into pinned staging, then the arena's H2D
    hf = bm.make_hash_functions(bm.seed_for(42, "matching"))
    arena = bm.DeviceArena(ppi * n_files, hf)

    def ingest():
        for i, (p, b) in enumerate(zip(files, bufs)):
            fs = F.read_features(p, pinned=lambda n, b=b: b, threads=16)
            arena.upload(i, fs.descriptors)
        arena.matcher.synchronize()
        for i in range(n_files):
            arena.evict(i)
        arena.matcher.synchronize()
    ingest()
    s = timed(ingest)
    res["files_to_hbm_gbs"] = total / s / 1e9
    keep.clear()
s = timed(lambda: [ref.read_features(p) for p in files], reps=1)
res["reference_read_gbs"] = total / s / 1e9
# parity on this data
a = F.read_features(files[-1])
b = ref.read_features(files[-1])
assert a.image_id == b[0] and np.array_equal(a.descriptors.view(np.uint32), b[1].view(np.uint32))

# BMMT: a shard16k-sized result (9,480 pairs x ~5.9k matches)
n_pairs, per = 9480, 5900
pairs = [(i // 15, i // 15 + 1 + i % 15, None) for i in range(n_pairs)]
qi = np.arange(per, dtype=np.int32)
plist, pm = [], []
for q, t, _ in pairs:
    m = np.stack([qi, rng.integers(0, ppi, per).astype(np.int32)], 1)
    plist.append((q, t, m))
    pm.append(bm.PairMatches(q, t, m))
o, r = tmp / "ours.bin", tmp / "ref.bin"
s_o = timed(lambda: bm.write_matches_binary(o, pm))
# the execute_plan result path: flat pinned-log arrays straight to the writer
import ctypes as C  # noqa: E402
from paper_2505_22089_b200 import _lib  # noqa: E402
ids = np.array([(q, t) for q, t, _ in plist], np.uint64).reshape(-1)
ends = np.cumsum([per] * n_pairs, dtype=np.uint64)
rngs = np.stack([ends - per, ends], 1).reshape(-1).astype(np.uint64)
log = np.ascontiguousarray(np.concatenate([m for _, _, m in plist]))
L = _lib.load()
s_f = timed(lambda: _lib.check(L.bmg_write_matches_binary(str(o).encode(), n_pairs, ids.ctypes.data,
                                                           rngs.ctypes.data, log.ctypes.data, None)))
res["native_bmmt_write_flat_gbs"] = o.stat().st_size / s_f / 1e9
s_r = timed(lambda: ref.write_matches_binary(r, plist), reps=1)
assert o.read_bytes() == r.read_bytes()
mb = o.stat().st_size
res.update({"bmmt_bytes": mb, "native_bmmt_write_gbs": mb / s_o / 1e9, "reference_bmmt_write_gbs": mb / s_r / 1e9})
for p in files + [o, r]:
    p.unlink()
tmp.rmdir()
print(json.dumps(res))
if out_json:
    Path(out_json).write_text(json.dumps(res, indent=1))
