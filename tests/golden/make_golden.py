"""Generate tests/golden fixtures by running the UNMODIFIED reference
(oracle/_ref/libbandmatch_ref.so, compiled in place from /root/reference by
oracle/Makefile).  Run here (where the reference exists):

    python tests/golden/make_golden.py

Fixtures:
  hash_functions.npz  planes for (seed, params) cases (make_hash_functions)
  scene_small.npz     5-image band scene: descriptors, plan, per-pair reference
                      execute_plan matches, codes of every image vs. a fixed mean
  pair_8192.npz       BASELINE config 1 pair (generate_synthetic(13, 8192, 11,
                      0.02, 0.2, 7), images 11 & 12): input digests, codes
                      digests, the reference's match list
"""
import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import Reference  # noqa: E402

HASH_CASES = [(42, 6, 8, 128), (12, 6, 8, 128), (99, 5, 8, 128), (99, 3, 7, 65), (7, 1, 1, 1),
              (2 ** 63 + 11, 4, 8, 300)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    r = Reference()
    matching_seed = r.seed_for(42, "matching")
    # hash functions
    out = {"cases": np.array(HASH_CASES, dtype=np.uint64), "matching_seed": np.uint64(matching_seed)}
    for i, (s, t, c, f) in enumerate(HASH_CASES):
        co, fi = r.make_hash_functions(s, t, c, f)
        out[f"coarse_{i}"], out[f"fine_{i}"] = co, fi
    np.savez_compressed(HERE / "hash_functions.npz", **out)

    # small scene through the reference execute_plan
    imgs, pairs = r.generate_synthetic(5, 200, 2, 0.02, 0.2, 7)
    with tempfile.TemporaryDirectory() as td:
        plan_path = Path(td) / "plan.json"
        r.iterate_schedule(np.arange(5), pairs, 2, 4, plan_path)
        plan_text = plan_path.read_text()
        res, counters, _ = r.execute_plan(plan_path, dict(enumerate(imgs)), matching_seed)
    coarse, fine = r.make_hash_functions(matching_seed)
    mean = np.linspace(-0.01, 0.01, 128).astype(np.float32)
    scene = {"plan_json": np.frombuffer(plan_text.encode(), np.uint8),
             "pairs": pairs.astype(np.uint64), "mean": mean,
             "counters": np.array([counters[k] for k in ("pairs_matched", "initial_matches",
                                                         "uploads", "evictions",
                                                         "units_uploaded", "peak_occupancy")],
                                  np.uint64)}
    for i, d in enumerate(imgs):
        scene[f"desc_{i}"] = d
        cc, ff = r.compute_codes(d, coarse, fine, mean, matching_seed)
        scene[f"coarse_{i}"], scene[f"fine_{i}"] = cc, ff
    scene["result_pairs"] = np.array(sorted(res), np.uint64).reshape(-1, 2)
    for (a, b), m in res.items():
        scene[f"matches_{a}_{b}"] = m
    # brute force known answers on the first pair
    scene["brute_0_1"] = r.brute_force_match(imgs[0], imgs[1], 0.5)
    np.savez_compressed(HERE / "scene_small.npz", **scene)

    # BASELINE config 1 pair at full size
    band = 11
    imgs, _ = r.generate_synthetic(band + 2, 8192, band, 0.02, 0.2, 7)
    q, t = imgs[band], imgs[band + 1]
    acc = np.zeros(128, np.float64)
    # row mean of the 2-image row, reference order (engine.cpp:449-461) is
    # produced by the oracle in the tests; here use the reference codes vs.
    # a zero-centred mean and vs. the row mean computed by sequential adds
    for d in (q, t):
        for row in d:
            for c in range(128):
                acc[c] += float(row[c])
    mean_row = (acc / float(len(q) + len(t))).astype(np.float32)
    qc = r.compute_codes(q, coarse, fine, mean_row, matching_seed)
    tc = r.compute_codes(t, coarse, fine, mean_row, matching_seed)
    m = r.match_pair(q, qc, t, tc, (6, 8, 128), seed=matching_seed)
    np.savez_compressed(HERE / "pair_8192.npz", q_sha=sha(q), t_sha=sha(t), mean=mean_row,
                        q_codes_sha=sha(*qc), t_codes_sha=sha(*tc), matches=m,
                        n_q=len(q), n_t=len(t))
    print(json.dumps({"hash_cases": len(HASH_CASES), "scene_pairs": len(res),
                      "pair_8192_matches": len(m)}))


if __name__ == "__main__":
    main()
