"""bench.py's sampled parity leg (used for the long plans, shard16k / config
4): the reference runs the plan's last block row with its whole needed set on
its first pairs, and those pairs' match lists are compared with the run's.
Checked here against the reference's own full run (equal) and a corrupted
copy (DIFFERENT), on a small block plan."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def test_sampled_parity_detects_equal_and_different(reference, tmp_path):
    imgs, _ = reference.generate_synthetic(43, 1024, 11, 0.02, 0.2, 7)
    images = {i - 11: d for i, d in enumerate(imgs) if i >= 11}
    hseed = reference.seed_for(bench.HASH_ROOT_SEED, "matching")
    plan = bench.ROOT / "bench_data" / "plan_block32.json"
    _, _, _, full = reference.execute_plan_rows(plan, images, hseed, threads=4, want_matches=True)
    ok = bench.sampled_parity(reference, hseed, images, plan, full, 4, n_pairs=12)
    assert ok["status"] == "equal" and ok["pairs"] == 12 and ok["digest_gpu"] == ok["digest_reference"]
    ids, offs, m = full
    bad = (ids, offs, m.copy())
    bad[2][:, 1] += 1  # every train index shifted
    assert bench.sampled_parity(reference, hseed, images, plan, bad, 4, n_pairs=12)["status"] == "DIFFERENT"
    # a pair missing from the run's result is a difference too
    keep = np.ones(len(ids), bool)
    last = bench.json.loads(plan.read_text())["iterations"][-1]["rows"][-1]["blocks"][0]["pairs"][0]
    keep[[p for p, (a, b) in enumerate(ids) if (int(a), int(b)) == tuple(last)]] = False
    cnt = np.diff(offs)[keep]
    offs2 = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    m2 = np.concatenate([m[offs[p]:offs[p + 1]] for p in range(len(ids)) if keep[p]])
    assert bench.sampled_parity(reference, hseed, images, plan, (ids[keep], offs2, m2), 4, n_pairs=12)["status"] == "DIFFERENT"
